# k_gemm with its chunk-load / B' rebuild loops kept rolled (GEMM_U1=1), interleaved A/B; k_gemm_fc now skips the
# constant-offset updates when no constant holds an output bit (124 registers)
O=gpurun_out/r7e; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
C=paper_2012_02430_b200/csrc
relink() { nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O3 $1 -c $C/launch_gemm.cu -o $C/build/launch_gemm.o &&
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o paper_2012_02430_b200/libtnb200.so $C/build/*.o; }
run() { tag=$1; wl=$2; timeout 600 python bench.py --workload $wl --steps 20 --warmup 5 --no-cpu-baseline > $O/bench_$tag.json 2>> $O/bench.err
python -c "
import json; d=json.load(open('$O/bench_$tag.json')); r=d['roofline']; print('$tag $wl', round(d['value'],2), 'e2e', round(d['e2e']['value'],2), r['kernel'], round(r['frac'],3), round(r['avg_launch_ms']*1e3,1), 'us', {k: round(v['ms_share_of_step'],3) for k,v in r.get('families',{}).items()})"; }
run g0_a C5a
relink "-DGEMM_U1=1"; run g1_a C5a
relink ""; run g0_b C5a; run g0_C4b C4b; run g0_C5r C5r
relink "-DGEMM_U1=1"; run g1_b C5a; run g1_C4b C4b; run g1_C5r C5r
timeout 1200 python -m pytest tests -q -m gpu -x -k "gemm or group or feed or fc or C5a or c5a or C2" > $O/pytest_gemm_u1.log 2>&1; tail -2 $O/pytest_gemm_u1.log
