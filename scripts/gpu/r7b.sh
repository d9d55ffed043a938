# k_gemm_fc with the chunk-load / B' rebuild loops kept rolled (FC_U1=1: 4,144 vs 6,480 SASS instructions,
# no_instruction stalls were 6.5 % of the issue cycles): interleaved A/B of the bench line
O=gpurun_out/r7b; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
C=paper_2012_02430_b200/csrc
relink() { # $1 = extra -D flags for launch_gemm_fc.cu
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O3 $1 -c $C/launch_gemm_fc.cu -o $C/build/launch_gemm_fc.o &&
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o paper_2012_02430_b200/libtnb200.so $C/build/*.o; }
run() { tag=$1; timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > $O/bench_$tag.json 2>> $O/bench.err
python -c "
import json; d=json.load(open('$O/bench_$tag.json')); r=d['roofline']; print('$tag C5a', round(d['value'],2), 'e2e', round(d['e2e']['value'],2), r['kernel'], round(r['frac'],3), round(r['avg_launch_ms']*1e3,1), 'us')"; }
run u0_a
relink "-DFC_U1=1"; run u1_a
relink ""; run u0_b
relink "-DFC_U1=1"; run u1_b
timeout 900 python -m pytest tests -q -m gpu -x -k "feed or fc or C5a or c5a" > $O/pytest_fc_u1.log 2>&1; tail -2 $O/pytest_fc_u1.log
