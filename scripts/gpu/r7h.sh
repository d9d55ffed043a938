# k_gemm_fc with prefetch.global.L1 of the tile's X lines at the tile start (FC_PREFETCH=1) re-measured in the
# final state (124 registers, rolled loops); interleaved A/B
O=gpurun_out/r7h; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
C=paper_2012_02430_b200/csrc
relink() { nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O3 $1 -c $C/launch_gemm_fc.cu -o $C/build/launch_gemm_fc.o &&
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o paper_2012_02430_b200/libtnb200.so $C/build/*.o; }
run() { tag=$1; timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > $O/bench_$tag.json 2>> $O/bench.err
python -c "
import json; d=json.load(open('$O/bench_$tag.json')); r=d['roofline']; print('$tag C5a', round(d['value'],2), 'e2e', round(d['e2e']['value'],2), r['kernel'], round(r['frac'],3), round(r['avg_launch_ms']*1e3,1), 'us')"; }
run pf0_a
relink "-DFC_PREFETCH=1"; run pf1_a
relink ""; run pf0_b
relink "-DFC_PREFETCH=1"; run pf1_b
