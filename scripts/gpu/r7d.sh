# k_gemm_fc with the consumer step software-pipelined across the tile loop (FC_PIPE=1: the X loads of tile t
# are consumed after the barrier + chunk issue of tile t + 1): parity, then interleaved A/B of the bench line
O=gpurun_out/r7d; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
C=paper_2012_02430_b200/csrc
relink() { nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O3 $1 -c $C/launch_gemm_fc.cu -o $C/build/launch_gemm_fc.o &&
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o paper_2012_02430_b200/libtnb200.so $C/build/*.o; }
run() { tag=$1; timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > $O/bench_$tag.json 2>> $O/bench.err
python -c "
import json; d=json.load(open('$O/bench_$tag.json')); r=d['roofline']; print('$tag C5a', round(d['value'],2), 'e2e', round(d['e2e']['value'],2), r['kernel'], round(r['frac'],3), round(r['avg_launch_ms']*1e3,1), 'us')"; }
timeout 900 python -m pytest tests -q -m gpu -x -k "feed or fc or C5a or c5a or C4b" > $O/pytest_fc_pipe.log 2>&1; tail -2 $O/pytest_fc_pipe.log
run p1_a
relink "-DFC_PIPE=0"; run p0_a
relink "-DFC_PIPE=1"; run p1_b
relink "-DFC_PIPE=0"; run p0_b
relink "-DFC_PIPE=1"
for s in 1 0; do TNB_FC_SPLIT=$s timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > $O/bench_split$s.json 2>> $O/bench.err; python -c "
import json; d=json.load(open('$O/bench_split$s.json')); r=d['roofline']; print('pipe split$s C5a', round(d['value'],2), round(r['avg_launch_ms']*1e3,1), 'us')"; done
