# k_gemm_hm in the product path: full GPU suite, shape timing, C5a bench with / without it
python -c "import __graft_entry__ as g; g.build()"
mkdir -p gpurun_out/r4f
timeout 300 python scripts/gemm_shape_bench.py --cls bcbaacaacacababcaabcaaaac --M 3 --kernels 1,5 > gpurun_out/r4f/shape_top.log 2>&1; tail -2 gpurun_out/r4f/shape_top.log
timeout 300 python scripts/gemm_shape_bench.py --cls abccabcaabcbabaaacaaaaacba --M 3 --kernels 1,5 > gpurun_out/r4f/shape_fcprod.log 2>&1; tail -2 gpurun_out/r4f/shape_fcprod.log
for v in 1 0; do TNB_GEMM_HM=$v timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/r4f/bench_hm$v.json 2> gpurun_out/r4f/bench_hm$v.err; python -c "
import json; d=json.load(open('gpurun_out/r4f/bench_hm$v.json')); r=d['roofline']; print('HM=$v C5a', d['value'], 'e2e', d['e2e']['value'], r['kernel'], r['frac'], {k: (round(v['ms_share_of_step'],3), round(v['GBps'])) for k,v in r['families'].items()})"; done
timeout 2400 python -m pytest tests -q -m gpu -x > gpurun_out/r4f/pytest_gpu.log 2>&1; tail -3 gpurun_out/r4f/pytest_gpu.log
