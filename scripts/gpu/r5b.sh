# k_gemm_hm64 (c128 on DMMA): parity, c128 configs, c128 bench with / without
python -c "import __graft_entry__ as g; g.build()"
O=gpurun_out/r5b; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "hm64" > $O/pytest_hm64.log 2>&1; tail -3 $O/pytest_hm64.log
for v in 1 0; do TNB_GEMM_HM64=$v timeout 900 python bench.py --steps 10 --warmup 3 --dtype c128 --no-cpu-baseline > $O/bench_c128_hm64$v.json 2> $O/bench_c128_hm64$v.err; python -c "
import json; d=json.load(open('$O/bench_c128_hm64$v.json')); r=d['roofline']; print('HM64=$v C5a c128', round(d['value'],2), r['kernel'], r['bound'], round(r['frac'],3), {k: round(v['ms_share_of_step'],3) for k,v in r['families'].items()})"; done
timeout 1500 python -m pytest tests -q -m gpu -k "c128 or C128 or TN_C128" > $O/pytest_c128.log 2>&1; tail -2 $O/pytest_c128.log
