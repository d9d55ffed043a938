# k_gemm_hm R-row padding (bank conflicts of the R gather): parity and time, with / without
python -c "import __graft_entry__ as g; g.build()"
O=gpurun_out/r5a; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "hm" > $O/pytest.log 2>&1; tail -1 $O/pytest.log
for v in 1 0; do TNB_HM_RPAD=$v timeout 300 python scripts/gemm_shape_bench.py --cls bcbaacaacacababcaabcaaaac --M 3 --kernels 5 --iters 50 2>&1 | grep kernel | sed "s/^/RPAD=$v /"; done
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > $O/bench.json 2> $O/bench.err; python -c "
import json; d=json.load(open('$O/bench.json')); print('C5a', round(d['value'],2), 'e2e', round(d['e2e']['value'],2))"
