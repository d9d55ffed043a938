# k_gemm_hm with the truncating TF32 split: parity (HM tests + C5a configs) and time
python -c "import __graft_entry__ as g; g.build()"
O=gpurun_out/r4z; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -q -m gpu -k "hm or c5a or C5a or fc_fast" > $O/pytest.log 2>&1; tail -1 $O/pytest.log
timeout 300 python scripts/gemm_shape_bench.py --cls bcbaacaacacababcaabcaaaac --M 3 --kernels 1,5 --iters 50 2>&1 | grep kernel
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > $O/bench.json 2> $O/bench.err; python -c "
import json; d=json.load(open('$O/bench.json')); print('C5a', round(d['value'],2), 'e2e', round(d['e2e']['value'],2))"
