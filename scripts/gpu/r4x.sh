# k_gemm_fc with C3_y folded into B' (TNB_FC_C3B=1): parity and time
python -c "import __graft_entry__ as g; g.build()"
O=gpurun_out/r4x; mkdir -p $O
TNB_FC_C3B=1 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -q -m gpu -k "feed_pairs or fc_fast or c5a or C5a" > $O/pytest.log 2>&1; tail -1 $O/pytest.log
for v in 1 0; do TNB_FC_C3B=$v TNB_ONE_LANE=1 timeout 300 python scripts/step_profile.py --workload C5a 2>&1 | grep "176-183" | sed "s/^/C3B=$v /"; done
for v in 1 0; do TNB_FC_C3B=$v timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > $O/bench_c3b$v.json 2> $O/bench_c3b$v.err; python -c "
import json; d=json.load(open('$O/bench_c3b$v.json')); print('C3B=$v C5a', round(d['value'],2), 'e2e', round(d['e2e']['value'],2))"; done
