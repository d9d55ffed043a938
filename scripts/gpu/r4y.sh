# k_gemm_fc with 16-warp CTAs (TNB_FC_WB=4) against 8-warp (default)
python -c "import __graft_entry__ as g; g.build()"
O=gpurun_out/r4y; mkdir -p $O
TNB_FC_WB=4 timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "feed_pairs or fc_fast" > $O/pytest.log 2>&1; tail -1 $O/pytest.log
for v in 4 3; do TNB_FC_WB=$v TNB_ONE_LANE=1 timeout 300 python scripts/step_profile.py --workload C5a 2>&1 | grep "176-183" | sed "s/^/WB=$v /"; done
for v in 4 3; do TNB_FC_WB=$v timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > $O/bench_wb$v.json 2> $O/bench_wb$v.err; python -c "
import json; d=json.load(open('$O/bench_wb$v.json')); print('WB=$v C5a', round(d['value'],2), 'e2e', round(d['e2e']['value'],2))"; done
