# k_gemm_fc bulk-copy chunks: parity subset, per-launch time and bench with / without
python -c "import __graft_entry__ as g; g.build()"
O=gpurun_out/r4l; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -q -m gpu -k "feed_pairs or fc_fast or slice_lanes or c5a or C5a or c4b or C4b" > $O/pytest.log 2>&1; tail -2 $O/pytest.log
for v in 1 0; do TNB_FC_BULK=$v TNB_ONE_LANE=1 timeout 300 python scripts/step_profile.py --workload C5a > $O/steps_bulk$v.txt 2>&1; head -1 $O/steps_bulk$v.txt; done
for v in 1 0; do TNB_FC_BULK=$v timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > $O/bench_bulk$v.json 2> $O/bench_bulk$v.err; python -c "
import json; d=json.load(open('$O/bench_bulk$v.json')); r=d['roofline']; print('BULK=$v C5a', d['value'], 'e2e', d['e2e']['value'], r['kernel'], r['frac'])"; done
