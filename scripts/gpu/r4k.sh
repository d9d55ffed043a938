# k_gemm_fc packed consumer + constant-offset skip: parity subset, step profile, bench
python -c "import __graft_entry__ as g; g.build()"
mkdir -p gpurun_out/r4k
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "feed_pairs or fc_fast or group_kernels or slice_lanes or c5a" > gpurun_out/r4k/pytest.log 2>&1; tail -2 gpurun_out/r4k/pytest.log
TNB_ONE_LANE=1 timeout 300 python scripts/step_profile.py --workload C5a > gpurun_out/r4k/steps.txt 2>&1; head -3 gpurun_out/r4k/steps.txt
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/r4k/bench.json 2> gpurun_out/r4k/bench.err; python -c "
import json; d=json.load(open('gpurun_out/r4k/bench.json')); r=d['roofline']; print('C5a', d['value'], 'e2e', d['e2e']['value'], r['kernel'], r['frac'], {k: (round(v['ms_share_of_step'],3), round(v['GBps'])) for k,v in r['families'].items()})"
