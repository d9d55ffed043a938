# k_fc_hm: fused-pair parity, C5a step profile and bench
python -c "import __graft_entry__ as g; g.build()"
mkdir -p gpurun_out/r4h
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "feed_pairs or fc_fast or hm or slice_lanes_with_fused" > gpurun_out/r4h/pytest.log 2>&1; tail -5 gpurun_out/r4h/pytest.log
TNB_ONE_LANE=1 timeout 300 python scripts/step_profile.py --workload C5a > gpurun_out/r4h/steps.txt 2>&1; head -6 gpurun_out/r4h/steps.txt
TNB_GEMM_DEBUG=1 TNB_ONE_LANE=1 TNB_GRAPH=0 timeout 300 python scripts/c5a_one_pass.py C5a 1 2>&1 | grep "k_gemm_hm R\|k_fc_hm" > gpurun_out/r4h/shapes.txt; cat gpurun_out/r4h/shapes.txt
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/r4h/bench.json 2> gpurun_out/r4h/bench.err; python -c "
import json; d=json.load(open('gpurun_out/r4h/bench.json')); r=d['roofline']; print('C5a', d['value'], 'e2e', d['e2e']['value'], r['kernel'], r['frac'], {k: (round(v['ms_share_of_step'],3), round(v['GBps'])) for k,v in r['families'].items()})"
