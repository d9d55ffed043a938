python -c "import __graft_entry__ as g; g.build()"
mkdir -p gpurun_out/r2j
TNB_FC_TC=1 TNB_FT_TRACE=1 timeout 300 python scripts/c5a_one_pass.py C5a 2 2>&1 | grep -a "k_fc_tc" | head -3
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "feed or fc_tc" > gpurun_out/r2j/pytest_fc.log 2>&1
tail -2 gpurun_out/r2j/pytest_fc.log
TNB_FC_TC=1 timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2j/bench_tc1.json 2> gpurun_out/r2j/bench_tc1.err
python -c "
import json; d=json.load(open('gpurun_out/r2j/bench_tc1.json')); r=d['roofline']; print('TC=1 VALUE', d['value'], r['kernel'], r['avg_launch_ms']); print(json.dumps(r['families']))"
