# k_fc_tc with 2 X-loader warps: trace (cp / tma X loads), parity, bench
python -c "import __graft_entry__ as g; g.build()"
mkdir -p gpurun_out/r2z
for xl in cp tma; do
TNB_FC_XLOAD=$xl TNB_FC_TC=1 TNB_FT_TRACE=1 timeout 300 python scripts/c5a_one_pass.py C5a 2 2>&1 | grep -a "k_fc_tc trace" | head -1
done
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "feed or fc_tc" > gpurun_out/r2z/pytest_fc.log 2>&1; tail -1 gpurun_out/r2z/pytest_fc.log
TNB_FC_XLOAD=cp timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "fc_tc" > gpurun_out/r2z/pytest_fc2.log 2>&1; tail -1 gpurun_out/r2z/pytest_fc2.log
for xl in cp tma; do
TNB_FC_XLOAD=$xl TNB_FC_TC=1 timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2z/bench_$xl.json 2> gpurun_out/r2z/bench_$xl.err
python -c "
import json; d=json.load(open('gpurun_out/r2z/bench_$xl.json')); r=d['roofline']; print('XLOAD=$xl VALUE', d['value'], json.dumps({k:(round(x['ms_share_of_step'],3), round(x['GBps'])) for k,x in r['families'].items()}))"
done
