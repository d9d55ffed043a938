python -c "import __graft_entry__ as g; g.build()"
mkdir -p gpurun_out/r2m
TNB_FC_TC=1 TNB_FT_TRACE=1 TNB_GEMM_DEBUG=1 timeout 300 python scripts/c5a_one_pass.py C5a 2 2>&1 | grep -a "k_fc_tc" | head -3
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "feed or fc_tc or lanes or batched or partition" > gpurun_out/r2m/pytest_fc.log 2>&1
tail -2 gpurun_out/r2m/pytest_fc.log
for v in 1 0; do
TNB_FC_TC=$v timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2m/bench_tc$v.json 2> gpurun_out/r2m/bench_tc$v.err
python -c "
import json; d=json.load(open('gpurun_out/r2m/bench_tc$v.json')); r=d['roofline']; print('TC=$v VALUE', d['value'], 'e2e', d['e2e']['value'], r['kernel'], r['avg_launch_ms']); print(json.dumps(r['families']))"
tail -3 gpurun_out/r2m/bench_tc$v.err
done
TNB_GRAPH=0 timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2m/bench_nograph.json 2> gpurun_out/r2m/bench_nograph.err
python -c "
import json; d=json.load(open('gpurun_out/r2m/bench_nograph.json')); print('NOGRAPH VALUE', d['value'], 'e2e', d['e2e']['value'])"
