# round 2: k_fc_tc with line bits -- shape trace, parity, timing (tc vs simt), ncu of the tc launch
python -c "import __graft_entry__ as g; g.build()"
mkdir -p gpurun_out/r2f
TNB_FC_TC=1 TNB_GEMM_DEBUG=1 timeout 300 python scripts/c5a_one_pass.py C5a 1 2>&1 | grep -a "k_fc_tc" | head -5
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "feed or fc_tc" > gpurun_out/r2f/pytest_fc.log 2>&1
tail -3 gpurun_out/r2f/pytest_fc.log
for v in 1 0; do
TNB_FC_TC=$v timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2f/bench_tc$v.json 2> gpurun_out/r2f/bench_tc$v.err
python -c "
import json; d=json.load(open('gpurun_out/r2f/bench_tc$v.json')); r=d['roofline']; print('TC=$v VALUE', d['value'], r['kernel'], r['avg_launch_ms']); print(json.dumps(r['families']))"
done
TNB_FC_TC=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_fc_tc -c 1 -o gpurun_out/r2f/fctc python scripts/c5a_one_pass.py > gpurun_out/r2f/ncu.log 2>&1
tail -2 gpurun_out/r2f/ncu.log
