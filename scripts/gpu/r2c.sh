# round 2: first k_fc_tc run -- shape trace, FEED-pair parity (tc and simt), config parity, bench
python -c "import __graft_entry__ as g; g.build()"
mkdir -p gpurun_out/r2c
TNB_GEMM_DEBUG=1 timeout 300 python -c "
import bench, torch, paper_2012_02430_b200 as T
plan,g,ga,be,meta=bench.build_workload_plan('C5a')
p=torch.zeros(2*plan.n_slices,dtype=torch.float64,device='cuda')
plan.contract_sliced(ga,be,0,1,p); torch.cuda.synchronize(); print(p[:2].tolist())
" > gpurun_out/r2c/debug.log 2>&1
grep -a "k_fc_tc\|Error\|error" gpurun_out/r2c/debug.log | head -20
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "feed or fc_tc or c5a or lanes" > gpurun_out/r2c/pytest_fc.log 2>&1
tail -15 gpurun_out/r2c/pytest_fc.log
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2c/bench.json 2> gpurun_out/r2c/bench.err
python -c "
import json; d=json.load(open('gpurun_out/r2c/bench.json')); print('VALUE', d['value'], 'e2e', d['e2e']['value']); print(json.dumps(d['roofline']['families']))"
TNB_NO_FC_TC=1 timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2c/bench_simt.json 2> gpurun_out/r2c/bench_simt.err
python -c "
import json; d=json.load(open('gpurun_out/r2c/bench_simt.json')); print('SIMT VALUE', d['value'])"
timeout 1500 python -m pytest tests/test_gpu_configs.py -q -m gpu > gpurun_out/r2c/pytest_configs.log 2>&1
tail -15 gpurun_out/r2c/pytest_configs.log
