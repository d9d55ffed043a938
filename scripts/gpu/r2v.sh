# validation after the k_gemm switch removal: full GPU suite, smoke, bench (with cpu_baseline), host enqueue
python -c "import __graft_entry__ as g; g.build()"
mkdir -p gpurun_out/r2v
timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/r2v/pytest_gpu.log 2>&1; tail -3 gpurun_out/r2v/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2v/smoke.log 2>&1; tail -1 gpurun_out/r2v/smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r2v/bench.json 2> gpurun_out/r2v/bench.err
python -c "
import json; d=json.load(open('gpurun_out/r2v/bench.json')); r=d['roofline']; print('C5a', d['value'], 'e2e', d['e2e']['value'], r['kernel'], r['frac'], r['traffic'], d['gpu_launches'], d.get('cpu_baseline',{}).get('value'))"
for v in 1 0; do TNB_GRAPH=$v timeout 300 python scripts/host_probe.py 2>&1 | tail -1; done
