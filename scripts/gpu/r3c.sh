# final validation of the default path: full GPU suite, smoke, bench (cpu_baseline), the reference arm
python -c "import __graft_entry__ as g; g.build()"
mkdir -p gpurun_out/r3c
timeout 2400 python -m pytest tests -q -m gpu --durations=10 > gpurun_out/r3c/pytest_gpu.log 2>&1; tail -14 gpurun_out/r3c/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r3c/smoke.log 2>&1; tail -1 gpurun_out/r3c/smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r3c/bench.json 2> gpurun_out/r3c/bench.err
python -c "
import json; d=json.load(open('gpurun_out/r3c/bench.json')); r=d['roofline']; print('C5a', d['value'], 'e2e', d['e2e']['value'], r['kernel'], r['frac'], d['gpu_launches'], d['clocks'], d.get('cpu_baseline',{}).get('value'), d['multi_gpu']['per_rank'])"
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r3c/ref.json 2> gpurun_out/r3c/ref.err; cut -c1-400 gpurun_out/r3c/ref.json
