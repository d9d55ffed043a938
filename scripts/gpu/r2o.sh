# full GPU suite, smoke, bench (default), the paper-replica workloads, 8-rank functional line
python -c "import __graft_entry__ as g; g.build()"
mkdir -p gpurun_out/r2o
timeout 2400 python -m pytest tests -q -m gpu --durations=25 > gpurun_out/r2o/pytest_gpu.log 2>&1
tail -30 gpurun_out/r2o/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2o/smoke.log 2>&1; tail -2 gpurun_out/r2o/smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r2o/bench_c5a.json 2> gpurun_out/r2o/bench_c5a.err
python -c "
import json; d=json.load(open('gpurun_out/r2o/bench_c5a.json')); r=d['roofline']; print('C5a', d['value'], 'e2e', d['e2e']['value'], r['kernel'], r['frac'], d.get('cpu_baseline',{}).get('value'), d['gpu_launches'])"
for w in C5r C5r6 C4b C2; do
timeout 900 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2o/bench_$w.json 2> gpurun_out/r2o/bench_$w.err
python -c "
import json; d=json.load(open('gpurun_out/r2o/bench_$w.json')); r=d['roofline']; print('$w', d['value'], 'ms', d['ms_per_step'], r['kernel'], r['frac'], json.dumps(r['families']))"
done
TNB_BENCH_BACKEND=gloo timeout 900 python bench.py --gpus 8 --steps 5 --warmup 3 > gpurun_out/r2o/bench_gloo8.json 2> gpurun_out/r2o/bench_gloo8.err
tail -c 1200 gpurun_out/r2o/bench_gloo8.json; grep -i error gpurun_out/r2o/bench_gloo8.err | head -3
