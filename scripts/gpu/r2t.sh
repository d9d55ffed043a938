# C5a recipe candidates (k = 5, 8, 7) on one GPU, default build
python -c "import __graft_entry__ as g; g.build()"
mkdir -p gpurun_out/r2t
for ix in 0 1 3; do
TNB_RECIPE_INDEX=$ix timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2t/bench_ix$ix.json 2> gpurun_out/r2t/bench_ix$ix.err
python -c "
import json; d=json.load(open('gpurun_out/r2t/bench_ix$ix.json')); print('IX=$ix', d['config']['plan']['k'], d['config']['plan']['width'], 'VALUE', d['value'], 'e2e', d['e2e']['value'], d['roofline']['kernel'], d['roofline']['frac'])"
done
for L in 4 2; do
TNB_LANES=$L timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2t/bench_lanes$L.json 2> gpurun_out/r2t/bench_lanes$L.err
python -c "
import json; d=json.load(open('gpurun_out/r2t/bench_lanes$L.json')); print('LANES=$L VALUE', d['value'])"
done
TNB_BENCH_BACKEND=gloo timeout 900 python bench.py --gpus 8 --steps 5 --warmup 3 > gpurun_out/r2t/bench_gloo8.json 2> gpurun_out/r2t/bench_gloo8.err
python -c "
import json; d=json.load(open('gpurun_out/r2t/bench_gloo8.json')); print('GLOO8', d['n_gpus'], d['value'], json.dumps(d['multi_gpu'])[:600])"
