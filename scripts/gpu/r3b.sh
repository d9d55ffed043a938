# slice lanes 16 / 24 / 32 (C5a, C4b), C5r at 16
python -c "import __graft_entry__ as g; g.build()"
for w in C5a C4b; do for L in 16 24 32; do
TNB_LANES=$L timeout 900 python bench.py --workload $w --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r3b_${w}_$L.json 2> gpurun_out/r3b_${w}_$L.err
python -c "
import json; d=json.load(open('gpurun_out/r3b_${w}_$L.json')); print('$w LANES=$L', d['value'], 'e2e', d['e2e']['value'], d['config']['parallelism'], d['config']['plan']['workspace_GB'])"
done; done
for L in 8 16; do
TNB_LANES=$L timeout 900 python bench.py --workload C5r --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r3b_C5r_$L.json 2> gpurun_out/r3b_C5r_$L.err
python -c "
import json; d=json.load(open('gpurun_out/r3b_C5r_$L.json')); print('C5r LANES=$L', d['value'], d['config']['parallelism'])"
done
