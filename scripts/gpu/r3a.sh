# slice lanes 8 / 12 / 16 with graph replay (C5a, C4b)
python -c "import __graft_entry__ as g; g.build()"
for w in C5a C4b; do for L in 8 12 16; do
TNB_LANES=$L timeout 900 python bench.py --workload $w --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r3a_${w}_$L.json 2> gpurun_out/r3a_${w}_$L.err
python -c "
import json; d=json.load(open('gpurun_out/r3a_${w}_$L.json')); print('$w LANES=$L', d['value'], 'e2e', d['e2e']['value'], d['config']['parallelism'])"
done; done
