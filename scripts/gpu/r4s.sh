# slice lanes with the final kernels: 12 / 16 / 24 / 32
python -c "import __graft_entry__ as g; g.build()"
O=gpurun_out/r4s; mkdir -p $O
for L in 16 24 32 12; do TNB_LANES=$L timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > $O/bench_l$L.json 2> $O/bench_l$L.err; python -c "
import json; d=json.load(open('$O/bench_l$L.json')); print('LANES=$L C5a', round(d['value'],2), 'e2e', round(d['e2e']['value'],2))"; done
