# end-of-round sanity: the reference arm as the driver launches it, and the default bench line once more
O=gpurun_out/r7i; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 900 python bench.py --impl reference --gpus 1 --steps 2 --warmup 1 > $O/bench_reference.json 2> $O/bench_reference.err; tail -c 700 $O/bench_reference.json
timeout 600 python bench.py --gpus 1 > $O/bench_default.json 2> $O/bench_default.err; python -c "
import json; d=json.load(open('$O/bench_default.json')); print('default', d['value'], d['e2e']['value'], d['steps'], d['warmup'], d['cpu_baseline']['value'])"
