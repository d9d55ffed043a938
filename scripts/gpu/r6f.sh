# multi-rank functional lines with the final kernels (gloo, ranks sharing one GPU: per-rank
# breakdown and the JSON path, not a scaling number) and the reference arm at N=1
python -c "import __graft_entry__ as g; g.build()"
O=gpurun_out/r6f; mkdir -p $O
for n in 2 8; do
TNB_BENCH_BACKEND=gloo timeout 900 python bench.py --gpus $n --steps 5 --warmup 3 > $O/bench_gloo$n.json 2> $O/bench_gloo$n.err
python -c "
import json; d=json.load(open('$O/bench_gloo$n.json')); print('GLOO$n', d['n_gpus'], round(d['value'],2), [ (r['rank'], r['slices'], round(r['slices_ms'],3)) for r in d['multi_gpu']['per_rank']])"
done
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > $O/ref.json 2> $O/ref.err
python -c "
import json; d=json.load(open('$O/ref.json')); print('REF', d['value'], d['steps'], d['cpu_baseline']['cores'], d['step_seconds'])"
