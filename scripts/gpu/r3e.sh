# prefix waves (independent phase-A ops on forked streams): parity and prefix time
python -c "import __graft_entry__ as g; g.build()"
mkdir -p gpurun_out/r3e
timeout 2400 python -m pytest tests -q -m gpu -x > gpurun_out/r3e/pytest_gpu.log 2>&1; tail -2 gpurun_out/r3e/pytest_gpu.log
for v in 1 0; do
TNB_PREFIX_WAVES=$v timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r3e/bench_w$v.json 2> gpurun_out/r3e/bench_w$v.err
python -c "
import json; d=json.load(open('gpurun_out/r3e/bench_w$v.json')); print('WAVES=$v', d['value'], 'e2e', d['e2e']['value'], d['multi_gpu']['per_rank'])"
done
for v in 1 0; do
TNB_PREFIX_WAVES=$v TNB_LANES=4 timeout 600 python - <<'PY'
import os, torch, statistics, bench
import paper_2012_02430_b200 as T
plan,g,ga,be,meta=bench.build_workload_plan('C5a')
n=plan.n_slices; part=torch.zeros(2*n,dtype=torch.float64,device='cuda')
def t(b,e,reps=10):
    for _ in range(3): plan.contract_sliced(ga,be,b,e,part)
    torch.cuda.synchronize(); xs=[]
    for _ in range(reps):
        e0,e1=torch.cuda.Event(enable_timing=True),torch.cuda.Event(enable_timing=True)
        e0.record(); plan.contract_sliced(ga,be,b,e,part); e1.record(); torch.cuda.synchronize(); xs.append(e0.elapsed_time(e1))
    return statistics.median(xs)
print('WAVES', os.environ['TNB_PREFIX_WAVES'], 'prefix only %.3f ms, a rank of 8 (4 slices, 4 lanes) %.3f ms' % (t(0,0), t(0,4)))
PY
done
