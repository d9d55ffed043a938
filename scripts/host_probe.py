import sys, time
sys.path.insert(0, '.')
import torch, bench
import paper_2012_02430_b200 as T
plan, g, ga, be, meta = bench.build_workload_plan("C5a")
n = plan.n_slices
part = torch.zeros(2 * n, dtype=torch.float64, device="cuda")
for _ in range(3):
    plan.contract_sliced(ga, be, 0, n, part)
torch.cuda.synchronize()
# host enqueue time per contraction (GPU runs behind)
t0 = time.perf_counter()
for _ in range(20):
    plan.contract_sliced(ga, be, 0, n, part)
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
print("host enqueue ms per contraction %.2f, wall incl. drain %.2f" % ((t1 - t0) / 20 * 1e3, (t2 - t0) / 20 * 1e3))
