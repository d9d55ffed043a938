"""Strong-scaling estimate on ONE GPU: the block of slices rank 0 of a G-GPU run would own
([0, 2^k / G), lanes sized from the block as scheduler.run_sliced does), timed alone with CUDA
events, for G = 1, 2, 4, 8.  T(G) excludes the all-reduce of the 2 * 2^k partial doubles (one
NCCL call on 512 bytes for C5a); every rank repeats the prefix, which is inside each T(G).
E(G) = T(1) / (G T(G)).  Not a multi-GPU measurement: the driver's SCALE run is that.

    python scripts/scaling_estimate.py [workload]
"""
import json
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402


def main():
    wl = sys.argv[1] if len(sys.argv) > 1 else "C5a"
    plan, g, ga, be, meta = bench.build_workload_plan(wl)
    n = plan.n_slices
    part = torch.zeros(2 * n, dtype=torch.float64, device="cuda")

    def t(b, e, reps=20):
        for _ in range(5):
            plan.contract_sliced(ga, be, b, e, part)
        torch.cuda.synchronize()
        xs = []
        for _ in range(reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            plan.contract_sliced(ga, be, b, e, part)
            e1.record()
            torch.cuda.synchronize()
            xs.append(e0.elapsed_time(e1))
        return statistics.median(xs)

    out = {"workload": wl, "n_slices": n, "prefix_ms": t(0, 0), "ranks": []}
    t1 = None
    for G in (1, 2, 4, 8):
        if n % G:
            continue
        ms = t(0, n // G)
        t1 = ms if t1 is None else t1
        out["ranks"].append({"G": G, "slices_per_rank": n // G, "rank0_block_ms": ms,
                             "efficiency_estimate": t1 / (G * ms)})
    print(json.dumps(out))


if __name__ == "__main__":
    main()
