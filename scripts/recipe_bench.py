#!/usr/bin/env python
"""Time a plan recipe of a workload on one GPU the way bench.py's timed region does (all slices,
default workspace with its slice lanes, CUDA-graph replay), for plan comparisons (reading A11:
predicted bytes do not always predict time).

    python scripts/recipe_bench.py --workload C5a --orderer rgreedy-fill --k 6 --q 16 --tau 0.3 --seed 2 --r 4
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="C5a")
    ap.add_argument("--orderer", default="min-fill")
    ap.add_argument("--k", type=int, default=0)
    ap.add_argument("--q", type=int, default=0)
    ap.add_argument("--tau", type=float, default=0.0)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--r", type=int, default=0)
    ap.add_argument("--steps", type=int, default=20)
    args = ap.parse_args()
    import torch

    import paper_2012_02430_b200 as T
    from tn_inputs import WORKLOADS, qaoa_angles, random_regular_graph

    w = WORKLOADS[args.workload]
    g = random_regular_graph(w.n, 3, 0)
    plan = T.build_plan(g, w.p, "amplitude", args.orderer, n_sliced=args.k, rg_q=args.q, rg_tau=args.tau,
                        rg_seed=args.seed, r=args.r)
    n = plan.n_slices
    part = torch.zeros(2 * n, dtype=torch.float64, device="cuda")
    params = [qaoa_angles(w.p, 1000 + s) for s in range(5 + args.steps)]
    for s in range(5):
        plan.contract_sliced(*params[s], 0, n, part)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for s in range(args.steps):
        plan.contract_sliced(*params[5 + s], 0, n, part)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.steps
    i = plan.info
    gb = (i["pred_bytes_per_slice"][0] * n + i["pred_bytes_prefix"][0]) / 1e9
    print(f"{args.workload} {args.orderer} k={args.k} q={args.q} tau={args.tau} seed={args.seed} r={args.r}: "
          f"width {plan.width}, {gb:.1f} GB, {ms:.2f} ms, {1000 / ms:.1f} /s, launches/slice {i['launches_per_slice']}")


if __name__ == "__main__":
    main()
