"""Time candidate plans (recipes) of a workload on the GPU: one whole contraction per repetition
(all slices, default slice lanes), CUDA events.  Used to pick the bench plan recipe.
    python scripts/plan_bench.py --workload C5a --recipes "k,orderer,q,tau,seed;..." """
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="C5a")
    ap.add_argument("--recipes", required=True)
    ap.add_argument("--reps", type=int, default=5)
    args = ap.parse_args()
    import torch
    import paper_2012_02430_b200 as T
    from tn_inputs import WORKLOADS, qaoa_angles, random_regular_graph
    w = WORKLOADS[args.workload]
    g = random_regular_graph(w.n, 3, 0)
    ga, be = qaoa_angles(w.p, 1)
    for rec in args.recipes.split(";"):
        k, o, q, tau, seed = rec.split(",")
        t0 = time.time()
        plan = T.build_plan(g, w.p, "amplitude", o, n_sliced=int(k), rg_q=int(q), rg_tau=float(tau),
                            rg_seed=int(seed))
        ps = time.time() - t0
        part = torch.zeros(2 * plan.n_slices, dtype=torch.float64, device="cuda")
        for _ in range(2):
            plan.contract_sliced(ga, be, 0, plan.n_slices, part)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.reps):
            plan.contract_sliced(ga, be, 0, plan.n_slices, part)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / args.reps
        gb = (plan.info["pred_bytes_per_slice"][0] * plan.n_slices + plan.info["pred_bytes_prefix"][0]) / 1e9
        print(f"{rec:40s} width {plan.width} slices {plan.n_slices} pred {gb:7.1f} GB  {ms:7.2f} ms  "
              f"{gb / ms:5.2f} TB/s  plan {ps:.1f} s ws {plan.workspace_bytes(0) / 1e9:.1f} GB", flush=True)
        plan.release_workspaces()
        del plan
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
