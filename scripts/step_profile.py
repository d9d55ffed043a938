"""Per-step device time and algorithmic GB/s of one slice (CUDA events around every standalone
launch) -- the data behind PAPER.md Fig. contract_cost, measured.  Usage:
    python scripts/step_profile.py [--workload C5a] [--dtype c64] [--out file.json]"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="C5a")
    ap.add_argument("--dtype", default="c64")
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    import torch
    import paper_2012_02430_b200 as T
    dt = T.TN_C64 if args.dtype == "c64" else T.TN_C128
    plan, g, ga, be, meta = bench.build_workload_plan(args.workload)
    steps = plan.steps()
    part = torch.zeros(2 * plan.n_slices, dtype=torch.float64, device="cuda")
    plan.contract_sliced(ga, be, 0, 1, part, dtype=dt)      # warm-up
    torch.cuda.synchronize()
    plan.profile_read()
    plan.profile(True)
    plan.contract_sliced(ga, be, 1, 2, part, dtype=dt)
    torch.cuda.synchronize()
    recs = plan.profile_records()
    plan.profile(False)
    plan.profile_read()
    tot_ms = sum(r["ms"] for r in recs)
    rows = []
    for r in sorted(recs, key=lambda r: -r["ms"]):
        s = steps[r["step_begin"]]
        rows.append({**r, "n_in": s["n_in"], "in_rank": s["in_rank"], "GBps": r["bytes"] / r["ms"] / 1e6,
                     "share": r["ms"] / tot_ms})
    for x in rows[:20]:
        print("%-13s %-5s steps %3d-%3d out %2d in %-16s %7.3f ms %6.0f GB/s share %.3f" % (
            x["kernel"], x["kind"], x["step_begin"], x["step_end"] - 1, x["out_rank"], x["in_rank"], x["ms"], x["GBps"], x["share"]))
    print("total standalone ms per slice: %.2f, GB: %.1f" % (tot_ms, sum(r["bytes"] for r in recs) / 1e9))
    if args.out:
        json.dump({"workload": args.workload, "dtype": args.dtype, "records": rows}, open(args.out, "w"), indent=1)


if __name__ == "__main__":
    main()
