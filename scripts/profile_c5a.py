"""Profiling driver for ncu: builds the bench plan (C5a), runs slice 0 once (warm-up), then slice 1
once.  `--print-skip STEP` prints how many k_bucket launches precede the launch of plan step
STEP in the second call, for `ncu -k regex:k_bucket -s <skip> -c <n>`.  `--list` prints the
standalone steps with their k_bucket ordinal and algorithmic bytes."""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="C5a")
    ap.add_argument("--print-skip", type=int, default=None)
    ap.add_argument("--list", action="store_true")
    ap.add_argument("--records", default=None, help="write the first call's per-launch records (JSON)")
    args = ap.parse_args()
    plan, g, ga, be, meta = bench.build_workload_plan(args.workload)
    steps = plan.steps()
    # k_bucket / k_group launches: standalone steps and the head of every fused group
    heads = lambda ph: [i for i, s in enumerate(steps) if s["phase"] == ph and (
        s["standalone"] == 1 or (s["standalone"] == 3 and (i == 0 or steps[i - 1]["standalone"] != 3
                                                             or steps[i]["n_in"] > 2)))]
    big_a = heads(0)
    big_b = heads(1)
    if args.list or args.print_skip is not None:
        if args.list:
            for o, i in enumerate(big_b):
                s = steps[i]
                print(o, i, s["out_rank"], s["in_rank"], s["inplace"], "%.2f GB" % (s["bytes_c64"] / 1e9))
        if args.print_skip is not None:
            first_call = len(big_a) + len(big_b)
            print(first_call + len(big_a) + big_b.index(args.print_skip))
        return
    import torch
    import paper_2012_02430_b200 as T

    torch.cuda.set_device(0)
    partials = torch.zeros(2 * plan.n_slices, dtype=torch.float64, device="cuda")
    plan.profile(True)                  # per-launch records of the first call (launch order)
    plan.contract_sliced(ga, be, 0, 1, partials, dtype=T.TN_C64)
    torch.cuda.synchronize()
    recs = plan.profile_records()
    plan.profile(False)
    plan.profile_read()
    plan.contract_sliced(ga, be, 1, 2, partials, dtype=T.TN_C64)
    torch.cuda.synchronize()
    if args.records:
        json.dump(recs, open(args.records, "w"), indent=1)
    print("ok", partials[:4].tolist())


if __name__ == "__main__":
    main()
