#!/usr/bin/env python
"""Planner reports: the analogues of the paper's planner figures.

  width_vs_n.csv   contraction width after step-dependent slicing of n indices (n = 0..12) for
                   N = 100 / 150 / 200, p = 1, seeds 0-2, orderers greedy min-degree (the paper's,
                   PAPER.md:461), greedy min-fill and rgreedy -- Fig.
                   `different_parvars`, "dependence of contraction width from
                   n".
  width_over_s.json for N = 210 (the paper's circuit) and N = 150, p = 1, seed 0, min-degree: the
                   width of the plan slicing at every candidate step s in [0, peak] for several n
                   -- Fig. `hist_of_cost` ("difference ... goes up to 9,
                   which translates to a 512x cost difference").

Calls only the planner (libtnb200.so host entry points tn_plan_build / tn_slice_scan).

    python scripts/planner_reports.py [--out profiles/r02/planner]
"""
from __future__ import annotations

import argparse
import collections
import csv
import json
import os
import sys
import time
from concurrent.futures import ThreadPoolExecutor

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2012_02430_b200 as T  # noqa: E402
from paper_2012_02430_b200 import _binding as B  # noqa: E402
from tn_inputs import random_regular_graph  # noqa: E402

ORDERERS = [("min-degree", 0, 0.0), ("min-fill", 0, 0.0), ("rgreedy", 8, 0.5)]


def width_row(job):
    n_q, seed, name, q, tau, n = job
    g = random_regular_graph(n_q, 3, seed)
    pl = T.build_plan(g, 1, "amplitude", name, n_sliced=n, rg_q=q, rg_tau=tau, small_log2=30)
    i = pl.info
    return {"N": n_q, "p": 1, "seed": seed, "orderer": name if not q else f"{name}(q={q},tau={tau})", "n": n,
            "width": i["width"], "unsliced_width": i["unsliced_width"], "slice_step": i["slice_step"],
            "pred_cost_log2": None}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r02", "planner"))
    ap.add_argument("--max-n", type=int, default=12)
    args = ap.parse_args()
    os.makedirs(args.out, exist_ok=True)
    t0 = time.perf_counter()
    jobs = [(N, seed, o, q, tau, n) for N in (100, 150, 200) for seed in range(3) for (o, q, tau) in ORDERERS
            for n in range(0, args.max_n + 1)]
    with ThreadPoolExecutor(max_workers=os.cpu_count() or 4) as ex:
        rows = list(ex.map(width_row, jobs))
    with open(os.path.join(args.out, "width_vs_n.csv"), "w", newline="") as f:
        w = csv.DictWriter(f, fieldnames=["N", "p", "seed", "orderer", "n", "width", "unsliced_width", "slice_step"])
        w.writeheader()
        for r in rows:
            w.writerow({k: r[k] for k in w.fieldnames})
    hist = {}
    for N in (210, 150):
        g = random_regular_graph(N, 3, 0)
        for n in (1, 3, 6, 9, 12):
            scan, peak = B.tn_slice_scan(N, g.edges, 1, n, orderer=B.TN_ORDER_MIN_DEGREE)
            ws = [wd for _, wd, _ in scan]
            hist[f"N{N}_n{n}"] = {"N": N, "p": 1, "seed": 0, "orderer": "min-degree", "n": n, "peak": peak,
                                  "candidates": [{"s": s, "width": wd, "cost": c} for s, wd, c in scan],
                                  "width_histogram": dict(sorted(collections.Counter(ws).items())),
                                  "width_min": min(ws), "width_max": max(ws),
                                  "spread": max(ws) - min(ws), "cost_ratio_2^spread": 2 ** (max(ws) - min(ws))}
    with open(os.path.join(args.out, "width_over_s.json"), "w") as f:
        json.dump(hist, f, indent=0)
    # summary table
    lines = ["# Planner reports (scripts/planner_reports.py)", "",
             "Width after step-dependent slicing of n indices, p = 1, mean over seeds 0-2 "
             "(Fig. different_parvars analogue, PAPER.md:497-507):", ""]
    agg = collections.defaultdict(list)
    for r in rows:
        agg[(r["N"], r["orderer"], r["n"])].append(r["width"])
    ords = sorted({r["orderer"] for r in rows})
    for N in (100, 150, 200):
        lines.append(f"N = {N}: n = " + ", ".join(str(n) for n in range(args.max_n + 1)))
        for o in ords:
            vals = [sum(agg[(N, o, n)]) / len(agg[(N, o, n)]) for n in range(args.max_n + 1)]
            lines.append(f"  {o:>24}: " + " ".join(f"{v:5.1f}" for v in vals))
        lines.append("")
    lines.append("Width over the candidate slice steps s (Fig. hist_of_cost analogue, PAPER.md:637-642), min-degree:")
    lines.append("")
    for k, h in hist.items():
        lines.append(f"  {k}: peak step {h['peak']}, widths {h['width_min']}..{h['width_max']} "
                     f"(spread {h['spread']} = {h['cost_ratio_2^spread']}x cost), histogram {h['width_histogram']}")
    lines.append("")
    lines.append(f"generated in {time.perf_counter() - t0:.1f} s")
    open(os.path.join(args.out, "SUMMARY.md"), "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
