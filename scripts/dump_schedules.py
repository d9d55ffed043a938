#!/usr/bin/env python
"""Write the product planner's schedules of the BASELINE workloads to tests/golden/schedules.json.

The schedule (prefix / sliced / residual labels of the elimination order) is the one piece of the
product path the oracle may take as DATA (reading A18): it changes the
rounding order of the oracle's sums, never their value.  With the schedules committed, the oracle
golden values (scripts/make_oracle_goldens.py, which imports only oracle/) and the reference arm of
bench.py (which must not load libtnb200.so) both read this file instead of calling the planner.

    python scripts/dump_schedules.py [--only C2,C5a]

Per workload: the bench plan (bench.build_workload_plan: the recorded recipe or the startup
search), its k / width / info, and the schedule.  C2 (unsliced, width 26) also gets an auxiliary
sliced schedule of width <= 22 so that the oracle's complex128 tensors stay small (Eq. 1 is exact).
"""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
import paper_2012_02430_b200 as T  # noqa: E402
from tn_inputs import WORKLOADS  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden", "schedules.json")
NAMES = ["C2", "C4a", "C4b", "C5a", "C5b", "C5r", "C5r6"]


def sched(plan) -> dict:
    pre, sl, res, deg = plan.schedule()
    return {"prefix": list(pre), "sliced": list(sl), "residual": list(res), "degrees": list(deg)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="")
    args = ap.parse_args()
    names = args.only.split(",") if args.only else NAMES
    out = json.load(open(OUT)) if os.path.exists(OUT) else {}
    for name in names:
        w = WORKLOADS[name]
        plan, g, ga, be, meta = bench.build_workload_plan(name)
        info = plan.info
        rec = {"workload": name, "n": w.n, "p": w.p, "graph_seed": 0, "angles_seed": 0,
               "orderer": plan.orderer, "recipe": meta["tried"][0].get("recipe") if meta.get("tried") else None,
               "plan_source": meta.get("source"), "k": info["k"], "width": info["width"],
               "unsliced_width": info["unsliced_width"], "slice_step": info["slice_step"],
               "n_slices": plan.n_slices, **sched(plan)}
        if info["k"] == 0:
            g_ = g
            aux, _ = T.select_sliced_plan(g_, w.p, 22, k_min=2, k_max=8, orderers=(("rgreedy-fill", 8, 0.3, 0),))
            rec["oracle_aux"] = {"k": aux.info["k"], "width": aux.info["width"], **sched(aux),
                                 "note": "auxiliary sliced schedule for the oracle only (Eq. 1, exact)"}
        out[name] = rec
        print(name, "k", info["k"], "width", info["width"], "steps", len(rec["prefix"]) + len(rec["residual"]),
              flush=True)
    with open(OUT, "w") as f:
        json.dump(out, f, indent=0)


if __name__ == "__main__":
    main()
