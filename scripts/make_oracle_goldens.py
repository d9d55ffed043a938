#!/usr/bin/env python
"""Oracle golden values for the BASELINE workloads -> tests/golden/oracle_configs.json.

Imports ONLY oracle/ and tn_inputs (no product code): the schedules are read as data from
tests/golden/schedules.json (written by scripts/dump_schedules.py).
Every value is complex128 bucket elimination (oracle/contract.py), sub-sliced (Eq. 1, exact) where
a slice is wider than the host RAM allows, summed in the fixed pairwise tree.  Angles: the seeded
generic draw qaoa_angles(p, 0) of the workload.

    python scripts/make_oracle_goldens.py [--only C2,C4a] [--workers N]

Values (the -m gpu tests compare the CUDA path with them, tests/test_gpu_configs.py):
  C2   whole sigma (the auxiliary sliced schedule; sigma does not depend on the schedule)
  C4a  whole sigma (all 256 slices) and slices 0, 128, 255 of the bench schedule
  C4b  whole sigma (all 256 slices) and slices 0, 128, 255
  C5a  whole sigma (all 32 slices) and slices 0, 16, 31; C5r / C5r6 (same instance) share sigma
  C5b  slice 0 (2^14 slices: the whole sigma is out of reach of the oracle)
"""
from __future__ import annotations

import argparse
import json
import os
import platform
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import contract, network  # noqa: E402
from tn_inputs import qaoa_angles, random_regular_graph  # noqa: E402

SCHED = os.path.join(ROOT, "tests", "golden", "schedules.json")
OUT = os.path.join(ROOT, "tests", "golden", "oracle_configs.json")

# (whole sigma?, sampled slices, sub-slice width cap)
JOBS = {
    "C2": (True, [], 22),
    "C4a": (True, [0, 128, 255], 22),
    "C4b": (True, [0, 128, 255], 23),
    "C5a": (True, [0, 16, 31], 23),
    "C5b": (False, [0], 24),
}


def cpx(z: complex):
    return [z.real, z.imag]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="")
    ap.add_argument("--workers", type=int, default=os.cpu_count() or 1)
    args = ap.parse_args()
    names = args.only.split(",") if args.only else list(JOBS)
    sch = json.load(open(SCHED))
    out = json.load(open(OUT)) if os.path.exists(OUT) else {}
    for name in names:
        whole, js, mw = JOBS[name]
        s = sch[name]
        g = random_regular_graph(s["n"], 3, s["graph_seed"])
        ga, be = qaoa_angles(s["p"], s["angles_seed"])
        tens = network.qaoa_amplitude_network(s["n"], g.edges, ga, be)
        rec = {"n": s["n"], "p": s["p"], "graph_seed": s["graph_seed"], "angles_seed": s["angles_seed"],
               "gammas": ga, "betas": be, "dtype": "complex128 (numpy, oracle/contract.py)"}
        t0 = time.perf_counter()
        if name == "C2":
            a = s["oracle_aux"]
            vals, extra = contract.slice_values(tens, a["prefix"], a["sliced"], a["residual"],
                                                range(1 << len(a["sliced"])), max_width=mw, workers=args.workers)
            rec["sigma"] = cpx(contract.pairwise_sum(vals))
            rec["sigma_schedule"] = "oracle_aux (schedules.json)"
            rec["subslice_labels"] = extra
        else:
            ids = list(range(1 << len(s["sliced"]))) if whole else sorted(set(js))
            vals, extra = contract.slice_values(tens, s["prefix"], s["sliced"], s["residual"], ids,
                                                max_width=mw, workers=args.workers)
            by = dict(zip(ids, vals))
            if whole:
                rec["sigma"] = cpx(contract.pairwise_sum(vals))
            rec["slices"] = {str(j): cpx(by[j]) for j in js}
            rec["schedule"] = f"{name} bench schedule (schedules.json: k={s['k']}, width {s['width']})"
            rec["schedule_sliced"] = s["sliced"]
            rec["schedule_prefix_len"] = len(s["prefix"])
            rec["subslice_labels"] = extra
        rec["oracle_seconds"] = time.perf_counter() - t0
        rec["workers"] = args.workers
        rec["host"] = platform.processor() or platform.machine()
        out[name] = rec
        print(name, json.dumps({k: rec[k] for k in rec if k in ("sigma", "slices", "oracle_seconds")}), flush=True)
        with open(OUT, "w") as f:
            json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
