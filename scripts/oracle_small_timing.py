#!/usr/bin/env python
"""One-core and all-core times of the oracle on the small BASELINE configs (SURVEY.md §8(d)
"Oracle timing": also report 1-core time for C1-C3).  The oracle as it stands (complex128 numpy);
C2 / C4a on their committed schedules (tests/golden/schedules.json).

    python scripts/oracle_small_timing.py [--out profiles/r02/oracle_timing.json]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    import bench
    from oracle import energy
    from tn_inputs import WORKLOADS, qaoa_angles, random_regular_graph

    hi = bench.host_info()
    res = {"host": hi, "rows": []}
    for name in ("C1", "C3"):
        w = WORKLOADS[name]
        g = random_regular_graph(w.n, 3, 0)
        ga, be = qaoa_angles(w.p, 0)
        t0 = time.perf_counter()
        E, _ = energy.maxcut_energy(w.n, g.edges, ga, be)
        res["rows"].append({"config": name, "what": f"energy ({len(g.edges)} light cones)", "cores": 1,
                            "seconds": time.perf_counter() - t0, "value": E})
    for name in ("C2", "C4a"):
        w = WORKLOADS[name]
        ga, be = qaoa_angles(w.p, 0)
        for workers in (1, hi["usable_cores"]):
            sig, t, ns, sub = bench.oracle_contraction(name, ga, be, workers=workers)
            res["rows"].append({"config": name, "what": f"sigma ({ns} slices x {sub} sub-slices)", "cores": workers,
                                "seconds": t, "value": [sig.real, sig.imag]})
    for r in res["rows"]:
        print(json.dumps(r))
    if args.out:
        json.dump(res, open(args.out, "w"), indent=1)


if __name__ == "__main__":
    main()
