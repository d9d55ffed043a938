"""Offline plan search (reading A11): for a workload, plan every (k, orderer) candidate --
greedy min-fill / min-degree and rgreedy / rgreedy-fill Boltzmann runs
 over a grid of (q, tau, seed) -- and record the candidates with width <= the
config's cap, fewest predicted algorithmic bytes first, in paper_2012_02430_b200/plan_recipes.json.  bench.py
rebuilds the recorded recipe deterministically (seconds) instead of searching at startup.

    python scripts/plan_search.py --workload C5a [--k-min 5 --k-max 8] [--seeds 6]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

RECIPES = os.path.join(ROOT, "paper_2012_02430_b200", "plan_recipes.json")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="C5a")
    ap.add_argument("--k-min", type=int, default=None)
    ap.add_argument("--k-max", type=int, default=None)
    ap.add_argument("--seeds", type=int, default=6)
    ap.add_argument("--q", type=int, default=16)
    ap.add_argument("--r", type=int, default=0, help="indices sliced per round (0: r = n, one round)")
    ap.add_argument("--dry", action="store_true", help="print only, do not update the recipe file")
    args = ap.parse_args()
    import bench
    import paper_2012_02430_b200 as T
    from tn_inputs import WORKLOADS, random_regular_graph
    w = WORKLOADS[args.workload]
    g = random_regular_graph(w.n, 3, 0)
    kmin, kmax = bench.K_RANGE.get(args.workload, (0, 12))
    kmin = args.k_min if args.k_min is not None else kmin
    kmax = args.k_max if args.k_max is not None else kmax
    orderers = list(T.DEFAULT_ORDERERS)
    orderers += [("rgreedy-fill", args.q, tau, s) for tau in (0.2, 0.3, 0.4) for s in range(args.seeds)]
    orderers += [("rgreedy", args.q, tau, s) for tau in (0.3, 0.5) for s in range(min(3, args.seeds))]
    t0 = time.time()
    _, tried = T.select_sliced_plan(g, w.p, bench.MAX_WIDTH.get(args.workload, 32), k_min=kmin, k_max=kmax,
                                    orderers=orderers, r=args.r)
    for t in tried:
        t["recipe"]["r"] = args.r
    ok = sorted([t for t in tried if t["width"] <= bench.MAX_WIDTH.get(args.workload, 32)],
                key=lambda t: (t["pred_bytes_c64"], t["k"]))
    for t in ok[:10]:
        print(t)
    if args.dry:
        return
    try:
        cur = json.load(open(RECIPES))
    except Exception:
        cur = {}
    cur[args.workload] = {"seed_graph": 0, "k_range": [kmin, kmax], "search_s": time.time() - t0,
                          "candidates": len(tried), "best": ok[:8]}
    json.dump(cur, open(RECIPES, "w"), indent=1)
    print("wrote", RECIPES, "search s %.0f" % (time.time() - t0))


if __name__ == "__main__":
    main()
