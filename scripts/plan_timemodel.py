#!/usr/bin/env python
"""Rank amplitude-plan candidates by a time model of the lowered program instead of predicted bytes
(reading A11: bytes alone mis-rank plans whose fused GEMM groups are FP32-bound).

Per phase-B op (tests/planbuf.py parses the plan buffer):
  t = max(algorithmic bytes / BW, flops / F32) + T_LAUNCH
(k_gemm_hm groups: HM_BW / HM_FL) with flops = 8 x 2^(R + M) for a fused group (one complex multiply-add per output and summed value;
a producer -> consumer pair adds its consumer's), BW / F32 the rates the kernels reach on one B200
(round-2 profiles: ~4.5 TB/s streaming, ~22 TFLOP/s for the SIMT GEMM groups), interpreter runs at
~1 us per step.  A plan's time = prefix + 2^k x per-slice time.

    python scripts/plan_timemodel.py --workload C5a [--k-min 5 --k-max 8] [--top 12]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

BW = 4.5e12
F32 = 22e12
# k_gemm_hm (round 2, second session): two-operand groups with M >= 3 and >= 2^22 outputs on the
# warp-level tensor cores -- C5a's top group 72 us for 335 MB / 2.15 GFLOP (4.6 TB/s, ~30 TFLOP/s)
HM_BW = 4.6e12
HM_FL = 30e12
T_LAUNCH = 4e-6
T_RUN_STEP = 1e-6


def plan_time(plan):
    import planbuf

    P = planbuf.parse(plan.buf)
    steps, ops = P["steps"], P["ops"]
    t_pre = t_sl = 0.0
    i = 0
    while i < len(ops):
        op = ops[i]
        st = [steps[j] for j in range(op.begin, op.end)]
        if op.type in (planbuf.OP_RUN, planbuf.OP_PRUN):
            t = T_RUN_STEP * len(st) + T_LAUNCH
        else:
            R = st[-1].out_rank
            by = 2.0 ** R + sum(2.0 ** st[0].in_[t].rank for t in range(st[0].n_in))
            by += sum(2.0 * (s.n_in - 1) for s in st[1:])
            fl = 8.0 * 2.0 ** (R + len(st)) if op.type in (planbuf.OP_GROUP, planbuf.OP_GROUP_FEED) else 0.0
            if op.type == planbuf.OP_GROUP_FEED and i + 1 < len(ops):
                nx = ops[i + 1]
                s3 = [steps[j] for j in range(nx.begin, nx.end)]
                R3 = s3[-1].out_rank
                by += 2.0 ** R3 + sum(2.0 ** s3[0].in_[t].rank for t in range(s3[0].n_in)) - 2.0 * 2.0 ** R
                fl += 8.0 * 2.0 ** (R3 + len(s3))
                i += 1
            hm = op.type == planbuf.OP_GROUP and len(st) >= 3 and R >= 22
            t = (max(by * 8 / HM_BW, fl / HM_FL) if hm else max(by * 8 / BW, fl / F32)) + T_LAUNCH
        if op.phase == 0:
            t_pre += t
        else:
            t_sl += t
        i += 1
    return t_pre + plan.n_slices * t_sl


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="C5a")
    ap.add_argument("--k-min", type=int, default=5)
    ap.add_argument("--k-max", type=int, default=8)
    ap.add_argument("--seeds", type=int, default=8)
    ap.add_argument("--top", type=int, default=12)
    ap.add_argument("--r", type=int, default=0)
    args = ap.parse_args()
    import bench
    import paper_2012_02430_b200 as T
    from tn_inputs import WORKLOADS, random_regular_graph
    from concurrent.futures import ThreadPoolExecutor

    w = WORKLOADS[args.workload]
    g = random_regular_graph(w.n, 3, 0)
    cap = bench.MAX_WIDTH.get(args.workload, 32)
    orderers = [("min-fill", 0, 0.0, 0), ("min-degree", 0, 0.0, 0)]
    orderers += [("rgreedy-fill", 16, tau, s) for tau in (0.2, 0.3, 0.4) for s in range(args.seeds)]
    orderers += [("rgreedy", 16, tau, s) for tau in (0.3, 0.5) for s in range(args.seeds // 2)]
    jobs = [(k, o) for k in range(args.k_min, args.k_max + 1) for o in orderers]

    def run(job):
        k, (o, q, tau, s) = job
        try:
            pl = T.build_plan(g, w.p, "amplitude", o, n_sliced=k, rg_q=q, rg_tau=tau, rg_seed=s, r=args.r)
        except T.TnError:
            return None
        if pl.width > cap:
            return None
        i = pl.info
        gb = (i["pred_bytes_per_slice"][0] * pl.n_slices + i["pred_bytes_prefix"][0]) / 1e9
        return (plan_time(pl), k, o, q, tau, s, pl.width, gb)

    with ThreadPoolExecutor(max_workers=os.cpu_count() or 4) as ex:
        res = [r for r in ex.map(run, jobs) if r]
    res.sort()
    for t, k, o, q, tau, s, wd, gb in res[:args.top]:
        print(f"model {t * 1e3:7.2f} ms  k={k} {o} q={q} tau={tau} seed={s} r={args.r} width {wd} {gb:.1f} GB")


if __name__ == "__main__":
    main()
