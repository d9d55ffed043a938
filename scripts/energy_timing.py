#!/usr/bin/env python
"""Energy (§8 a12) timing: one tn_energy call and a 256-set tn_energy_batch for C1 and C3, both dtypes,
CUDA events after warm-up; the value is checked against the oracle.

    python scripts/energy_timing.py
"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    import paper_2012_02430_b200 as T
    from oracle import energy
    from tn_inputs import WORKLOADS, qaoa_angles, random_regular_graph

    for name in ("C1", "C3"):
        w = WORKLOADS[name]
        g = random_regular_graph(w.n, 3, 0)
        ga, be = qaoa_angles(w.p, 0)
        plan = T.build_plan(g, w.p, "energy", "min-fill")
        Eref, _ = energy.maxcut_energy(w.n, g.edges, ga, be)
        for dt, dn in ((T.TN_C64, "c64"), (T.TN_C128, "c128")):
            zz, im, E = plan.energy(ga, be, dtype=dt)
            ts = []
            for _ in range(20):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                plan.energy(ga, be, dtype=dt)
                e1.record()
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1))
            sets = [qaoa_angles(w.p, 1000 + b) for b in range(256)]
            plan.energy_batch([s[0] for s in sets], [s[1] for s in sets], dtype=dt)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            plan.energy_batch([s[0] for s in sets], [s[1] for s in sets], dtype=dt)
            e1.record()
            torch.cuda.synchronize()
            tb = e0.elapsed_time(e1)
            print(f"{name} {dn}: |E - E_oracle| {abs(E - Eref):.2e}, {statistics.median(ts) * 1e3:.0f} us per call, "
                  f"batch of 256: {tb * 1e3 / 256:.1f} us per energy")


if __name__ == "__main__":
    main()
