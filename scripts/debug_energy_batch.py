import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2012_02430_b200 as T
from oracle import energy
from tn_inputs import qaoa_angles, random_regular_graph
g = random_regular_graph(30, 3, 3)
plan = T.build_plan(g, 2, "energy", "min-fill")
sets = [qaoa_angles(2, 100 + b) for b in range(3)]
zzs, ims, ens = plan.energy_batch([s[0] for s in sets], [s[1] for s in sets], dtype=T.TN_C128)
for b, (ga, be) in enumerate(sets):
    zz1, im1, e1 = plan.energy(ga, be, dtype=T.TN_C128)
    Eref, zref = energy.maxcut_energy(30, g.edges, ga, be)
    print(b, "batch", ens[b], zzs[b][:3], "single", e1, zz1[:3], "oracle", Eref, [z.real for z in zref[:3]])
