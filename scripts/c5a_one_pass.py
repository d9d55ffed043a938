#!/usr/bin/env python
"""One lane, two slices of the C5a bench plan through tn_contract_sliced (a short run for ncu)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2012_02430_b200 as T  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C5a"
nsl = int(sys.argv[2]) if len(sys.argv) > 2 else 2
plan, g, ga, be, meta = bench.build_workload_plan(name)
p = torch.zeros(2 * plan.n_slices, dtype=torch.float64, device="cuda")
ws = plan.workspace(T.TN_C64, batch=1)
T._binding.tn_contract_sliced(plan.handle, T.TN_C64, ga, be, 0, nsl, ws.data_ptr(), ws.numel(),
                              torch.cuda.current_stream().cuda_stream, p.data_ptr())
torch.cuda.synchronize()
print(p[:4].tolist())
