"""B200-native sliced bucket-elimination contractor for QAOA MaxCut tensor networks
(arXiv:2012.02430, "Tensor Network Quantum Simulator With Step-Dependent Parallelization").

Layers:
  include/tn_b200.h + csrc/     the C-ABI library libtnb200.so (planner, executor, sm_100a kernels)
  _binding.py                   ctypes marshalling, C names
  this module                   Plan (handle + workspace), plan selection (reading A11)
  scheduler.py                  slice partition over torch.distributed ranks + one all-reduce

PyTorch supplies device memory, streams and process groups only.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Dict, List, Optional, Sequence, Tuple

from . import _binding as B
from ._binding import (TN_C64, TN_C128, TN_KIND_AMPLITUDE, TN_KIND_ENERGY, TN_ORDER_MIN_DEGREE,
                       TN_ORDER_MIN_FILL, TnError)

__all__ = ["Plan", "TN_C64", "TN_C128", "TN_KIND_AMPLITUDE", "TN_KIND_ENERGY", "TN_ORDER_MIN_FILL",
           "TN_ORDER_MIN_DEGREE", "TnError", "build_plan", "select_sliced_plan"]

ORDERERS = {"min-fill": TN_ORDER_MIN_FILL, "min-degree": TN_ORDER_MIN_DEGREE, "rgreedy": B.TN_ORDER_RGREEDY,
            "rgreedy-fill": B.TN_ORDER_RGREEDY_FILL}


class Plan:
    """A loaded plan (tn_plan_load) plus cached device workspaces (torch.empty)."""

    def __init__(self, buf: bytes):
        self.buf = buf
        self.handle = B.tn_plan_load(buf)
        self.info = B.tn_plan_info(self.handle)
        self._ws: Dict[Tuple[int, str], object] = {}

    def __del__(self):
        h = getattr(self, "handle", None)
        if h and B is not None and getattr(B, "_lib", None) is not None:
            B.tn_plan_free(h)
            self.handle = None

    # ------------------------------------------------------------ properties
    @property
    def n_slices(self) -> int:
        return int(self.info["n_slices"])

    @property
    def width(self) -> int:
        return int(self.info["width"])

    @property
    def batch(self) -> int:
        """2^a amplitudes per result (a = open output indices; 1 for a single amplitude)."""
        return 1 << int(self.info["n_open"])

    def schedule(self):
        """(prefix, sliced, residual, degrees) label lists (tn_plan_schedule)."""
        return B.tn_plan_schedule(self.handle)

    def steps(self):
        """Per-step records (tn_plan_steps): the Fig. contract_cost profile of the plan."""
        return B.tn_plan_steps(self.handle)

    def workspace_bytes(self, dtype: int) -> int:
        return int(self.info["workspace_bytes"][dtype])

    # slice batching: windows for up to this many bytes of per-slice tensors
    BATCH_WINDOW_BYTES = 4 << 30

    # slice lanes (independent slices overlap on TNB_LANES streams, default 16) while the extra
    # windows of per-slice tensors cost at most this many bytes in total
    LANE_WINDOW_BYTES = 48 << 30

    def batch_windows(self, dtype: int, n_run: int = 0) -> int:
        """Windows of per-slice tensors in the default workspace for a call that runs n_run slices
        (0: all 2^k; a rank runs only its block, so its lanes are sized from the block): slices run
        per launch when every per-slice step is an interpreter step (slice batching); otherwise
        one window per concurrent slice lane (TNB_LANES, default 16) within LANE_WINDOW_BYTES."""
        n_run = self.n_slices if n_run <= 0 else min(n_run, self.n_slices)
        if n_run <= 1:
            return 1
        one = B.tn_workspace_bytes(self.handle, dtype, 2) - B.tn_workspace_bytes(self.handle, dtype, 1)
        if not self.info["slices_batchable"]:
            import os
            lanes = max(1, min(32, int(os.environ.get("TNB_LANES", "16"))))
            lanes = 1 if os.environ.get("TNB_ONE_LANE") == "1" else lanes
            return int(max(1, min(lanes, n_run, self.LANE_WINDOW_BYTES // max(1, one))))
        return int(max(1, min(n_run, self.BATCH_WINDOW_BYTES // max(1, one))))

    def workspace(self, dtype: int, device=None, batch: int = 0, n_run: int = 0):
        """Device workspace (torch.empty), cached per (dtype, device, windows).  batch = 0: the
        plan's default for a call running n_run slices (batch_windows)."""
        import torch

        dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
        nb = self.batch_windows(dtype, n_run) if batch == 0 else batch
        key = (dtype, str(dev), nb)
        ws = self._ws.get(key)
        if ws is None:
            ws = torch.empty(B.tn_workspace_bytes(self.handle, dtype, nb), dtype=torch.uint8, device=dev)
            self._ws[key] = ws
        return ws

    def release_workspaces(self):
        self._ws.clear()

    # ------------------------------------------------------------ calls
    def _stream(self, stream):
        import torch

        s = torch.cuda.current_stream() if stream is None else stream
        return s.cuda_stream

    def contract(self, gammas, betas, dtype: int = TN_C64, stream=None) -> complex:
        ws = self.workspace(dtype)
        return B.tn_contract(self.handle, dtype, gammas, betas, ws.data_ptr(), ws.numel(), self._stream(stream))

    def contract_sliced(self, gammas, betas, begin: int, end: int, partials, dtype: int = TN_C64,
                        stream=None) -> None:
        ws = self.workspace(dtype, n_run=max(1, end - begin))
        B.tn_contract_sliced(self.handle, dtype, gammas, betas, begin, end, ws.data_ptr(), ws.numel(),
                             self._stream(stream), partials.data_ptr())

    def sum_partials(self, partials_host) -> complex:
        return B.tn_sum_partials(self.handle, partials_host)

    def energy(self, gammas, betas, dtype: int = TN_C64, stream=None):
        ws = self.workspace(dtype, batch=1)
        return B.tn_energy(self.handle, dtype, gammas, betas, ws.data_ptr(), ws.numel(), self._stream(stream))

    def energy_batch(self, gammas_sets, betas_sets, dtype: int = TN_C64, stream=None):
        """B parameter sets in one launch (tn_energy_batch): (zz[B][E], imag_max[B], energy[B])."""
        ws = self.workspace(dtype, batch=len(gammas_sets))
        return B.tn_energy_batch(self.handle, dtype, gammas_sets, betas_sets, ws.data_ptr(), ws.numel(),
                                 self._stream(stream))

    def profile(self, enable: bool = True):
        B.tn_profile_enable(self.handle, enable)

    def profile_read(self):
        return B.tn_profile_read(self.handle)

    def profile_records(self):
        """Per-launch (step range, kernel, ms, algorithmic bytes); call before profile_read()."""
        return B.tn_profile_records(self.handle)


def build_plan(graph, p: int, kind: str = "amplitude", orderer: str = "min-fill", n_sliced: int = 0,
               r: int = 0, max_width: int = 0, small_log2: int = -1, rg_q: int = 0, rg_tau: float = 0.0,
               rg_seed: int = 0, open_qubits=()) -> Plan:
    """Plan for a tn_inputs.Graph (or any object with .n and .edges).  open_qubits: output wires
    left open -- the plan then yields the batch of 2^a amplitudes (§6)."""
    k = TN_KIND_AMPLITUDE if kind == "amplitude" else TN_KIND_ENERGY
    buf = B.tn_plan_build(graph.n, graph.edges, p, kind=k, orderer=ORDERERS[orderer], n_sliced=n_sliced,
                          r=r, max_width=max_width, small_log2=small_log2, rg_q=rg_q, rg_tau=rg_tau,
                          rg_seed=rg_seed, open_qubits=open_qubits)
    plan = Plan(buf)
    plan.orderer = orderer
    return plan


DEFAULT_ORDERERS = (("min-fill", 0, 0.0, 0), ("min-degree", 0, 0.0, 0),
                    ("rgreedy", 8, 0.5, 0), ("rgreedy-fill", 8, 0.3, 0), ("rgreedy-fill", 8, 0.5, 0),
                    ("rgreedy-fill", 8, 1.0, 0), ("rgreedy-fill", 8, 0.3, 1), ("rgreedy-fill", 8, 0.5, 1))


def select_sliced_plan(graph, p: int, max_width: int, k_min: int = 0, k_max: int = 12,
                       orderers=DEFAULT_ORDERERS, r: int = 0, small_log2: int = -1,
                       workers: int = 0) -> Tuple[Plan, List[dict]]:
    """Reading A11: among k in [k_min, k_max] and the orderers -- greedy min-fill /
    min-degree and rgreedy given as (name, q, tau, seed)
    -- the plan with the fewest predicted bytes subject to width <= max_width (ties -> smaller k,
    then the earlier orderer).  Candidates are planned in parallel host threads (the C planner
    runs with the GIL released)."""
    import os
    from concurrent.futures import ThreadPoolExecutor

    jobs = [(k, idx, spec) for k in range(k_min, k_max + 1) for idx, spec in enumerate(orderers)]

    def run(job):
        k, idx, spec = job
        o, q, tau, seed = spec if len(spec) == 4 else (*spec, 0)
        pl = build_plan(graph, p, "amplitude", o, n_sliced=k, r=r, small_log2=small_log2,
                        rg_q=q, rg_tau=tau, rg_seed=seed)
        pl.orderer = o if not q else f"{o}(q={q},tau={tau},seed={seed})"
        total = pl.info["pred_bytes_per_slice"][0] * pl.n_slices + pl.info["pred_bytes_prefix"][0]
        return k, idx, pl, total

    nw = workers or min(len(jobs), max(1, (os.cpu_count() or 4)))
    with ThreadPoolExecutor(max_workers=nw) as ex:
        results = list(ex.map(run, jobs))
    tried, cands = [], []
    for k, idx, pl, total in results:
        o, q, tau, seed = orderers[idx] if len(orderers[idx]) == 4 else (*orderers[idx], 0)
        tried.append({"k": k, "orderer": pl.orderer, "width": pl.width, "pred_bytes_c64": total,
                      "unsliced_width": pl.info["unsliced_width"], "slice_step": pl.info["slice_step"],
                      "recipe": {"orderer": o, "n_sliced": k, "rg_q": q, "rg_tau": tau, "rg_seed": seed}})
        if pl.width <= max_width:
            cands.append((total, k, idx, pl))
    if not cands:
        raise TnError(-3, f"no plan with width <= {max_width} for k in [{k_min}, {k_max}]")
    cands.sort(key=lambda c: (c[0], c[1], c[2]))
    return cands[0][3], tried
