#!/usr/bin/env python
"""Benchmark: sliced single-amplitude contraction of the paper's 210-qubit QAOA circuit (C5a).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--workload C5a]

One STEP = one whole-job contraction sigma = <0^N|U(gamma, beta)|0^N> for a fresh (gamma, beta)
draw: leaf materialization, the shared prefix, this rank's block of the 2^k slices (Eq. 1), the
NCCL all-reduce of the per-slice partials (N > 1) -- every row of SURVEY.md §8(a) a6-a11.  The
plan (a1-a5: instance, network, ordering, step-dependent slicing, lowering) depends only on the
graph and is reused across parameters; its build time is reported
separately in config.plan_s.

value = contractions per second of the whole job (strong scaling: the total work -- one
amplitude -- is fixed, the slices are split across ranks).  Rank 0 prints ONE JSON line.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

from tn_inputs import WORKLOADS, qaoa_angles, random_regular_graph  # noqa: E402

MAX_WIDTH = {"C4a": 30, "C4b": 30, "C5a": 32, "C5b": 32, "C2": 62, "C5r": 32, "C5r6": 33}
K_RANGE = {"C4a": (8, 12), "C4b": (8, 12), "C5a": (5, 8), "C5b": (8, 16), "C2": (0, 0), "C5r": (9, 9), "C5r6": (6, 6)}
METRIC = "sliced single-amplitude contraction throughput (QAOA MaxCut, 3-regular)"


RECIPES = os.path.join(ROOT, "paper_2012_02430_b200", "plan_recipes.json")


def build_workload_plan(name: str = "C5a", seed: int = 0, search: bool = False):
    """Instance + plan for a named workload.  The plan is the best recipe recorded by the offline
    search (scripts/plan_search.py -> paper_2012_02430_b200/plan_recipes.json; reading A11),
    rebuilt deterministically; without a recipe (or search=True) the search runs here."""
    import paper_2012_02430_b200 as T

    w = WORKLOADS[name]
    g = random_regular_graph(w.n, 3, seed)
    ga, be = qaoa_angles(w.p, seed)
    cap = MAX_WIDTH.get(name, 32)
    t0 = time.perf_counter()
    rec = None
    if not search and os.path.exists(RECIPES):
        ent = json.load(open(RECIPES)).get(name)
        if ent and ent.get("seed_graph") == seed and ent.get("best"):
            # TNB_RECIPE_INDEX: another recorded candidate (plan comparisons; default the best)
            ix = int(os.environ.get("TNB_RECIPE_INDEX", "0"))
            rec = ent["best"][min(ix, len(ent["best"]) - 1)]
    if rec is not None:
        r = rec["recipe"]
        plan = T.build_plan(g, w.p, "amplitude", r["orderer"], n_sliced=r["n_sliced"], rg_q=r["rg_q"],
                            rg_tau=r["rg_tau"], rg_seed=r["rg_seed"], r=r.get("r", 0))
        if plan.width > cap:
            raise RuntimeError(f"recipe for {name} gives width {plan.width} > {cap}")
        plan.orderer = rec["orderer"]
        meta = {"plan_s": time.perf_counter() - t0, "tried": [rec],
                "source": "recipe from scripts/plan_search.py (paper_2012_02430_b200/plan_recipes.json)"}
        return plan, g, ga, be, meta
    kmin, kmax = K_RANGE.get(name, (0, 12))
    plan, tried = T.select_sliced_plan(g, w.p, cap, k_min=kmin, k_max=kmax)
    plan_s = time.perf_counter() - t0
    meta = {"plan_s": plan_s, "tried": tried, "candidates": len(tried), "source": "search at startup"}
    return plan, g, ga, be, meta


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            pk = json.load(f)
        return float(pk["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def fp32_peak_tflops() -> float:
    """FP32 FMA peak of the B200: 148 SMs x 128 FP32 lanes x 2 flops x the max SM clock."""
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            mhz = float(json.load(f).get("sm_max_mhz", 1965.0))
    except Exception:
        mhz = 1965.0
    return 148 * 128 * 2 * mhz * 1e6 / 1e12


# mma.sync m16n8k8 tf32 throughput measured on this pool's B200 (scripts/probe/mma_rate.cu,
# profiles/r02/hm/mma_rate.txt: 138.4 TMAC/s = 276.8 TFLOP/s dense tf32 on the warp-level path)
MMA_SYNC_TF32_TFLOPS = 276.8
TENSOR_FAMILIES = {"k_gemm_hm", "k_fc_hm"}


# FP64 FMA throughput measured on this pool's B200 (DFMA 18.1 TMAC/s, profiles/r02/hm/mma_rate.txt)
FP64_TFLOPS = 36.2


def alu_peak_tflops(kernel: str, c128: bool = False):
    """(peak, source) of a kernel family's arithmetic: FP32 FFMA for the SIMT kernels; for the
    mma.sync 3xTF32 kernels the measured tf32 rate / 3 (three products per complex-as-real MAC set),
    i.e. the FP32-equivalent rate of the flops bench counts (8 per complex multiply-add)."""
    if c128:
        return FP64_TFLOPS, "measured DFMA 18.1 TMAC/s (FP64 arithmetic of the c128 path), profiles/r02/hm/mma_rate.txt"
    if kernel in TENSOR_FAMILIES:
        return MMA_SYNC_TF32_TFLOPS / 3.0, ("measured mma.sync tf32 276.8 TFLOP/s / 3 (3xTF32), "
                                           "profiles/r02/hm/mma_rate.txt")
    return fp32_peak_tflops(), "148 SM x 128 FP32 lanes x 2 x sm_max_mhz (DESIGN.md section 5)"


def load_traffic(kernel: str) -> dict:
    """DRAM bytes per launch of `kernel` from the committed ncu --set full capture
    (profiles/traffic.json, written by scripts/ncu_traffic.py)."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            return json.load(f).get(kernel, {})
    except Exception:
        return {}


# ---------------------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:6]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------- oracle timing
SCHEDULES = os.path.join(ROOT, "tests", "golden", "schedules.json")


def host_info() -> dict:
    """CPU model, logical cores and the cores this process may use."""
    model = None
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                model = ln.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    try:
        usable = len(os.sched_getaffinity(0))
    except AttributeError:
        usable = os.cpu_count() or 1
    return {"cpu_model": model, "nproc": os.cpu_count(), "usable_cores": usable}


def committed_schedule(name: str) -> dict:
    """The workload's schedule as DATA (tests/golden/schedules.json, scripts/dump_schedules.py):
    the oracle arm reads it instead of calling the product planner."""
    with open(SCHEDULES) as f:
        return json.load(f)[name]


def oracle_contraction(name: str, ga, be, slices=None, workers: int = 1, max_width: int = 22,
                       sched: dict | None = None):
    """The oracle (as it stands: complex128 numpy.einsum per bucket, oracle/contract.py) on the
    workload's committed schedule: prefix once, then the given slices (default: all 2^k), each
    sub-sliced exactly (Eq. 1) to max_width, the (slice, sub-slice) evaluations spread over
    `workers` processes.  Returns (sum of the slice values, seconds, n_slices run, sub-slices per
    slice)."""
    from oracle import contract, network

    s = committed_schedule(name) if sched is None else sched
    if s["k"] == 0 and "oracle_aux" in s:
        s = s["oracle_aux"]
    g = random_regular_graph(WORKLOADS[name].n, 3, 0)
    n_sl = 1 << len(s["sliced"])
    js = list(range(n_sl)) if slices is None else list(slices)
    t0 = time.perf_counter()
    tens = network.qaoa_amplitude_network(g.n, g.edges, ga, be)
    vals, extra = contract.slice_values(tens, s["prefix"], s["sliced"], s["residual"], js,
                                        max_width=max_width, workers=workers)
    dt = time.perf_counter() - t0
    return contract.pairwise_sum(vals), dt, len(js), 1 << len(extra)


def oracle_cpu_baseline(name: str, ga, be, budget_s: float = 20.0) -> dict:
    """cpu_baseline of the ours arm: the oracle on all usable host cores on a BOUNDED sample of the
    same contraction -- the prefix plus as many WHOLE slices (each = its 2^m exact sub-slices) as
    fit in about budget_s, scaled to contractions/s by 2^k / (slices run).  When the whole
    contraction fits in the budget it is timed whole (sample fraction 1)."""
    hi = host_info()
    P = hi["usable_cores"]
    s = committed_schedule(name)
    n_sl = 1 << s["k"]
    # probe: slice 0 alone (its sub-slices over all cores); a batch of slices keeps every core busy
    _, t1, _, sub = oracle_contraction(name, ga, be, slices=[0], workers=P)
    per_slice = t1 * min(1.0, sub / P)
    if s["k"] == 0 or per_slice * n_sl <= budget_s:
        _, t, ns, sub = oracle_contraction(name, ga, be, workers=P)
        frac, cps = 1.0, 1.0 / t
        what = f"the whole contraction ({ns} slice(s) x {sub} exact sub-slices)"
    else:
        cnt = int(min(n_sl, max(1, budget_s // per_slice)))
        _, t, ns, sub = oracle_contraction(name, ga, be, slices=range(cnt), workers=P)
        frac = ns / n_sl
        cps = frac / t
        what = f"the prefix + {ns} of {n_sl} whole slices (each {sub} exact sub-slices), scaled x {n_sl}/{ns}"
    return {"value": cps, "unit": "contractions/s", "cores": P, "kind": "oracle",
            "sample": (f"{what}; committed schedule (tests/golden/schedules.json), complex128 numpy.einsum per "
                       f"bucket, {P} worker processes on {hi['cpu_model']} ({hi['nproc']} logical CPUs)"),
            "sample_fraction": frac, "sample_seconds": t, "host": hi}


# ---------------------------------------------------------------------------- main
def spawn_ranks(n: int):
    """Re-exec this command under torch.distributed.run with n ranks on this node (127.0.0.1)."""
    import socket

    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    os.execv(sys.executable, cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="C5a")
    ap.add_argument("--dtype", default="c64", choices=["c64", "c128"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--oracle-budget", type=float, default=20.0)
    ap.add_argument("--reference-budget", type=float, default=240.0)
    args = ap.parse_args()

    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # `python bench.py --gpus N` without a launcher: re-exec under torchrun, one rank per GPU
        spawn_ranks(args.gpus)
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}: launch one rank per GPU")

    if args.impl == "reference":
        return main_reference(args, rank, world)

    import torch
    import torch.distributed as dist

    import paper_2012_02430_b200 as T

    # one process per GPU (torchrun); TNB_BENCH_BACKEND=gloo and local % device_count exist only for a
    # functional check of the multi-rank path on a one-GPU box (not a measurement)
    local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    if world > 1:
        backend = os.environ.get("TNB_BENCH_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    dtype = T.TN_C64 if args.dtype == "c64" else T.TN_C128
    plan, g, ga0, be0, meta = build_workload_plan(args.workload)
    info = plan.info
    n = plan.n_slices
    from paper_2012_02430_b200.scheduler import slice_block
    begin, end = slice_block(n, rank, world)
    w = WORKLOADS[args.workload]
    params = [qaoa_angles(w.p, 1000 + s) for s in range(args.warmup + args.steps)]
    stream = torch.cuda.current_stream()
    dev = torch.device("cuda", local)
    partials = torch.zeros(2 * n, dtype=torch.float64, device=dev)
    ws = plan.workspace(dtype, dev, n_run=end - begin)
    lanes = plan.batch_windows(dtype, end - begin) if not info["slices_batchable"] else 1

    def step(ga, be):
        partials.zero_()
        if end > begin:
            plan.contract_sliced(ga, be, begin, end, partials, dtype=dtype)
        if world > 1:
            dist.all_reduce(partials)

    for s in range(args.warmup):
        step(*params[s])
    torch.cuda.synchronize()
    plan.profile_read()                      # reset counters
    sampler = ClockSampler(local)
    sampler.start()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for s in range(args.steps):
        step(*params[args.warmup + s])
    ev1.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = sampler.stop()
    prof = plan.profile_read()               # launch count of the timed region
    ms = ev0.elapsed_time(ev1)
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    ms_step = ms_max / args.steps
    value = 1000.0 / ms_step

    # ---- e2e through the public API: host params in, host result out (D2H + host sum inside)
    e2e_ms = []
    for s in range(max(1, min(args.steps, 3))):
        ga, be = params[s]
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        partials.zero_()
        if end > begin:
            plan.contract_sliced(ga, be, begin, end, partials, dtype=dtype)
        if world > 1:
            dist.all_reduce(partials)
        host = partials.cpu()
        sigma = plan.sum_partials(host.tolist())
        e1.record(stream)
        torch.cuda.synchronize()
        e2e_ms.append(e0.elapsed_time(e1))
    te = torch.tensor([statistics.mean(e2e_ms)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_value = 1000.0 / float(te.item())

    # ---- per-rank breakdown (after the timed region): prefix alone (an empty slice range runs the
    # leaves and the shared prefix only), this rank's slices without the all-reduce, the all-reduce
    def ev_ms(fn, reps):
        out = []
        for _ in range(reps):
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            fn()
            b.record(stream)
            torch.cuda.synchronize()
            out.append(a.elapsed_time(b))
        return statistics.median(out)

    ga_b, be_b = params[args.warmup]
    prefix_ms = ev_ms(lambda: plan.contract_sliced(ga_b, be_b, begin, begin, partials, dtype=dtype), 5)
    slices_ms = ev_ms(lambda: plan.contract_sliced(ga_b, be_b, begin, end, partials, dtype=dtype), 3) \
        if end > begin else 0.0
    ar_ms = ev_ms(lambda: dist.all_reduce(partials), 10) if world > 1 else 0.0
    mine = torch.tensor([prefix_ms, slices_ms, ar_ms, float(end - begin)], dtype=torch.float64, device=dev)
    if world > 1:
        allr = [torch.zeros_like(mine) for _ in range(world)]
        dist.all_gather(allr, mine)
        per_rank = [r.tolist() for r in allr]
    else:
        per_rank = [mine.tolist()]
    # 1-GPU reference time for the scaling efficiency: rank 0 alone runs every slice (the others
    # wait at a barrier); E(G) = T(1) / (G T(G)), with and without the (replicated) prefix
    t1_ms = None
    if world > 1:
        dist.barrier()
        if rank == 0:
            t1_ms = ev_ms(lambda: plan.contract_sliced(ga_b, be_b, 0, n, partials, dtype=dtype), 3)
            plan.release_workspaces()
        dist.barrier()
    else:
        t1_ms = ms_step
    pmax = max(r[0] for r in per_rank)
    multi = {"per_rank": [{"rank": i, "slices": int(r[3]), "prefix_ms": r[0], "slices_ms": r[1],
                           "allreduce_us": r[2] * 1e3} for i, r in enumerate(per_rank)],
             "max_slices_ms": max(r[1] for r in per_rank), "max_prefix_ms": pmax,
             "t1_ms_rank0_all_slices": t1_ms,
             "efficiency": (t1_ms / (world * ms_step)) if t1_ms else None,
             "efficiency_without_prefix": ((t1_ms - pmax) / (world * (ms_step - pmax)))
             if t1_ms and ms_step > pmax else None,
             "what": "per rank: materialise + prefix alone, its block of slices (lanes sized from the block), "
                     "the NCCL all-reduce of the 2*2^k partials; T(1) = rank 0 running all 2^k slices alone; "
                     "E = T(1) / (G T(G)) -- the driver computes its own scaling from the per-N values"}

    # ---- kernel pass: the timed region runs `lanes` slices concurrently, so a launch's duration
    # there includes sharing the GPU with other lanes.  Per-launch rates are therefore measured in
    # an isolated pass right after it: the same step, one lane (a one-window workspace), CUDA events
    # around every launch on its stream.
    ws1 = plan.workspace(dtype, dev, batch=1)
    kp_steps = max(1, min(args.steps, 2))
    torch.cuda.synchronize()
    plan.profile(True)
    k0, k1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    k0.record(stream)
    for s in range(kp_steps):
        ga, be = params[args.warmup + s]
        partials.zero_()
        if end > begin:
            T._binding.tn_contract_sliced(plan.handle, dtype, ga, be, begin, end, ws1.data_ptr(), ws1.numel(),
                                          stream.cuda_stream, partials.data_ptr())
    k1.record(stream)
    torch.cuda.synchronize()
    plan.profile(False)
    recs = plan.profile_records()
    plan.profile_read()
    ms_iso = k0.elapsed_time(k1) / kp_steps

    # ---- roofline of the dominant kernel family (by device time in the isolated pass)
    peak, peak_src = load_peaks()
    fam = {}
    for r in recs:
        f = fam.setdefault(r["kernel"], {"ms": 0.0, "bytes": 0.0, "flops": 0.0, "launches": 0})
        f["ms"] += r["ms"]
        f["bytes"] += r["bytes"]
        f["flops"] += r["flops"]
        f["launches"] += 1
    kb_ms = sum(f["ms"] for f in fam.values())
    dom = max(fam, key=lambda k: fam[k]["ms"]) if fam else None
    roof = {"bound": "hbm", "achieved": None, "peak": peak, "unit": "GB/s", "frac": None, "traffic": None}
    if dom is not None:
        d = fam[dom]
        # arithmetic peak of the family: FP32 FFMA for the SIMT kernels, the measured mma.sync tf32
        # rate / 3 (3xTF32 products) for the warp-level tensor-core kernels
        fp32_peak, alu_src = alu_peak_tflops(dom, dtype == T.TN_C128)
        achieved = d["bytes"] / (d["ms"] / 1e3) / 1e9
        t_hbm = d["bytes"] / (peak * 1e9)
        t_alu = d["flops"] / (fp32_peak * 1e12)
        tr = load_traffic(dom)
        bound = "hbm" if t_hbm >= t_alu else "alu"
        # an ALU-bound family is reported against its arithmetic peak (TFLOP/s); its HBM rate stays in "hbm"
        tflops = d["flops"] / (d["ms"] / 1e3) / 1e12
        roof = {"bound": bound,
                "achieved": achieved if bound == "hbm" else tflops,
                "peak": peak if bound == "hbm" else fp32_peak,
                "unit": "GB/s" if bound == "hbm" else "TFLOP/s",
                "frac": achieved / peak if bound == "hbm" else tflops / fp32_peak,
                "hbm": {"achieved_GBps": achieved, "peak_GBps": peak, "frac": achieved / peak},
                "traffic": tr.get("dram_bytes_per_launch"),
                "kernel": dom, "launches": d["launches"],
                "algorithmic_bytes_per_launch": d["bytes"] / d["launches"],
                "avg_launch_ms": d["ms"] / d["launches"],
                "kernel_share_of_step": (d["ms"] / kp_steps) / ms_iso if ms_iso else None,
                "measured": (f"isolated pass after the timed region: {kp_steps} step(s), 1 slice lane, CUDA "
                             f"events around every launch ({ms_iso:.2f} ms/step; the timed region runs "
                             f"{lanes} lanes)"),
                "flops_per_launch": d["flops"] / d["launches"],
                "alu": {"achieved_tflops": tflops, "peak_tflops": fp32_peak, "frac": tflops / fp32_peak,
                        "peak_source": alu_src},
                "peak_source": peak_src,
                "traffic_source": tr.get("source"),
                "traffic_algorithmic_bytes_per_launch": tr.get("algorithmic_bytes_per_launch"),
                "families": {k: {"ms_share_of_step": (v["ms"] / kp_steps) / ms_iso, "launches": v["launches"],
                                 "GBps": v["bytes"] / (v["ms"] / 1e3) / 1e9 if v["ms"] else None}
                             for k, v in sorted(fam.items(), key=lambda kv: -kv[1]["ms"])}}
        if tr.get("dram_bytes_per_launch") is None:
            roof["traffic"] = None
        # the timed region runs `lanes` slices concurrently; the per-kernel rates above come from
        # the isolated one-lane pass, the path-level rate (all algorithmic bytes of a step / the
        # timed step time) is the aggregate HBM throughput of the real run
        roof["concurrent_slice_lanes"] = lanes
    algo_bytes_step0 = (info["pred_bytes_per_slice"][dtype] * n + info["pred_bytes_prefix"][dtype] * world)
    # the largest per-slice tensor a launch writes: a group's final output (fused groups never write
    # the head's wider output); approximated by the largest out_rank among steps ending a launch
    st_ = [s_ for s_ in plan.steps() if s_["phase"] == 1]
    max_mat = max([s_["out_rank"] for i_, s_ in enumerate(st_)
                   if i_ + 1 == len(st_) or not st_[i_ + 1]["inplace"]] or [0])
    roof["path"] = {"achieved_GBps": algo_bytes_step0 / (ms_step / 1e3) / 1e9,
                    "frac": algo_bytes_step0 / (ms_step / 1e3) / 1e9 / peak,
                    "what": "algorithmic bytes of every launch of the contraction (fused groups: inputs + "
                            "final output; an OP_GROUP_FEED pair: its intermediate never moves) / device "
                            "time per contraction"}
    # the same time against the method's own bytes: every bucket step reading its inputs and writing
    # its output once (no fusion) -- the traffic a step-by-step contraction would need
    bsz = 8 if dtype == T.TN_C64 else 16
    meth = 0.0
    for s_ in plan.steps():
        mult = n if s_["phase"] == 1 else world
        meth += mult * s_["bytes_c64"] * bsz / 8
    roof["path"]["method_GB_per_step"] = meth / 1e9
    roof["path"]["method_GBps"] = meth / (ms_step / 1e3) / 1e9
    roof["path"]["method_frac"] = meth / (ms_step / 1e3) / 1e9 / peak
    roof["path"]["method_what"] = ("bytes a step-by-step bucket elimination moves (every step reads its inputs and "
                                   "writes its output, SURVEY 8(d) 'method bytes') / the same device time: an "
                                   "equivalent rate, > peak because fusion avoids most of those bytes")
    gpu_launches = prof["all_launches"]
    algo_bytes_step = (info["pred_bytes_per_slice"][dtype] * n + info["pred_bytes_prefix"][dtype] * world)

    line = {
        "metric": METRIC,
        "value": value,
        "unit": "contractions/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms_step,
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "c64 (fp32 complex)" if dtype == T.TN_C64 else "c128 (fp64 complex)",
        "data": "synthetic: seeded random 3-regular graph + U(0,pi) angles (tn_inputs)",
        "config": {
            "workload": f"{args.workload}: QAOA MaxCut p={w.p}, N={w.n} ({len(g.edges)} edges), single amplitude",
            "n_qubits": w.n, "p": w.p, "seed": 0,
            "plan": {"orderer": plan.orderer,
                     "k": info["k"], "n_slices": n, "slice_step": info["slice_step"],
                     "width": info["width"], "unsliced_width": info["unsliced_width"],
                     "steps_per_slice": info["steps_per_slice"], "prefix_steps": info["prefix_steps"],
                     "workspace_GB": info["workspace_bytes"][dtype] / 1e9},
            "plan_s": meta["plan_s"], "plan_source": meta.get("source"),
            "parallelism": f"slices x{world} (contiguous blocks, 1 NCCL all-reduce); {lanes} concurrent slice lanes per GPU",
            "l2": "no flush needed: every slice writes and reads intermediates of up to 2^%d x %d B "
                  "(%.0f MB; the widest step's output is consumed in registers when fused) >> the 126 MB L2, "
                  "and %d slices per step cycle through %.1f GB of workspace" % (
                      max_mat, 8 if dtype == T.TN_C64 else 16, (2 ** max_mat) * (8 if dtype == T.TN_C64 else 16) / 1e6,
                      n, info["workspace_bytes"][dtype] * lanes / 1e9),
            "algorithmic_GB_per_step": algo_bytes_step / 1e9,
            "step_GBps_algorithmic": algo_bytes_step / (ms_step / 1e3) / 1e9,
        },
        "roofline": roof,
        "clocks": clocks,
        "e2e": {"value": e2e_value, "unit": "contractions/s",
                "h2d_bytes_per_step": 2 * w.p * 8, "d2h_bytes_per_step": 16 * n},
        "gpu_launches": gpu_launches,
        "multi_gpu": multi,
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            line["cpu_baseline"] = oracle_cpu_baseline(args.workload, ga0, be0, budget_s=args.oracle_budget)
        except Exception as e:  # never let the baseline break the bench line
            line["cpu_baseline"] = {"value": None, "unit": "contractions/s", "cores": None, "kind": "oracle",
                                    "sample": f"failed: {e!r}"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main_reference(args, rank, world):
    """--impl reference: the oracle (as it stands: complex128 numpy.einsum per bucket) on all usable
    host cores, rank 0 only (other ranks exit 0 without work).  It reads the workload's schedule as
    data from tests/golden/schedules.json and loads NO product code (no libtnb200.so).  One step =
    one WHOLE contraction for a fresh (gamma, beta) draw (the ours arm's parameter sequence):
    the prefix and every slice, each slice sub-sliced exactly (Eq. 1) so numpy's complex128
    tensors stay small, the (slice, sub-slice) evaluations over a process pool.  Steps run until
    --steps are done or --reference-budget seconds are spent (at least one), so the run ends
    within a few minutes; the line reports the steps actually timed.  Warm-up: each warm-up step
    builds the network and contracts the prefix (the oracle has no caches or compiled state)."""
    if rank != 0:
        return
    hi = host_info()
    P = hi["usable_cores"]
    w = WORKLOADS[args.workload]
    sch = committed_schedule(args.workload)
    params = [qaoa_angles(w.p, 1000 + s) for s in range(args.warmup + args.steps)]
    from oracle import contract, network

    g = random_regular_graph(w.n, 3, 0)
    for s in range(args.warmup):
        ga, be = params[s]
        sc = sch["oracle_aux"] if sch["k"] == 0 and "oracle_aux" in sch else sch
        tens = network.qaoa_amplitude_network(w.n, g.edges, ga, be)
        contract.partial_eliminate(tens, sc["prefix"])
    times, sub, ns = [], 0, 0
    t_start = time.perf_counter()
    for s in range(args.steps):
        ga, be = params[args.warmup + s]
        _, t, ns, sub = oracle_contraction(args.workload, ga, be, workers=P, sched=sch)
        times.append(t)
        if time.perf_counter() - t_start + t > args.reference_budget:
            break
    ms = 1000.0 * statistics.mean(times)
    v = 1000.0 / ms
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "contractions/s",
            "n_gpus": world, "steps": len(times), "steps_requested": args.steps, "warmup": args.warmup,
            "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "c128 (fp64 complex, numpy)", "data": "synthetic",
            "config": {"workload": f"{args.workload}: QAOA MaxCut p={w.p}, N={w.n}", "k": sch["k"],
                       "width": sch["width"], "schedule": "tests/golden/schedules.json (the ours arm's plan)"},
            "cpu_baseline": {"value": v, "unit": "contractions/s", "cores": P, "kind": "oracle",
                             "sample": (f"whole contractions ({ns} slices x {sub} exact sub-slices each), "
                                        f"{len(times)} timed, {P} worker processes on {hi['cpu_model']} "
                                        f"({hi['nproc']} logical CPUs)"),
                             "sample_fraction": 1.0, "host": hi},
            "e2e": {"value": v, "unit": "contractions/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "step_seconds": times}
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
