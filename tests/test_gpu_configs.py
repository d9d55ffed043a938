"""GPU parity of every BASELINE amplitude config at its bench plan and full size, against committed
oracle values (tests/golden/oracle_configs.json, written by scripts/make_oracle_goldens.py, which
imports only oracle/), and against closed forms at full scale in the large-tensor regime.

Tolerances (BASELINE.json north_star): relative error <= 1e-4 for complex64, <= 1e-10 for
complex128.  A per-slice value is compared relative to the largest sampled slice of the same
config (a single slice can be a small term of the Eq. (1) sum).

The plans are rebuilt exactly as bench.py builds them (bench.build_workload_plan); the per-slice
golden values hold for the committed schedule only, so each test first checks that the rebuilt
plan's schedule is the committed one (tests/golden/schedules.json).
"""
import json
import math
import os

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # the -m gpu suite runs on a B200 only
    pytest.skip("no CUDA device", allow_module_level=True)

import bench  # noqa: E402
import paper_2012_02430_b200 as T  # noqa: E402
from paper_2012_02430_b200 import _binding as B  # noqa: E402
from paper_2012_02430_b200.scheduler import run_sliced  # noqa: E402
from oracle import closed_forms as cf  # noqa: E402
from tn_inputs import random_regular_graph  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = json.load(open(os.path.join(HERE, "golden", "oracle_configs.json")))
SCHED = json.load(open(os.path.join(HERE, "golden", "schedules.json")))
TOL = {T.TN_C64: 1e-4, T.TN_C128: 1e-10}
_PLANS = {}


def rel(a, b):
    return abs(a - b) / max(abs(b), 1e-300)


def _plan(name):
    if name not in _PLANS:
        plan, g, ga, be, meta = bench.build_workload_plan(name)
        pre, sl, res, _ = plan.schedule()
        s = SCHED[name]
        assert (list(pre), list(sl), list(res)) == (s["prefix"], s["sliced"], s["residual"]), \
            f"{name}: the rebuilt bench plan's schedule differs from tests/golden/schedules.json"
        _PLANS.clear()                     # one big plan (and its workspaces) at a time
        torch.cuda.empty_cache()
        _PLANS[name] = (plan, g, ga, be)
    return _PLANS[name]


def _gold_angles(name):
    src = "C5a" if name in ("C5r", "C5r6") else name
    return GOLD[src]


@pytest.mark.parametrize("dtype", [T.TN_C64, T.TN_C128])
@pytest.mark.parametrize("name", ["C2", "C4a", "C4b", "C5a", "C5r"])
def test_config_sigma_vs_oracle(name, dtype):
    """The whole amplitude sigma of the config (every slice, the default workspace with its slice
    lanes, one all-reduce-free sum) vs the oracle's complex128 sigma.  C5r (the paper-replica
    min-degree plan, width 30: bucket steps on 2^28-2^30-element tensors) is the same instance
    and angles as C5a, so it has the same sigma."""
    plan, g, ga, be = _plan(name)
    gd = _gold_angles(name)
    assert (ga, be) == (gd["gammas"], gd["betas"])
    ref = complex(*gd["sigma"])
    got, _ = run_sliced(plan, ga, be, dtype=dtype)
    assert rel(got, ref) < TOL[dtype], (name, got, ref)


def test_c2_min_fill_plan_vs_oracle():
    """C2 with BASELINE's own orderer (greedy min-fill, unsliced) -- the oracle's sigma does not
    depend on the plan.  (Width 27 on this seed's instance; BASELINE's "<= 2^24" is the survey's
    networkx instance: widths depend on the instance.)"""
    g = random_regular_graph(56, 3, 0)
    ga, be = GOLD["C2"]["gammas"], GOLD["C2"]["betas"]
    plan = T.build_plan(g, 2, "amplitude", "min-fill")
    assert plan.width <= 28
    for dt in (T.TN_C64, T.TN_C128):
        assert rel(plan.contract(ga, be, dtype=dt), complex(*GOLD["C2"]["sigma"])) < TOL[dt]


@pytest.mark.parametrize("dtype", [T.TN_C64, T.TN_C128])
@pytest.mark.parametrize("name", ["C4a", "C4b", "C5a", "C5b"])
def test_config_slices_vs_oracle(name, dtype):
    """Sampled slices of the bench plan (its schedule as data) vs the oracle's per-slice values:
    C4a / C4b {0, 128, 255}, C5a {0, 16, 31}, C5b {0} (2^14 slices of width 30)."""
    plan, g, ga, be = _plan(name)
    gd = GOLD[name]
    n = plan.n_slices
    part = torch.zeros(2 * n, dtype=torch.float64, device="cuda")
    js = sorted(int(j) for j in gd["slices"])
    for j in js:
        plan.contract_sliced(ga, be, j, j + 1, part, dtype=dtype)
    torch.cuda.synchronize()
    h = part.cpu().tolist()
    scale = max(abs(complex(*gd["slices"][str(j)])) for j in js)
    for j in js:
        got, ref = complex(h[2 * j], h[2 * j + 1]), complex(*gd["slices"][str(j)])
        assert abs(got - ref) / scale < TOL[dtype], (name, j, got, ref)


@pytest.mark.parametrize("which", ["gamma0", "beta0", "gammapi"])
@pytest.mark.parametrize("name", ["C2", "C4a", "C4b", "C5r"])
def test_config_closed_forms_full_scale(name, which):
    """Closed forms that hold at any N (oracle/closed_forms.py, pinned against the state vector):
    every config's whole contraction at its bench plan, c64."""
    plan, g, ga, be = _plan(name)
    n, p = g.n, len(ga)
    if which == "gamma0":
        ga, ref = [0.0] * p, cf.amp_gamma0(n, be)
    elif which == "beta0":
        be, ref = [0.0] * p, cf.amp_beta0(n)
    else:
        ga, ref = [math.pi] * p, cf.amp_gamma_pi(n, be)
    got, _ = run_sliced(plan, ga, be, dtype=T.TN_C64)
    assert rel(got, ref) < TOL[T.TN_C64], (name, which, got, ref)


def test_c5r_large_tensor_regime_runs_and_matches():
    """The paper-replica plan (min-degree, k = 9) materialises 2^28+-element
    intermediates in standalone launches: the profile shows launches writing outputs of rank >= 28
    (k_group_t / k_chain / k_bucket on 2-8 GiB tensors), and the contraction matches the oracle."""
    plan, g, ga, be = _plan("C5r")
    n = plan.n_slices
    ws = plan.workspace(T.TN_C64)
    part = torch.zeros(2 * n, dtype=torch.float64, device="cuda")
    plan.profile(True)
    B.tn_contract_sliced(plan.handle, T.TN_C64, ga, be, 0, n, ws.data_ptr(), ws.numel(),
                         torch.cuda.current_stream().cuda_stream, part.data_ptr())
    torch.cuda.synchronize()
    recs = plan.profile_records()
    plan.profile(False)
    plan.profile_read()
    big = [r for r in recs if r["out_rank"] >= 28]
    assert big, "no launch wrote a 2^28+ tensor"
    assert {r["kernel"] for r in big} - {"k_program"}
    got = plan.sum_partials(part.cpu().tolist())
    assert rel(got, complex(*GOLD["C5a"]["sigma"])) < TOL[T.TN_C64]


def test_c5r6_width33_paper_plan_closed_form():
    """The paper's n = 6 plan (min-degree, 41 -> 33 on this instance; the paper's 44 -> 32):
    a 2^33-element (64 GiB c64) step, inside one B200's HBM; gamma = pi closed form and sigma."""
    plan, g, ga, be = _plan("C5r6")
    assert plan.width == 33
    got, _ = run_sliced(plan, [math.pi], be, dtype=T.TN_C64)
    assert rel(got, cf.amp_gamma_pi(g.n, be)) < TOL[T.TN_C64]
    got, _ = run_sliced(plan, ga, be, dtype=T.TN_C64)
    assert rel(got, complex(*GOLD["C5a"]["sigma"])) < TOL[T.TN_C64]
    plan.release_workspaces()
