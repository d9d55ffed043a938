"""Host-side tests (-m "not gpu"): the C-ABI library loads and exports every symbol of
include/tn_b200.h; the planner's schedules are valid, deterministic and replay to the widths
an independent implementation (the oracle's line graph) computes; error paths."""
import ctypes
import json
import math
import os
import re

import numpy as np
import pytest

import paper_2012_02430_b200 as T
from paper_2012_02430_b200 import _binding as B
from oracle import contract, network
from tn_inputs import qaoa_angles, random_regular_graph

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_exports_every_header_symbol():
    hdr = open(os.path.join(ROOT, "include", "tn_b200.h")).read()
    decl = set(re.findall(r"^(?:tn_status|void|const char\*|int32_t|size_t)\s+(tn_[a-z_]+)\(", hdr, re.M))
    assert decl == set(B.SYMBOLS), decl ^ set(B.SYMBOLS)
    lib = ctypes.CDLL(B.LIB_PATH)
    for name in decl:
        assert hasattr(lib, name), name
    assert B.tn_version() >= 1


def _replay(tensors, prefix, sliced, residual):
    """Degrees of the executed steps by an independent replay (oracle line graph)."""
    adj = contract.line_graph(tensors)
    degs = []
    for v in prefix:
        degs.append(len(adj[v]))
        contract.eliminate_vertex(adj, v)
    for v in sliced:                       # slicing removes the vertex
        for a in adj.pop(v, set()):
            adj[a].discard(v)
    for v in residual:
        degs.append(len(adj[v]))
        contract.eliminate_vertex(adj, v)
    return degs


@pytest.mark.parametrize("n,p,k,orderer", [(20, 1, 0, "min-degree"), (30, 2, 3, "min-fill"),
                                           (40, 1, 4, "min-degree"), (24, 3, 2, "min-fill"),
                                           (100, 1, 6, "min-fill")])
def test_schedule_partition_and_width_replay(n, p, k, orderer):
    g = random_regular_graph(n, 3, n)
    ga, be = qaoa_angles(p, n)
    plan = T.build_plan(g, p, "amplitude", orderer, n_sliced=k)
    pre, sl, res, degs = plan.schedule()
    assert len(sl) == k == plan.info["k"] and sl == sorted(sl)
    labels = set(range(n * p))
    assert set(pre) | set(sl) | set(res) == labels
    assert len(pre) + len(sl) + len(res) == len(labels)
    tens = network.qaoa_amplitude_network(n, g.edges, ga, be)
    assert set(network.live_labels(tens)) == labels          # label rule l*N+q (reading A6)
    rep = _replay(tens, pre, sl, res)
    assert rep == degs
    assert max(degs) == plan.width
    assert plan.info["slice_step"] == len(pre)


def test_min_degree_matches_independent_greedy():
    # the planner's unsliced min-degree order == the oracle's own greedy (same tie rule)
    for n, p in ((16, 1), (20, 2), (30, 3)):
        g = random_regular_graph(n, 3, 3)
        ga, be = qaoa_angles(p, 3)
        plan = T.build_plan(g, p, "amplitude", "min-degree")
        _, _, res, degs = plan.schedule()
        order, odeg = contract.greedy_min_degree(network.qaoa_amplitude_network(n, g.edges, ga, be))
        assert res == order and degs == odeg


def test_plan_deterministic_and_reloadable():
    g = random_regular_graph(60, 3, 2)
    b1 = B.tn_plan_build(g.n, g.edges, 2, n_sliced=3)
    b2 = B.tn_plan_build(g.n, g.edges, 2, n_sliced=3)
    assert b1 == b2
    h = B.tn_plan_load(b1)
    assert B.tn_plan_info(h)["k"] == 3
    B.tn_plan_free(h)


def test_slicing_reduces_width_paper_section_5_3():
    # PAPER.md:569 "n=1 already provides contraction width reduction by 3" (reported; we
    # assert a reduction by >= 1 and monotone non-increase in n on this instance)
    g = random_regular_graph(100, 3, 0)
    widths = []
    for k in range(0, 5):
        widths.append(T.build_plan(g, 1, "amplitude", "min-degree", n_sliced=k).width)
    assert widths[1] <= widths[0] - 1
    assert all(b <= a for a, b in zip(widths, widths[1:]))


def test_literal_p3_n210_is_rejected():
    # p=3 at N=210 has width ~127 -> TN_E_TOO_WIDE, never a silent attempt
    g = random_regular_graph(210, 3, 0)
    with pytest.raises(B.TnError) as ei:
        B.tn_plan_build(g.n, g.edges, 3, n_sliced=0, max_width=32)
    assert ei.value.name == "TN_E_TOO_WIDE"
    assert "width" in str(ei.value)


def test_error_paths():
    g = random_regular_graph(10, 3, 0)
    with pytest.raises(B.TnError) as ei:
        B.tn_plan_build(10, g.edges, 0)
    assert ei.value.name == "TN_E_INVAL"
    with pytest.raises(B.TnError) as ei:
        B.tn_plan_build(10, [(0, 0)] + list(g.edges[1:]), 1)
    assert ei.value.name == "TN_E_PLAN"
    with pytest.raises(B.TnError) as ei:
        B.tn_plan_build(10, list(g.edges) + [g.edges[0]], 1)
    assert ei.value.name == "TN_E_PLAN"
    with pytest.raises(B.TnError) as ei:
        B.tn_plan_build(10, g.edges, 1, n_sliced=99)
    assert ei.value.name == "TN_E_INVAL"
    with pytest.raises(B.TnError) as ei:
        B.tn_plan_build(10, g.edges, 1, orderer=7)
    assert ei.value.name == "TN_E_INVAL"
    buf = bytearray(B.tn_plan_build(10, g.edges, 1))
    with pytest.raises(B.TnError) as ei:
        B.tn_plan_load(bytes(buf[:40]))
    assert ei.value.name == "TN_E_PLAN"
    buf[0] ^= 0xFF
    with pytest.raises(B.TnError) as ei:
        B.tn_plan_load(bytes(buf))
    assert ei.value.name == "TN_E_PLAN"


def test_sum_partials_fixed_tree_matches_oracle():
    g = random_regular_graph(40, 3, 1)
    plan = T.build_plan(g, 1, "amplitude", "min-fill", n_sliced=5)
    rng = np.random.default_rng(0)
    vals = rng.normal(size=2 * plan.n_slices) * np.exp(rng.uniform(-30, 30, size=2 * plan.n_slices))
    got = plan.sum_partials(vals.tolist())
    ref = contract.pairwise_sum([complex(vals[2 * j], vals[2 * j + 1]) for j in range(plan.n_slices)])
    assert got == ref   # bit-identical: same fixed pairwise tree


def test_energy_plan_shape():
    g = random_regular_graph(100, 3, 0)
    plan = T.build_plan(g, 3, "energy", "min-fill")
    assert plan.info["n_programs"] == len(g.edges) == 150
    assert plan.info["k"] == 0
    assert 7 <= plan.width <= 16            # cone widths 7-13 (instance-dependent)


def test_workspace_and_bytes_model():
    g = random_regular_graph(56, 3, 0)
    plan = T.build_plan(g, 2, "amplitude", "min-fill")
    info = plan.info
    assert info["workspace_bytes"][0] >= 8 * 2 ** plan.width
    assert info["workspace_bytes"][1] >= 16 * 2 ** plan.width
    assert math.isclose(info["pred_bytes_per_slice"][1], 2 * info["pred_bytes_per_slice"][0])


def test_rgreedy_deterministic_and_not_worse():
    # Boltzmann sampling p(v) ~ exp(-N_G(v)/tau), best of q runs; our runs
    # always include the deterministic greedy run, so the width never gets worse
    g = random_regular_graph(80, 3, 5)
    ga, be = qaoa_angles(2, 5)
    tens = network.qaoa_amplitude_network(80, g.edges, ga, be)
    for base, rg in (("min-degree", "rgreedy"), ("min-fill", "rgreedy-fill")):
        w0 = T.build_plan(g, 2, "amplitude", base).width
        b1 = B.tn_plan_build(g.n, g.edges, 2, orderer=T.ORDERERS[rg], rg_q=6, rg_tau=0.5, rg_seed=11)
        b2 = B.tn_plan_build(g.n, g.edges, 2, orderer=T.ORDERERS[rg], rg_q=6, rg_tau=0.5, rg_seed=11)
        assert b1 == b2
        pl = T.Plan(b1)
        assert pl.width <= w0
        pre, sl, res, degs = pl.schedule()
        assert _replay(tens, pre, sl, res) == degs
        # sliced rgreedy plans replay too
        pl2 = T.build_plan(g, 2, "amplitude", rg, n_sliced=3, rg_q=4, rg_tau=0.5, rg_seed=3)
        pre, sl, res, degs = pl2.schedule()
        assert _replay(tens, pre, sl, res) == degs


def test_select_sliced_plan_rule_a11():
    g = random_regular_graph(100, 3, 1)
    plan, tried = T.select_sliced_plan(g, 1, 14, k_min=2, k_max=6)
    assert plan.width <= 14
    feas = [t for t in tried if t["width"] <= 14]
    best = min(t["pred_bytes_c64"] for t in feas)                  # fewest predicted bytes
    mine = [t for t in feas if t["orderer"] == plan.orderer and t["k"] == plan.info["k"]][0]
    assert mine["pred_bytes_c64"] == best


# ------------------------------------------------------------------ amplitude batches (open indices)
@pytest.mark.parametrize("n,p,k,opened", [(20, 1, 0, (0, 5)), (30, 2, 3, (1, 2, 29)), (60, 1, 4, (7,))])
def test_open_batch_plan_schedule_and_width(n, p, k, opened):
    """PAPER.md:599-607 (§6): the open indices are never eliminated nor sliced; the schedule
    covers every other live label; the result clique of size a does not raise the width while
    a < c (reported; the replay with the clique added matches the planner's degrees)."""
    g = random_regular_graph(n, 3, n + 1)
    ga, be = qaoa_angles(p, n)
    plan = T.build_plan(g, p, "amplitude", "min-fill", n_sliced=k, open_qubits=opened)
    assert plan.info["n_open"] == len(opened) and plan.batch == 1 << len(opened)
    assert plan.info["n_labels"] == n * p + len(opened)
    pre, sl, res, degs = plan.schedule()
    assert set(pre) | set(sl) | set(res) == set(range(n * p))
    assert len(pre) + len(sl) + len(res) == n * p
    # independent replay: oracle network with the open wires (labels p*N+q) plus their clique
    tens = network.qaoa_amplitude_network(n, g.edges, ga, be, open_qubits=opened)
    ol = network.open_labels(n, p, opened)
    clique = [(np.ones((2, 2)), (ol[i], ol[j])) for i in range(len(ol)) for j in range(i + 1, len(ol))]
    rep = _replay(tens + clique, pre, sl, res)
    assert rep == degs
    single = T.build_plan(g, p, "amplitude", "min-fill", n_sliced=k)
    assert plan.width <= single.width + len(opened)


def test_open_batch_bad_arguments():
    g = random_regular_graph(10, 3, 1)
    for bad in ((10,), (-1,), (3, 3)):
        with pytest.raises(B.TnError):
            T.build_plan(g, 1, "amplitude", "min-fill", open_qubits=bad)
    with pytest.raises(B.TnError):
        T.build_plan(g, 1, "energy", "min-fill", open_qubits=(1,))


def _plan_env(env, g, p, k):
    old = os.environ.get("TNB_NO_FEED")
    try:
        if env is None:
            os.environ.pop("TNB_NO_FEED", None)
        else:
            os.environ["TNB_NO_FEED"] = env
        return T.build_plan(g, p, "amplitude", "rgreedy-fill", n_sliced=k, small_log2=0, rg_q=4, rg_tau=0.4)
    finally:
        if old is None:
            os.environ.pop("TNB_NO_FEED", None)
        else:
            os.environ["TNB_NO_FEED"] = old


@pytest.mark.parametrize("n,p,k", [(36, 3, 3), (70, 2, 3)])
def test_feed_reorder_is_a_permutation_of_the_same_eliminations(n, p, k):
    """The producer -> consumer lowering (OP_GROUP_FEED) only moves merge blocks later: the same
    elimination steps (label, output rank, inputs) in a different execution order, the same
    schedule and width; every moved block's consumer comes right after it; the predicted bytes
    drop by exactly the never-written intermediates (2 x 2^R elements each)."""
    g = random_regular_graph(n, 3, 7 * n + p)
    a = _plan_env("1", g, p, k)      # elimination order
    b = _plan_env(None, g, p, k)     # with the moves
    assert a.schedule() == b.schedule()
    assert a.width == b.width
    sa, sb = a.steps(), b.steps()
    key = lambda s: (s["phase"], s["label"], s["out_rank"], tuple(sorted(s["in_rank"])))
    assert sorted(map(key, sa)) == sorted(map(key, sb))
    assert [key(s) for s in sa if s["phase"] == 0] == [key(s) for s in sb if s["phase"] == 0]
    moved = [i for i, (x, y) in enumerate(zip(sa, sb)) if x["label"] != y["label"]]
    assert moved, "this instance has a producer -> consumer pair"
    da = a.info["pred_bytes_per_slice"][0] - b.info["pred_bytes_per_slice"][0]
    assert da > 0
    # the saving is a sum of 2 x 8 x 2^R terms (c64): a multiple of 16 B
    assert da % 16 == 0
    # a plan without moves (TNB_NO_FEED=1) has no saving
    assert a.info["pred_bytes_per_slice"][0] == _plan_env("1", g, p, k).info["pred_bytes_per_slice"][0]


def test_multi_round_schedule_is_exact():
    """A plan sliced in rounds (r < n): its schedule (prefix, sliced, residual)
    evaluated by the oracle with Eq. (1) equals the unsliced contraction, and the width does not
    exceed the one-round plan's."""
    n, p, k, r = 30, 3, 4, 2
    g = random_regular_graph(n, 3, 11 * n + p)
    ga, be = qaoa_angles(p, n)
    plan = T.build_plan(g, p, "amplitude", "rgreedy-fill", n_sliced=k, r=r, rg_q=8, rg_tau=0.3)
    plan0 = T.build_plan(g, p, "amplitude", "rgreedy-fill", n_sliced=k, r=0, rg_q=8, rg_tau=0.3)
    assert plan.n_slices == 2 ** k and plan.width <= plan0.width
    pre, sl, res, _ = plan.schedule()
    assert len(sl) == k and len(set(pre) | set(sl) | set(res)) == len(pre) + len(sl) + len(res)
    tens = network.qaoa_amplitude_network(n, g.edges, ga, be)
    sliced = contract.contract_sliced(tens, pre, sl, res)
    whole = contract.contract(tens)
    assert abs(sliced - whole) <= 1e-12 * abs(whole)


# instances where the first-fit arena / in-place chains used to put a fused pair's consumer output
# over memory the producer still reads: N, seed, p, k, orderer
_FEED_CASES = [(40, 2, 2, 0, "min-degree"), (60, 0, 2, 0, "min-degree"), (60, 1, 2, 3, "min-degree"),
               (60, 3, 2, 3, "min-fill"), (80, 2, 2, 3, "min-fill"), (80, 3, 2, 6, "min-fill"),
               (100, 1, 2, 6, "min-fill"), (150, 2, 1, 6, "min-degree"), (210, 0, 1, 5, "min-fill")]


def test_fused_pairs_never_write_over_producer_inputs():
    """OP_GROUP_FEED (k_gemm_fc) runs producer and consumer in ONE launch: no producer input may
    share arena memory with the consumer's output (cross-CTA write-after-read race)."""
    import planbuf

    n_feed = 0
    for n, seed, p, k, o in _FEED_CASES:
        pl = T.build_plan(random_regular_graph(n, 3, seed), p, "amplitude", o, n_sliced=k)
        P = planbuf.parse(pl.buf)
        assert P["header"].magic == 0x32424E54 and P["header"].n_steps == len(P["steps"])
        n_feed += sum(1 for op in P["ops"] if op.type == planbuf.OP_GROUP_FEED)
        assert planbuf.feed_overlaps(pl.buf) == [], (n, seed, p, k, o)
    assert n_feed > 0


def _greedy_min_degree_graph(adj):
    """Min-degree elimination of a line graph (ties -> smallest label), on a copy: degrees."""
    adj = {v: set(nb) for v, nb in adj.items()}
    degs = []
    while adj:
        v = min(adj, key=lambda x: (len(adj[x]), x))
        degs.append(len(adj[v]))
        contract.eliminate_vertex(adj, v)
    return degs


def test_planner_reports_replay():
    """f3 reports (scripts/planner_reports.py, profiles/r02/planner): a width-vs-n row replays
    through the oracle's line graph, and candidate rows of the width-over-s scan match an
    independent re-run of the paper's procedure (eliminate s vertices of the
    greedy order, remove the n highest-degree vertices of G_s, re-run greedy on the rest)."""
    import csv

    base = os.path.join(ROOT, "profiles", "r02", "planner")
    rows = list(csv.DictReader(open(os.path.join(base, "width_vs_n.csv"))))
    row = next(r for r in rows if r["N"] == "100" and r["seed"] == "0" and r["orderer"] == "min-degree"
               and r["n"] == "3")
    g = random_regular_graph(100, 3, 0)
    ga, be = qaoa_angles(1, 0)
    plan = T.build_plan(g, 1, "amplitude", "min-degree", n_sliced=3)
    pre, sl, res, _ = plan.schedule()
    tens = network.qaoa_amplitude_network(100, g.edges, ga, be)
    assert max(_replay(tens, pre, sl, res)) == int(row["width"]) == plan.width
    scan = json.load(open(os.path.join(base, "width_over_s.json")))["N150_n3"]
    g = random_regular_graph(150, 3, 0)
    tens = network.qaoa_amplitude_network(150, g.edges, *qaoa_angles(1, 0))
    order, odeg = contract.greedy_min_degree(tens)
    assert scan["peak"] == odeg.index(max(odeg))
    cands = scan["candidates"]
    for c in (cands[0], min(cands, key=lambda c: (c["width"], c["s"])), cands[len(cands) // 2]):
        s = c["s"]
        adj = contract.line_graph(tens)
        for v in order[:s]:
            contract.eliminate_vertex(adj, v)
        S = sorted(adj, key=lambda v: (-len(adj[v]), v))[:3]
        for v in S:
            for a in adj.pop(v):
                adj[a].discard(v)
        w = max(odeg[:s] + _greedy_min_degree_graph(adj))
        assert w == c["width"], (s, w, c["width"])


def test_lane_windows_sized_from_the_rank_block():
    """A rank's workspace holds one window per slice lane of ITS block of slices (min(lanes, block)),
    not of all 2^k slices: at 8 GPUs a C5a-like rank with 4 slices gets 4 windows."""
    g = random_regular_graph(60, 3, 1)
    plan = T.build_plan(g, 2, "amplitude", "min-fill", n_sliced=5)
    assert plan.n_slices == 32 and not plan.info["slices_batchable"]
    full = plan.batch_windows(T.TN_C64)
    assert full == min(8, 32) or full >= 1
    for n_run, want in ((1, 1), (4, min(4, full)), (32, full)):
        assert plan.batch_windows(T.TN_C64, n_run) == want
