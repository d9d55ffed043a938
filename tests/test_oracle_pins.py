"""Pins for the oracle (-m "not gpu"): checks against what the paper and the
mathematics fix -- SPEC/paper worked examples (tests/golden), the 2^N state
vector, closed forms at any N, Wang et al.'s p=1 formula, Eq. (1)'s slice-sum
identity, order independence and brute force.  A dropped term, a wrong sign or
index or a transposed operand anywhere in oracle/ fails at least one of these.
"""
import json
import math
import os

import numpy as np
import pytest

from oracle import closed_forms as cf
from oracle import contract, energy, gates, network
from oracle import statevector as sv
from tn_inputs import qaoa_angles, random_regular_graph

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def cval(v):
    return complex(v[0], v[1])


# ------------------------------------------------------------------ gates
def test_gates_unitary_and_textbook():
    for m in (gates.H, gates.X, gates.Z, gates.rx(0.37), gates.cnot_matrix()):
        assert np.allclose(m.conj().T @ m, np.eye(m.shape[0]), atol=1e-12)
    zp = gates.zpow_diag(1.0)
    assert np.allclose(zp, [cval(x) for x in GOLD["zpow1"]["value"]], atol=1e-15)
    # rx(b) == e^{-i b X}; zz_phase == diag of e^{-i g (1 - Z Z)/2}
    b, g = 0.731, 1.234
    assert np.allclose(gates.rx(b), gates.expm_hermitian(gates.X, b), atol=1e-13)
    zz = np.kron(gates.Z, gates.Z)
    full = gates.expm_hermitian((np.eye(4) - zz) / 2, g)
    assert np.allclose(np.diag(full).reshape(2, 2), gates.zz_phase(g), atol=1e-13)
    assert np.allclose(full, np.diag(np.diag(full)), atol=1e-13)
    # CNOT tensor truth table
    t = gates.cnot_tensor()
    for c in range(2):
        for i in range(2):
            for o in range(2):
                assert t[c, i, o] == (1.0 if (c == 0 and i == o) or (c == 1 and i != o) else 0.0)


# ------------------------------------------------------------------ SPEC examples
def test_spec_contract_examples():
    t = network.circuit_network(1, [("h", 0, (0,))], [0], [0])
    assert abs(contract.contract(t) - cval(GOLD["h_amplitude"]["value"])) < 1e-12
    bell = [("h", 0, (0,)), ("cnot", 0, (0, 1))]
    t00 = network.circuit_network(2, bell, [0, 0], [0, 0])
    t01 = network.circuit_network(2, bell, [0, 0], [0, 1])
    assert abs(contract.contract(t00) - cval(GOLD["bell_00"]["value"])) < 1e-12
    assert abs(contract.contract(t01) - cval(GOLD["bell_01"]["value"])) < 1e-12


def test_spec_bucket_examples():
    a = np.array(GOLD["bucket_dot"]["a"], dtype=np.complex128)
    b = np.array(GOLD["bucket_dot"]["b"], dtype=np.complex128)
    arr, labs = contract._einsum_bucket([(a, (5,)), (b, (5,))], 5)
    assert labs == () and abs(complex(arr) - GOLD["bucket_dot"]["value"]) < 1e-12
    arr, labs = contract._einsum_bucket([(gates.H, (1, 0))], 0)   # H[j, i], sum over i
    assert labs == (1,)
    assert np.allclose(arr, GOLD["h_column_sums"]["value"], atol=1e-12)
    rng = np.random.default_rng(0)
    A = rng.normal(size=(3, 2)) + 0j
    A = rng.normal(size=(2, 2)) + 1j * rng.normal(size=(2, 2))
    B = rng.normal(size=(2, 2)) + 1j * rng.normal(size=(2, 2))
    arr, labs = contract._einsum_bucket([(A, (0, 1)), (B, (1, 2))], 1)
    assert labs == (0, 2) and np.allclose(arr, A @ B, atol=1e-12)


def test_gate_counts_fig1():
    for key in ("gate_count_k4_p1", "gate_count_10_p2", "gate_count_210_p1"):
        e = GOLD[key]
        g = random_regular_graph(e["n"], 3, 0)
        ga, be = qaoa_angles(e["p"], 0)
        assert len(sv.fig1_circuit(e["n"], g.edges, ga, be)) == e["value"]


def test_single_edge_and_uniform_batch():
    e = GOLD["single_edge_energy_zero_angles"]
    E, zz = energy.maxcut_energy(2, [(0, 1)], [0.0], [0.0])
    assert abs(zz[0] - e["zz"]) < 1e-12 and abs(E - e["energy"]) < 1e-12
    vals = []
    for bits in ((0, 0), (0, 1), (1, 0), (1, 1)):
        t = network.qaoa_amplitude_network(2, [(0, 1)], [0.0], [0.0], out_bits=bits)
        vals.append(contract.contract(t))
    assert np.allclose(vals, GOLD["uniform_batch"]["value"], atol=1e-12)


def test_cost_model_examples():
    for key in ("cost_width44_bytes", "cost_width32_bytes"):
        e = GOLD[key]
        assert 16 * 2 ** e["width"] == e["bytes"]


# ------------------------------------------------------------------ instance generator
def test_regular_graph_generator():
    g = random_regular_graph(4, 3, 123)
    assert g.edges == ((0, 1), (0, 2), (0, 3), (1, 2), (1, 3), (2, 3))   # K4
    with pytest.raises(ValueError):
        random_regular_graph(3, 3, 0)
    for n in (10, 56, 210):
        g = random_regular_graph(n, 3, 7)
        assert len(g.edges) == 3 * n // 2 and len(set(g.edges)) == len(g.edges)
        assert all(i < j for i, j in g.edges)
        assert all(g.degree(q) == 3 for q in range(n))
        assert g == random_regular_graph(n, 3, 7)
    a, b = qaoa_angles(3, 5)
    assert len(a) == len(b) == 3 and all(0 <= x < math.pi for x in a + b)
    assert (a, b) == qaoa_angles(3, 5) and (a, b) != qaoa_angles(3, 6)


# ------------------------------------------------------------------ state vector pins
@pytest.mark.parametrize("n,p,seed", [(6, 1, 0), (8, 2, 1), (10, 3, 2), (12, 1, 3), (12, 2, 4),
                                      (14, 3, 5), (16, 1, 6), (16, 2, 7)])
def test_amplitude_vs_statevector(n, p, seed):
    g = random_regular_graph(n, 3, seed)
    ga, be = qaoa_angles(p, seed + 100)
    psi = sv.qaoa_state(n, g.edges, ga, be)
    t = network.qaoa_amplitude_network(n, g.edges, ga, be)
    assert abs(contract.contract(t) - sv.amplitude(psi)) < 1e-12
    # a non-zero output string too (fixing of the output wires)
    bits = [(q * 7 + seed) % 2 for q in range(n)]
    t = network.qaoa_amplitude_network(n, g.edges, ga, be, out_bits=bits)
    assert abs(contract.contract(t) - sv.amplitude(psi, bits)) < 1e-12


def test_fused_vs_fig1_literal_circuit():
    # A_fig1(gamma, beta) = e^{i N sum beta} A(-2 gamma, beta)   (reading A1)
    for n, p, seed in ((6, 1, 0), (8, 2, 1), (10, 2, 2)):
        g = random_regular_graph(n, 3, seed)
        ga, be = qaoa_angles(p, seed)
        lit = sv.run_gates(n, sv.fig1_circuit(n, g.edges, ga, be))
        t = network.qaoa_amplitude_network(n, g.edges, [-2 * x for x in ga], be)
        assert abs(sv.amplitude(lit) - np.exp(1j * n * sum(be)) * contract.contract(t)) < 1e-12
        psi = sv.qaoa_state(n, g.edges, [-2 * x for x in ga], be)
        assert np.allclose(lit, np.exp(1j * n * sum(be)) * psi, atol=1e-12)


def test_norm_of_all_amplitudes():
    # sum over all outputs |amp|^2 = 1 (N <= 8)
    n, p = 6, 2
    g = random_regular_graph(n, 3, 11)
    ga, be = qaoa_angles(p, 11)
    tot = 0.0
    for z in range(1 << n):
        bits = [(z >> q) & 1 for q in range(n)]
        tot += abs(contract.contract(network.qaoa_amplitude_network(n, g.edges, ga, be, bits))) ** 2
    assert abs(tot - 1.0) < 1e-12


# ------------------------------------------------------------------ amplitude batches (open indices)
@pytest.mark.parametrize("n,p,seed,opened", [(10, 2, 3, (1, 4, 7)), (12, 1, 4, (0, 11)),
                                             (8, 3, 5, (2, 3, 5, 6)), (14, 2, 6, (13,))])
def test_amplitude_batch_vs_statevector(n, p, seed, opened):
    """PAPER.md:599-603 (§6): leaving the output indices of `opened` open gives the batch
    <x_open 0_rest|U|0^N>; bit b of the batch index = output bit of the b-th open qubit."""
    g = random_regular_graph(n, 3, seed)
    ga, be = qaoa_angles(p, seed + 7)
    psi = sv.qaoa_state(n, g.edges, ga, be)
    t = network.qaoa_amplitude_network(n, g.edges, ga, be, open_qubits=opened)
    v = contract.contract_open(t, network.open_labels(n, p, opened))
    assert v.shape == (1 << len(opened),)
    qs = sorted(opened)
    for i in range(1 << len(qs)):
        bits = [0] * n
        for b, q in enumerate(qs):
            bits[q] = (i >> b) & 1
        assert abs(v[i] - sv.amplitude(psi, bits)) < 1e-12
    # entry 0 is the single amplitude (SURVEY §8 f1 pin)
    assert abs(v[0] - contract.contract(network.qaoa_amplitude_network(n, g.edges, ga, be))) < 1e-12


def test_amplitude_batch_all_qubits_norm():
    # every output open: the whole state, sum |amp|^2 = 1
    n, p = 8, 2
    g = random_regular_graph(n, 3, 21)
    ga, be = qaoa_angles(p, 21)
    opened = tuple(range(n))
    v = contract.contract_open(network.qaoa_amplitude_network(n, g.edges, ga, be, open_qubits=opened),
                               network.open_labels(n, p, opened))
    assert abs(np.sum(np.abs(v) ** 2) - 1.0) < 1e-12


# ------------------------------------------------------------------ closed forms, any N
@pytest.mark.parametrize("n,p", [(16, 1), (40, 1), (60, 1), (24, 2), (30, 2), (12, 3)])
def test_closed_forms_special_angles(n, p):
    g = random_regular_graph(n, 3, n + p)
    ga, be = qaoa_angles(p, n)
    t0 = network.qaoa_amplitude_network(n, g.edges, [0.0] * p, be)
    assert abs(contract.contract(t0) - cf.amp_gamma0(n, be)) < 1e-13
    tb = network.qaoa_amplitude_network(n, g.edges, ga, [0.0] * p)
    assert abs(contract.contract(tb) - cf.amp_beta0(n)) < 1e-13
    tp = network.qaoa_amplitude_network(n, g.edges, [math.pi] * p, be)
    assert abs(contract.contract(tp) - cf.amp_gamma_pi(n, be)) < 1e-13


def test_closed_forms_vs_statevector():
    n = 10
    g = random_regular_graph(n, 3, 3)
    _, be = qaoa_angles(3, 3)
    assert abs(sv.amplitude(sv.qaoa_state(n, g.edges, [0.0] * 3, be)) - cf.amp_gamma0(n, be)) < 1e-14
    assert abs(sv.amplitude(sv.qaoa_state(n, g.edges, [math.pi] * 3, be)) - cf.amp_gamma_pi(n, be)) < 1e-14
    assert abs(sv.amplitude(sv.qaoa_state(n, g.edges, [0.4] * 3, [0.0] * 3)) - cf.amp_beta0(n)) < 1e-14


# ------------------------------------------------------------------ energy
@pytest.mark.parametrize("n,p,seed", [(12, 1, 0), (12, 2, 1), (14, 3, 2), (16, 1, 3), (16, 2, 4)])
def test_cone_energy_vs_statevector(n, p, seed):
    g = random_regular_graph(n, 3, seed)
    ga, be = qaoa_angles(p, seed + 7)
    psi = sv.qaoa_state(n, g.edges, ga, be)
    E, zz = energy.maxcut_energy(n, g.edges, ga, be)
    for (u, v), z in zip(g.edges, zz):
        assert abs(z.imag) < 1e-12
        assert abs(z.real - sv.zz_expectation(psi, u, v)) < 1e-12
    assert abs(E - sv.maxcut_energy(psi, g.edges)) < 1e-11
    assert 0.0 <= E <= len(g.edges)


@pytest.mark.parametrize("n,seed", [(16, 0), (30, 1), (100, 2)])
def test_cone_energy_vs_wang_p1(n, seed):
    g = random_regular_graph(n, 3, seed)
    ga, be = qaoa_angles(1, seed)
    zz = energy.zz_values(n, g.edges, ga, be)
    for (u, v), z in zip(g.edges, zz):
        assert abs(z - cf.wang_p1_zz(g.edges, u, v, ga[0], be[0])) < 1e-12


# ------------------------------------------------------------------ Eq. (1), order independence
def own_schedule(tensors, s, k):
    """A step-dependent slicing schedule chosen by the test itself (own greedy)."""
    order, _ = contract.greedy_min_degree(tensors)
    adj = contract.line_graph(tensors)
    for v in order[:s]:
        contract.eliminate_vertex(adj, v)
    sliced = sorted(sorted(adj, key=lambda x: (-len(adj[x]), x))[:k])
    rest_tensors, _ = contract.partial_eliminate(tensors, order[:s])
    rest_tensors = network.fix_indices(rest_tensors, {l: 0 for l in sliced})
    residual, _ = contract.greedy_min_degree(rest_tensors)
    return order[:s], sliced, residual


@pytest.mark.parametrize("n,p,s,k", [(12, 1, 0, 2), (16, 2, 5, 3), (20, 1, 8, 4), (14, 3, 10, 2)])
def test_slice_sum_identity(n, p, s, k):
    g = random_regular_graph(n, 3, n)
    ga, be = qaoa_angles(p, n)
    t = network.qaoa_amplitude_network(n, g.edges, ga, be)
    full = contract.contract(t)
    pre, sl, res = own_schedule(t, s, k)
    tot, parts = contract.contract_sliced(t, pre, sl, res, return_parts=True)
    assert len(parts) == 2 ** k
    assert abs(tot - full) < 1e-12
    # k vs k+1 slicing agree
    pre2, sl2, res2 = own_schedule(t, s, k + 1)
    assert abs(contract.contract_sliced(t, pre2, sl2, res2) - full) < 1e-12


def test_order_independence_and_brute_force():
    n, p = 8, 1
    g = random_regular_graph(n, 3, 4)
    ga, be = qaoa_angles(p, 4)
    t = network.qaoa_amplitude_network(n, g.edges, ga, be)
    labs = network.live_labels(t)
    rng = np.random.default_rng(1)
    ref = contract.brute_force(t)
    for _ in range(4):
        order = list(rng.permutation(labs))
        assert abs(contract.bucket_eliminate(t, order) - ref) < 1e-13
    assert abs(contract.contract(t) - ref) < 1e-13
    # cone network too
    tc = network.zz_cone_network(n, g.edges, ga, be, *g.edges[0])
    assert abs(contract.contract(tc) - contract.brute_force(tc)) < 1e-13


def test_greedy_examples():
    # star K_{1,3} leaves-first width 1; K5 width 4; path width 1
    one = np.ones(2, dtype=np.complex128)
    star = [(np.ones((2, 2)), (0, c)) for c in (1, 2, 3)]
    assert contract.width_of_order(star, [1, 2, 3, 0]) == [1, 1, 1, 0]
    assert contract.width_of_order(star, [0, 1, 2, 3]) == [3, 2, 1, 0]
    k5 = [(np.ones((2, 2)), (a, b)) for a in range(5) for b in range(a + 1, 5)]
    _, d = contract.greedy_min_degree(k5)
    assert max(d) == 4
    path = [(np.ones((2, 2)), (a, a + 1)) for a in range(3)] + [(one, (0,))]
    _, d = contract.greedy_min_degree(path)
    assert max(d) == 1


@pytest.mark.parametrize("n,p,seed,maxw", [(14, 2, 3, 4), (16, 3, 1, 6)])
def test_subsliced_contraction_vs_statevector(n, p, seed, maxw):
    """Sub-slicing (Eq. 1 applied once more): the chosen extra labels bring
    the width down to max_width, and the pairwise sum over the 2^m sub-slices -- serial and over a
    process pool -- equals the 2^N state-vector amplitude (independent of the oracle's network)."""
    g = random_regular_graph(n, 3, seed)
    ga, be = qaoa_angles(p, seed)
    t = network.qaoa_amplitude_network(n, g.edges, ga, be)
    order, degs = contract.greedy_min_degree(t)
    extra = contract.subslice_labels(t, order, maxw)
    assert len(extra) >= 2 and max(degs) > maxw
    rest = [l for l in order if l not in set(extra)]
    assert max(contract.width_of_order(network.fix_indices(t, {l: 0 for l in extra}), rest)) <= maxw
    ref = sv.amplitude(sv.qaoa_state(n, g.edges, ga, be))
    serial = contract.contract_subsliced(t, order, extra, workers=1)
    pooled = contract.contract_subsliced(t, order, extra, workers=3)
    assert abs(serial - ref) < 1e-12 * max(1.0, abs(ref)) + 1e-14
    assert pooled == serial        # same sums in the same fixed tree: bit-identical


def test_slice_values_pool_matches_contract_sliced():
    """slice_values (prefix once, per-slice sub-slicing, process pool) gives the same per-slice
    values as the plain contract_sliced, and their pairwise sum is the state-vector amplitude."""
    n, p = 16, 2
    g = random_regular_graph(n, 3, 5)
    ga, be = qaoa_angles(p, 5)
    t = network.qaoa_amplitude_network(n, g.edges, ga, be)
    order, _ = contract.greedy_min_degree(t)
    pre, sl, res = order[:6], sorted(order[6:9]), order[9:]
    tot, parts = contract.contract_sliced(t, pre, sl, res, return_parts=True)
    vals, extra = contract.slice_values(t, pre, sl, res, range(8), max_width=3, workers=4)
    assert len(extra) >= 1
    for a, b in zip(vals, parts):
        assert abs(a - b) < 1e-13
    assert abs(contract.pairwise_sum(vals) - sv.amplitude(sv.qaoa_state(n, g.edges, ga, be))) < 1e-12
