"""GPU parity: the CUDA path (through the C-ABI) vs the oracle on the same seeded inputs.

Tolerances (BASELINE.json north_star): relative error <= 1e-10 for complex128 and <= 1e-4 for
complex64, relative to |oracle value| (amplitudes) or absolute on <Z_u Z_v> in [-1, 1].
"""
import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # the -m gpu suite runs on a B200 only
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2012_02430_b200 as T  # noqa: E402
from paper_2012_02430_b200 import _binding as B  # noqa: E402
from paper_2012_02430_b200.scheduler import run_sliced  # noqa: E402
from oracle import closed_forms as cf  # noqa: E402
from oracle import contract, energy, network  # noqa: E402
from oracle import statevector as sv  # noqa: E402
from tn_inputs import qaoa_angles, random_regular_graph  # noqa: E402

TOL = {T.TN_C64: 1e-4, T.TN_C128: 1e-10}
DT = {T.TN_C64: torch.complex64, T.TN_C128: torch.complex128}


def rel(a, b):
    return abs(a - b) / max(abs(b), 1e-300)


# ------------------------------------------------------------------ one bucket step (tn_eliminate)
def _random_step(rng, out_rank, n_in):
    masks, pvs, shapes = [], [], []
    for t in range(n_in):
        m = 0
        for b in range(out_rank):
            if rng.random() < 0.6:
                m |= 1 << b
        if t == 0 and out_rank > 0:
            m = (1 << out_rank) - 1          # one input holds every output bit (reduce-like)
        r_in = bin(m).count("1") + 1
        masks.append(m)
        pvs.append(int(rng.integers(0, r_in)))
        shapes.append(r_in)
    return masks, pvs, shapes


def _oracle_step(arrays, masks, pvs, out_rank):
    # labels: output bit b -> label b ; summed index -> label 100.  Input axes are most
    # significant first: input bit position q -> axis (rank-1-q).
    ts = []
    for a, m, pv in zip(arrays, masks, pvs):
        bits = [b for b in range(out_rank) if (m >> b) & 1]   # input positions 0.. (skipping pv)
        pos_labels = []
        it = iter(bits)
        for q in range(len(bits) + 1):
            pos_labels.append(100 if q == pv else next(it))
        labs = tuple(reversed(pos_labels))                      # axis 0 = most significant
        ts.append((a.reshape((2,) * len(labs)) if labs else a, labs))
    arr, labs = contract._einsum_bucket(ts, 100)
    # oracle output axes are ascending labels = ascending output bit; flatten most-significant first
    want = tuple(reversed(range(out_rank)))
    # output bits held by no input: the result is constant along them (broadcast)
    for l in want:
        if l not in labs:
            arr = np.stack([arr, arr], axis=-1)
            labs = tuple(labs) + (l,)
    if labs:
        arr = np.transpose(arr, [labs.index(l) for l in want])
    return arr.reshape(-1)


@pytest.mark.parametrize("dtype", [T.TN_C64, T.TN_C128])
@pytest.mark.parametrize("out_rank,n_in", [(0, 1), (0, 3), (1, 2), (2, 3), (5, 1), (9, 2), (12, 4),
                                           (13, 3), (14, 8), (17, 2), (18, 5), (21, 3)])
def test_eliminate_vs_oracle(dtype, out_rank, n_in):
    rng = np.random.default_rng(out_rank * 31 + n_in * 7 + dtype)
    masks, pvs, shapes = _random_step(rng, out_rank, n_in)
    arrays = [rng.uniform(-1, 1, 2 ** r) + 1j * rng.uniform(-1, 1, 2 ** r) for r in shapes]
    dev = [torch.tensor(a, dtype=DT[dtype], device="cuda") for a in arrays]
    out = torch.empty(2 ** out_rank, dtype=DT[dtype], device="cuda")
    B.tn_eliminate(dtype, [d.data_ptr() for d in dev], masks, pvs, out.data_ptr(), out_rank,
                   torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    got = out.cpu().numpy().astype(np.complex128)
    ref = _oracle_step(arrays, masks, pvs, out_rank)
    scale = np.max(np.abs(ref)) + 1e-30
    assert np.max(np.abs(got - ref)) / scale < TOL[dtype] * 0.1


@pytest.mark.parametrize("dtype", [T.TN_C64, T.TN_C128])
@pytest.mark.parametrize("out_rank,kinds", [(13, "FS"), (14, "FSC"), (15, "SSC"), (16, "FFS"), (17, "SC"),
                                            (18, "FSSC"), (20, "FC"), (21, "SSSC"), (22, "FFSC"), (19, "CS")])
def test_eliminate_specialised_vs_oracle(dtype, out_rank, kinds):
    # plan-like steps (summed index on top of every input): F = holds every low tile bit,
    # S = some low bits (staged in shared memory), C = no low bit (per-tile constant)
    rng = np.random.default_rng(out_rank * 13 + len(kinds) + dtype)
    tb = 12 if dtype == T.TN_C64 else 11
    masks, pvs, shapes = [], [], []
    for k in kinds:
        low = (1 << tb) - 1 if k == "F" else (0 if k == "C" else int(rng.integers(1, (1 << tb) - 1)))
        high = 0
        for b in range(tb, out_rank):
            if rng.random() < 0.5:
                high |= 1 << b
        m = low | high
        masks.append(m)
        pvs.append(bin(m).count("1"))
        shapes.append(bin(m).count("1") + 1)
    arrays = [rng.uniform(-1, 1, 2 ** r) + 1j * rng.uniform(-1, 1, 2 ** r) for r in shapes]
    dev = [torch.tensor(a, dtype=DT[dtype], device="cuda") for a in arrays]
    out = torch.empty(2 ** out_rank, dtype=DT[dtype], device="cuda")
    B.tn_eliminate(dtype, [d.data_ptr() for d in dev], masks, pvs, out.data_ptr(), out_rank,
                   torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    got = out.cpu().numpy().astype(np.complex128)
    ref = _oracle_step(arrays, masks, pvs, out_rank)
    assert np.max(np.abs(got - ref)) / (np.max(np.abs(ref)) + 1e-30) < TOL[dtype] * 0.1


# ------------------------------------------------------------------ fused groups (tn_eliminate_group)
def _oracle_group(arrays, out_masks, x_masks, M, out_rank):
    """The oracle's bucket elimination of x_0 .. x_{M-1} (labels 100 + i) over the caller tensors;
    output bit b = label b.  Input positions: output bits low (ascending), held x_i on top with
    x_0 the most significant; numpy axis 0 = the most significant position."""
    ts = []
    for a, m, xm in zip(arrays, out_masks, x_masks):
        pos_labels = [b for b in range(out_rank) if (m >> b) & 1]
        pos_labels += [100 + i for i in reversed(range(M)) if (xm >> i) & 1]
        labs = tuple(reversed(pos_labels))
        ts.append((a.reshape((2,) * len(labs)), labs))
    rest, scalar = contract.partial_eliminate(ts, [100 + i for i in range(M)])
    arr, labs = rest[0]
    for a2, l2 in rest[1:]:          # inputs holding no summed index pass through: multiply in
        arr, labs = contract._einsum_bucket([(arr, labs), (a2, l2), (np.full(2, 0.5), (999,))], 999)
    arr = arr * scalar
    want = tuple(reversed(range(out_rank)))
    for l in want:
        if l not in labs:
            arr = np.stack([arr, arr], axis=-1)
            labs = tuple(labs) + (l,)
    arr = np.transpose(arr, [labs.index(l) for l in want])
    return arr.reshape(-1)


def _gemm_group(rng, out_rank, M, cls, xa=None, xb=None, cmask_hi=0, weights=True):
    """A merge group as in a plan: A and B hold the output bits of classes a/c and b/c (cls[b] for
    bit b), summed indices xa / xb (default: all); rank-1 weights on each x_i; optionally a constant
    input holding high output bits `cmask_hi` and x_0."""
    full_x = (1 << M) - 1
    mA = sum(1 << b for b in range(out_rank) if cls[b] in "ac")
    mB = sum(1 << b for b in range(out_rank) if cls[b] in "bc")
    masks = [mA, mB]
    xms = [full_x if xa is None else xa, full_x if xb is None else xb]
    if weights:
        for i in range(M):
            masks.append(0)
            xms.append(1 << i)
    if cmask_hi:
        masks.append(cmask_hi)
        xms.append(1)
    shapes = [bin(m).count("1") + bin(x).count("1") for m, x in zip(masks, xms)]
    return masks, xms, shapes


def _cls(rng, out_rank, low="abccc"):
    c = list(low[::-1]) if low else []
    while len(c) < out_rank:
        c.append("abcc"[int(rng.integers(0, 4))])
    if len(low) < 9:   # at least two a and two b bits above the lanes
        for k, want in ((5, "a"), (6, "a"), (7, "b"), (8, "b")):
            c[k] = want
    return c


GROUP_CASES = [
    # (out_rank, M, low-bit classes (bit 4..0), xa, xb, cmask_hi)
    (12, 1, "abccc", None, None, 0),
    (14, 2, "ccbca", None, None, 0),
    (16, 3, "abccc", None, None, 0),
    (17, 3, "bbaac", 0b011, None, 0),       # A lacks x_2: chunk rows shared
    (18, 4, "ccccb", None, 0b1010, 0),      # B lacks x_0, x_2
    (17, 2, "aabbcbbbbb", None, None, 0),   # A's lowest bit (5, class c) outside the tile -> 8-byte copies
    (15, 5, "cacab", None, None, 0),
    (19, 3, "abccc", None, None, 1 << 18),  # tile-dependent constant factor
    (20, 2, "caaab", None, None, 0),
]


@pytest.mark.parametrize("kernel", [1, 2, 3, 0])
@pytest.mark.parametrize("case", range(len(GROUP_CASES)))
def test_group_kernels_vs_oracle(case, kernel):
    out_rank, M, low, xa, xb, chi = GROUP_CASES[case]
    rng = np.random.default_rng(1000 + case)
    cls = _cls(rng, out_rank, low)
    masks, xms, shapes = _gemm_group(rng, out_rank, M, cls, xa, xb, chi)
    for dtype in (T.TN_C64, T.TN_C128):
        if kernel == 1 and dtype == T.TN_C128:
            continue
        arrays = [rng.uniform(-1, 1, 2 ** r) + 1j * rng.uniform(-1, 1, 2 ** r) for r in shapes]
        dev = [torch.tensor(a, dtype=DT[dtype], device="cuda") for a in arrays]
        out = torch.full((2 ** out_rank,), float("nan"), dtype=DT[dtype], device="cuda")
        try:
            B.tn_eliminate_group(dtype, M, [d.data_ptr() for d in dev], masks, xms, out.data_ptr(), out_rank,
                                 kernel, torch.cuda.current_stream().cuda_stream)
        except T.TnError:
            # k_gemm stages all 2^M rows of a tile's chunks in shared memory: M >= 4 shapes whose
            # chunks exceed the budget fall back to k_pair / k_group_t (kernel 0 never fails)
            assert kernel in (2, 3) or (kernel == 1 and M >= 4), "k_gemm must take this GEMM-shaped group"
            continue
        torch.cuda.synchronize()
        got = out.cpu().numpy().astype(np.complex128)
        ref = _oracle_group(arrays, masks, xms, M, out_rank)
        assert np.all(np.isfinite(got)), "output element not written"
        assert np.max(np.abs(got - ref)) / (np.max(np.abs(ref)) + 1e-30) < TOL[dtype] * 0.1


def test_group_kernels_each_take_some_cases():
    """Each explicitly named group kernel (1 k_gemm, 2 k_pair, 3 k_group_t) accepts -- and then
    matches the oracle on -- at least one GROUP_CASES shape: the parametrised test above skips the
    shapes a kernel declines, so this guards against a kernel that declines everything."""
    for kernel, want in ((1, 5), (2, 1), (3, 1)):
        took = 0
        for case, (out_rank, M, low, xa, xb, chi) in enumerate(GROUP_CASES):
            rng = np.random.default_rng(1000 + case)
            cls = _cls(rng, out_rank, low)
            masks, xms, shapes = _gemm_group(rng, out_rank, M, cls, xa, xb, chi)
            arrays = [rng.uniform(-1, 1, 2 ** r) + 1j * rng.uniform(-1, 1, 2 ** r) for r in shapes]
            dev = [torch.tensor(a, dtype=torch.complex64, device="cuda") for a in arrays]
            out = torch.full((2 ** out_rank,), float("nan"), dtype=torch.complex64, device="cuda")
            try:
                B.tn_eliminate_group(T.TN_C64, M, [d.data_ptr() for d in dev], masks, xms, out.data_ptr(),
                                     out_rank, kernel, torch.cuda.current_stream().cuda_stream)
            except T.TnError:
                continue
            torch.cuda.synchronize()
            got = out.cpu().numpy().astype(np.complex128)
            ref = _oracle_group(arrays, masks, xms, M, out_rank)
            assert np.max(np.abs(got - ref)) / (np.max(np.abs(ref)) + 1e-30) < TOL[T.TN_C64] * 0.1
            took += 1
        assert took >= want, f"kernel {kernel} took only {took} of {len(GROUP_CASES)} shapes"


TC_CASES = [
    # (out_rank, M, classes from bit 0 up (a: A only, b: B only, c: both), xa, xb, cmask_hi)
    (18, 3, "abccabcaabcbabaaac", None, None, 0),          # the bit pattern of C5a's top group
    (17, 3, "bacbbcabbabbbcbbb", None, None, 0),           # B holds the most exclusive bits (swap)
    (16, 1, "aaaacaaabbbbbccc", None, None, 0),            # K' = 4 zero-padded to one K-chunk
    (17, 2, "ccaaaaaaabbbbbcbb", 0b01, None, 0),           # A lacks x_1; low diag bits
    (18, 5, "aabbcaaaaabbbcccab", None, 0b10110, 0),       # K = 32, B lacks x_0 and x_3
    (19, 3, "abcabcaaaabbbcccaab", None, None, 1 << 18),   # tile-dependent constant factor
    (20, 4, "acbcacbcaaaaabbbbccc", None, None, 0),
]


@pytest.mark.parametrize("case", range(len(TC_CASES)))
def test_gemm_tc_vs_oracle(case):
    """k_gemm_tc (tcgen05 kind::tf32, 3xTF32 split) on GEMM-shaped merge groups vs the oracle at
    the complex64 tolerance; several tiles per CTA, ragged diag / col splits."""
    out_rank, M, cls_s, xa, xb, chi = TC_CASES[case]
    rng = np.random.default_rng(5000 + case)
    cls = list(cls_s)
    assert len(cls) == out_rank
    masks, xms, shapes = _gemm_group(rng, out_rank, M, cls, xa, xb, chi)
    arrays = [rng.uniform(-1, 1, 2 ** r) + 1j * rng.uniform(-1, 1, 2 ** r) for r in shapes]
    dev = [torch.tensor(a, dtype=torch.complex64, device="cuda") for a in arrays]
    out = torch.full((2 ** out_rank,), float("nan"), dtype=torch.complex64, device="cuda")
    B.tn_eliminate_group(T.TN_C64, M, [d.data_ptr() for d in dev], masks, xms, out.data_ptr(), out_rank,
                         4, torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    got = out.cpu().numpy().astype(np.complex128)
    ref = _oracle_group(arrays, masks, xms, M, out_rank)
    assert np.all(np.isfinite(got)), "output element not written"
    err = np.max(np.abs(got - ref)) / (np.max(np.abs(ref)) + 1e-30)
    assert err < TOL[T.TN_C64] * 0.1, err


HM_CASES = [
    # (out_rank, M, classes from bit 0 up (a: A only, b: B only, c: both), xa, xb, expected (FA, FB))
    (21, 3, "bcbaacaacacababcaabca", None, None),   # the low bits of C5a's top standalone group
    (20, 3, "abccabcaabcbabaaacaa", None, None),    # the low bits of C5a's producer group (FB = 3)
    (17, 3, "bacbbcabbabbbcbbb", None, None),       # B holds the most exclusive bits (roles swap)
    (19, 2, "ccaaaaaaabbbbbcbbac", 0b01, None),     # A lacks x_1: chunk rows shared; K = 4 (one k-step)
    (18, 5, "aabbcaaaaabbbcccab", None, 0b10110),   # K = 32, B lacks x_0 and x_3
    (20, 4, "acbcacbcaaaaabbbbccc", None, None),
    (18, 3, "aaaaaaaaabbccccaca", None, None),      # two B-only bits: FB = 0, FA = 3
    (22, 3, "cbcbaacaaacabcaabbacac", None, None),  # several tiles per CTA
]


@pytest.mark.parametrize("case", range(len(HM_CASES)))
def test_gemm_hm_vs_oracle(case):
    """k_gemm_hm (mma.sync m16n8k8 tf32, 3xTF32 split) on GEMM-shaped merge groups vs the oracle at
    the complex64 tolerance (the tile covers the lanes' a/b bits, rows shared across x, K = 4 .. 32,
    swapped operand roles, every fragment-block split)."""
    out_rank, M, cls_s, xa, xb = HM_CASES[case]
    rng = np.random.default_rng(7000 + case)
    cls = list(cls_s)
    assert len(cls) == out_rank
    masks, xms, shapes = _gemm_group(rng, out_rank, M, cls, xa, xb)
    arrays = [rng.uniform(-1, 1, 2 ** r) + 1j * rng.uniform(-1, 1, 2 ** r) for r in shapes]
    dev = [torch.tensor(a, dtype=torch.complex64, device="cuda") for a in arrays]
    out = torch.full((2 ** out_rank,), float("nan"), dtype=torch.complex64, device="cuda")
    B.tn_eliminate_group(T.TN_C64, M, [d.data_ptr() for d in dev], masks, xms, out.data_ptr(), out_rank,
                         5, torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    got = out.cpu().numpy().astype(np.complex128)
    ref = _oracle_group(arrays, masks, xms, M, out_rank)
    assert np.all(np.isfinite(got)), "output element not written"
    err = np.max(np.abs(got - ref)) / (np.max(np.abs(ref)) + 1e-30)
    assert err < TOL[T.TN_C64] * 0.1, err


HM64_CASES = HM_CASES + [
    (18, 1, "abcaacaabbcacbaaca", None, None),      # M = 1: one k-step (K = 2 complex)
    (19, 2, "bacbaacaabcacbcabaa", None, None),     # output bit 0 held by Q only
]


@pytest.mark.parametrize("case", range(len(HM64_CASES)))
def test_gemm_hm64_vs_oracle(case):
    """k_gemm_hm64 (complex128 merge groups on mma.sync m8n8k4 f64: one FP64 product, no split) vs the
    oracle at the complex128 tolerance; the HM shapes plus M = 1 and a Q-held output bit 0."""
    out_rank, M, cls_s, xa, xb = HM64_CASES[case]
    rng = np.random.default_rng(7200 + case)
    cls = list(cls_s)
    assert len(cls) == out_rank
    masks, xms, shapes = _gemm_group(rng, out_rank, M, cls, xa, xb)
    arrays = [rng.uniform(-1, 1, 2 ** r) + 1j * rng.uniform(-1, 1, 2 ** r) for r in shapes]
    dev = [torch.tensor(a, dtype=torch.complex128, device="cuda") for a in arrays]
    out = torch.full((2 ** out_rank,), float("nan"), dtype=torch.complex128, device="cuda")
    B.tn_eliminate_group(T.TN_C128, M, [d.data_ptr() for d in dev], masks, xms, out.data_ptr(), out_rank,
                         5, torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    got = out.cpu().numpy()
    ref = _oracle_group(arrays, masks, xms, M, out_rank)
    assert np.all(np.isfinite(got)), "output element not written"
    err = np.max(np.abs(got - ref)) / (np.max(np.abs(ref)) + 1e-30)
    assert err < TOL[T.TN_C128] * 0.1, err


def test_gemm_hm_declines_tile_dependent_constants():
    """A constant factor holding an output bit would force the Q fragments to be rebuilt every
    tile: k_gemm_hm declines (the library's choice then takes k_gemm)."""
    rng = np.random.default_rng(7100)
    out_rank, M = 19, 3
    cls = list("abcabcaaaabbbcccaab")
    masks, xms, shapes = _gemm_group(rng, out_rank, M, cls, None, None, 1 << 18)
    dev = [torch.zeros(2 ** r, dtype=torch.complex64, device="cuda") for r in shapes]
    out = torch.empty(2 ** out_rank, dtype=torch.complex64, device="cuda")
    with pytest.raises(T.TnError):
        B.tn_eliminate_group(T.TN_C64, M, [d.data_ptr() for d in dev], masks, xms, out.data_ptr(), out_rank,
                             5, torch.cuda.current_stream().cuda_stream)


# ------------------------------------------------------------------ amplitudes, small/medium
@pytest.mark.parametrize("dtype", [T.TN_C64, T.TN_C128])
@pytest.mark.parametrize("n,p,k,orderer", [(12, 1, 0, "min-fill"), (14, 2, 0, "min-degree"),
                                           (16, 3, 2, "min-fill"), (20, 2, 3, "min-degree"),
                                           (24, 1, 4, "min-fill"), (30, 2, 2, "min-fill")])
def test_amplitude_vs_oracle(dtype, n, p, k, orderer):
    g = random_regular_graph(n, 3, n + p)
    ga, be = qaoa_angles(p, n)
    plan = T.build_plan(g, p, "amplitude", orderer, n_sliced=k, small_log2=4)
    got = plan.contract(ga, be, dtype=dtype)
    ref = contract.contract(network.qaoa_amplitude_network(n, g.edges, ga, be))
    assert rel(got, ref) < TOL[dtype]
    if n <= 16:
        assert rel(got, sv.amplitude(sv.qaoa_state(n, g.edges, ga, be))) < TOL[dtype]


@pytest.mark.parametrize("dtype", [T.TN_C64, T.TN_C128])
def test_interpreter_only_and_big_only_agree(dtype):
    n, p = 22, 2
    g = random_regular_graph(n, 3, 5)
    ga, be = qaoa_angles(p, 5)
    ref = contract.contract(network.qaoa_amplitude_network(n, g.edges, ga, be))
    for small in (0, 3, 30):   # 0: every step standalone; 30: everything in the interpreter
        plan = T.build_plan(g, p, "amplitude", "min-fill", n_sliced=2, small_log2=small)
        assert rel(plan.contract(ga, be, dtype=dtype), ref) < TOL[dtype]


@pytest.mark.parametrize("dtype", [T.TN_C64, T.TN_C128])
@pytest.mark.parametrize("n,p,k,orderer", [(50, 2, 2, "min-fill"), (36, 3, 3, "rgreedy-fill"),
                                           (90, 1, 2, "rgreedy-fill"), (70, 2, 3, "rgreedy-fill")])
def test_fused_groups_vs_oracle(dtype, n, p, k, orderer):
    # every step standalone (small_log2 = 0): reduce chains (k_chain), merge groups (k_group_t,
    # k_pair) and single steps all run at moderate widths, checked against the oracle
    g = random_regular_graph(n, 3, 7 * n + p)
    ga, be = qaoa_angles(p, n + 1)
    plan = T.build_plan(g, p, "amplitude", orderer, n_sliced=k, small_log2=0, rg_q=4, rg_tau=0.4)
    kinds = {s["standalone"] for s in plan.steps()}
    assert 3 in kinds or 2 in kinds
    pre, sl, res, _ = plan.schedule()
    ref = contract.contract_sliced(network.qaoa_amplitude_network(n, g.edges, ga, be), pre, sl, res)
    assert rel(plan.contract(ga, be, dtype=dtype), ref) < TOL[dtype]


FUSED_PAIR = {"k_gemm_fc", "k_fc_tc", "k_fc_hm"}   # the kernels of an OP_GROUP_FEED pair (SIMT / tcgen05 / mma.sync)
FC_ENV = {"tc": {"TNB_FC_TC": "1"}, "simt": {"TNB_FC_TC": "0", "TNB_FC_HM": "0", "TNB_FC_SPLIT": "0"},
          "hm": {"TNB_FC_TC": "0", "TNB_FC_HM": "1"},
          "split": {"TNB_FC_TC": "0", "TNB_FC_HM": "0", "TNB_FC_SPLIT": "1"}}


@pytest.mark.parametrize("kernel", ["tc", "simt", "hm"])
@pytest.mark.parametrize("n,p,k,fused", [(36, 3, 3, True), (70, 2, 3, True), (44, 3, 3, False),
                                          (50, 2, 2, False)])
def test_feed_pairs_run_fused_and_match_oracle(n, p, k, fused, kernel, monkeypatch):
    """OP_GROUP_FEED: a GEMM-shaped group whose output is a full input of the next group runs as ONE
    launch (the intermediate is never written) -- k_fc_tc (tcgen05, TNB_FC_TC=1), k_fc_hm (mma.sync,
    TNB_FC_HM=1) or k_gemm_fc (FP32 SIMT, the default) when the shape qualifies; the contraction still matches the oracle
    (c64 tolerance), and the fused launch is the one that ran (profile records).  Pairs whose
    consumer output has fewer bits than a k_gemm_fc tile (fused=False) run as the two groups."""
    for key, val in FC_ENV[kernel].items():
        monkeypatch.setenv(key, val)
    g = random_regular_graph(n, 3, 7 * n + p)
    ga, be = qaoa_angles(p, n + 1)
    plan = T.build_plan(g, p, "amplitude", "rgreedy-fill", n_sliced=k, small_log2=0, rg_q=4, rg_tau=0.4)
    plan.profile(True)
    got = plan.contract(ga, be, dtype=T.TN_C64)
    recs = plan.profile_records()
    plan.profile(False)
    ran = {r["kernel"] for r in recs}
    assert bool(ran & FUSED_PAIR) == fused, sorted(ran)
    if kernel != "tc":
        assert "k_fc_tc" not in ran
    if kernel == "simt":
        assert "k_fc_hm" not in ran
    pre, sl, res, _ = plan.schedule()
    ref = contract.contract_sliced(network.qaoa_amplitude_network(n, g.edges, ga, be), pre, sl, res)
    assert rel(got, ref) < TOL[T.TN_C64]


@pytest.mark.parametrize("fast", ["tc", "hm", "split"])
def test_fc_fast_kernels_run_on_c5a_and_match_simt_per_slice(fast, monkeypatch):
    """C5a's producer -> consumer pair (R = 26 -> 21, the bench's largest launch) runs on k_fc_tc
    (tcgen05) / k_fc_hm (mma.sync) / k_gemm_fc with consumer blocks split between neighbouring CTAs
    (TNB_FC_SPLIT=1: 512 blocks on 296 CTAs, so the split path really runs); every per-slice partial
    agrees with the default FP32 SIMT k_gemm_fc within the c64 tolerance."""
    plan, g, ga, be, meta = _bench_plan()
    n = plan.n_slices
    parts = {}
    for kern in (fast, "simt"):
        for key, val in FC_ENV[kern].items():
            monkeypatch.setenv(key, val)
        part = torch.zeros(2 * n, dtype=torch.float64, device="cuda")
        plan.profile(True)
        plan.contract_sliced(ga, be, 0, n, part, dtype=T.TN_C64)
        torch.cuda.synchronize()
        ran = {r["kernel"] for r in plan.profile_records()}
        plan.profile(False)
        plan.profile_read()
        assert {"tc": "k_fc_tc", "hm": "k_fc_hm", "simt": "k_gemm_fc", "split": "k_gemm_fc"}[kern] in ran, sorted(ran)
        h = part.cpu().tolist()
        parts[kern] = [complex(h[2 * j], h[2 * j + 1]) for j in range(n)]
    scale = max(abs(v) for v in parts["simt"])
    for j in range(n):
        assert abs(parts[fast][j] - parts["simt"][j]) / scale < 2e-5, (j, parts[fast][j], parts["simt"][j])



def test_slice_partials_vs_oracle_per_slice():
    """Every per-slice partial of a sliced plan vs the oracle's slice (plan schedule as data)."""
    n, p, k = 40, 1, 3
    g = random_regular_graph(n, 3, 40)
    ga, be = qaoa_angles(p, 40)
    plan = T.build_plan(g, p, "amplitude", "min-fill", n_sliced=k)
    pre, sl, res, _ = plan.schedule()
    tens = network.qaoa_amplitude_network(n, g.edges, ga, be)
    tot, parts = contract.contract_sliced(tens, pre, sl, res, return_parts=True)
    partials = torch.zeros(2 * plan.n_slices, dtype=torch.float64, device="cuda")
    plan.contract_sliced(ga, be, 0, plan.n_slices, partials, dtype=T.TN_C128)
    torch.cuda.synchronize()
    h = partials.cpu().numpy()
    for j in range(plan.n_slices):
        assert abs(complex(h[2 * j], h[2 * j + 1]) - parts[j]) <= 1e-10 * abs(tot)
    assert rel(plan.sum_partials(h.tolist()), tot) < 1e-10


def test_partition_is_bit_identical():
    n, p = 30, 1
    g = random_regular_graph(n, 3, 9)
    ga, be = qaoa_angles(p, 9)
    plan = T.build_plan(g, p, "amplitude", "min-fill", n_sliced=4)
    full = torch.zeros(2 * plan.n_slices, dtype=torch.float64, device="cuda")
    plan.contract_sliced(ga, be, 0, plan.n_slices, full, dtype=T.TN_C64)
    parts = torch.zeros_like(full)
    cuts = [0, 3, 8, 9, 16]
    for a, b in zip(cuts[:-1], cuts[1:]):
        plan.contract_sliced(ga, be, a, b, parts, dtype=T.TN_C64)
    torch.cuda.synchronize()
    assert torch.equal(full, parts)
    s1 = plan.sum_partials(full.cpu().tolist())
    s2, _ = run_sliced(plan, ga, be, dtype=T.TN_C64)
    assert s1 == s2


# ------------------------------------------------------------------ energy (C1, C3)
@pytest.mark.parametrize("dtype", [T.TN_C128, T.TN_C64])
def test_energy_c1_vs_statevector(dtype):
    n, p = 16, 1
    g = random_regular_graph(n, 3, 0)
    ga, be = qaoa_angles(p, 0)
    plan = T.build_plan(g, p, "energy", "min-fill")
    zz, im, E = plan.energy(ga, be, dtype=dtype)
    psi = sv.qaoa_state(n, g.edges, ga, be)
    for (u, v), z in zip(g.edges, zz):
        assert abs(z - sv.zz_expectation(psi, u, v)) < TOL[dtype]
        assert abs(z - cf.wang_p1_zz(g.edges, u, v, ga[0], be[0])) < TOL[dtype]
    assert abs(E - sv.maxcut_energy(psi, g.edges)) < TOL[dtype] * len(g.edges)
    assert im < TOL[dtype]


@pytest.mark.parametrize("dtype", [T.TN_C128, T.TN_C64])
@pytest.mark.parametrize("n,p", [(16, 2), (16, 3), (100, 3)])
def test_energy_vs_oracle(dtype, n, p):
    g = random_regular_graph(n, 3, 0)
    ga, be = qaoa_angles(p, 0)
    plan = T.build_plan(g, p, "energy", "min-fill")
    zz, im, E = plan.energy(ga, be, dtype=dtype)
    Eref, zref = energy.maxcut_energy(n, g.edges, ga, be)
    assert max(abs(a - b.real) for a, b in zip(zz, zref)) < TOL[dtype]
    assert abs(E - Eref) < TOL[dtype] * len(g.edges)
    assert 0.0 <= E <= len(g.edges)


@pytest.mark.parametrize("dtype", [T.TN_C64, T.TN_C128])
@pytest.mark.parametrize("n,p,k,r", [(40, 3, 6, 2), (44, 3, 8, 4), (60, 2, 6, 3)])
def test_multi_round_slicing_vs_oracle(dtype, n, p, k, r):
    """Step-dependent slicing in rounds of r < n indices (reading A18: later
    rounds' prefixes run inside every slice) -- the plans C4b / C5b use -- vs the oracle with the
    plan's schedule as data (Eq. 1)."""
    g = random_regular_graph(n, 3, 11 * n + p)
    ga, be = qaoa_angles(p, n)
    plan = T.build_plan(g, p, "amplitude", "rgreedy-fill", n_sliced=k, r=r, rg_q=8, rg_tau=0.3)
    assert plan.n_slices == 2 ** k
    pre, sl, res, _ = plan.schedule()
    ref = contract.contract_sliced(network.qaoa_amplitude_network(n, g.edges, ga, be), pre, sl, res)
    assert rel(plan.contract(ga, be, dtype=dtype), ref) < TOL[dtype]


# ------------------------------------------------------------------ full-scale closed forms
def _bench_plan():
    import bench
    return bench.build_workload_plan("C5a")


@pytest.mark.parametrize("which", ["gamma0", "beta0", "gammapi"])
def test_c5a_full_scale_closed_forms(which):
    """C5a (N=210, p=1) at the bench's plan and dtype vs closed forms that hold at any N."""
    plan, g, ga, be, meta = _bench_plan()
    n = g.n
    if which == "gamma0":
        ga, ref = [0.0], cf.amp_gamma0(n, be)
    elif which == "beta0":
        be, ref = [0.0], cf.amp_beta0(n)
    else:
        ga, ref = [math.pi], cf.amp_gamma_pi(n, be)
    got, _ = run_sliced(plan, ga, be, dtype=T.TN_C64)
    assert rel(got, ref) < 1e-4


def test_c5a_full_scale_sampled_slice_vs_oracle():
    """C5a (N=210, p=1) at the bench's plan, dtype and launch configuration (every slice, the
    default workspace with its slice lanes, the producer -> consumer launches): slice 16 of the 32
    against the oracle's value of that slice (complex128, the plan's schedule as data)."""
    plan, g, ga, be, meta = _bench_plan()
    n = plan.n_slices
    ws = plan.workspace(T.TN_C64)
    part = torch.zeros(2 * n, dtype=torch.float64, device="cuda")
    plan.profile(True)
    B.tn_contract_sliced(plan.handle, T.TN_C64, ga, be, 0, n, ws.data_ptr(), ws.numel(),
                         torch.cuda.current_stream().cuda_stream, part.data_ptr())
    torch.cuda.synchronize()
    assert {r["kernel"] for r in plan.profile_records()} & FUSED_PAIR
    plan.profile(False)
    j = n // 2
    pre, sl, res, _ = plan.schedule()
    tens = network.qaoa_amplitude_network(g.n, g.edges, ga, be)
    _, parts = contract.contract_sliced(tens, pre, sl, res, slices=[j], return_parts=True)
    got = complex(*part[2 * j:2 * j + 2].tolist())
    assert rel(got, parts[0]) < TOL[T.TN_C64]


# ------------------------------------------------------------------ batching
@pytest.mark.parametrize("dtype", [T.TN_C64, T.TN_C128])
def test_batched_slices_match_sequential_and_oracle(dtype):
    n, p = 40, 2
    g = random_regular_graph(n, 3, 17)
    ga, be = qaoa_angles(p, 17)
    plan = T.build_plan(g, p, "amplitude", "min-fill", n_sliced=5, small_log2=30)
    assert plan.info["slices_batchable"] == 1 and plan.batch_windows(dtype) == plan.n_slices
    outs = []
    for batch in (1, 3, plan.n_slices):
        ws = plan.workspace(dtype, batch=batch)
        part = torch.zeros(2 * plan.n_slices, dtype=torch.float64, device="cuda")
        B.tn_contract_sliced(plan.handle, dtype, ga, be, 0, plan.n_slices, ws.data_ptr(), ws.numel(),
                             torch.cuda.current_stream().cuda_stream, part.data_ptr())
        torch.cuda.synchronize()
        outs.append(part.cpu())
    assert torch.equal(outs[0], outs[1]) and torch.equal(outs[0], outs[2])   # same arithmetic
    pre, sl, res, _ = plan.schedule()
    ref = contract.contract_sliced(network.qaoa_amplitude_network(n, g.edges, ga, be), pre, sl, res)
    assert rel(plan.sum_partials(outs[2].tolist()), ref) < TOL[dtype]


@pytest.mark.parametrize("dtype", [T.TN_C128, T.TN_C64])
def test_energy_batch_matches_single_and_oracle(dtype):
    n, p = 30, 2
    g = random_regular_graph(n, 3, 3)
    plan = T.build_plan(g, p, "energy", "min-fill")
    sets = [qaoa_angles(p, 100 + b) for b in range(5)]
    zzs, ims, ens = plan.energy_batch([s[0] for s in sets], [s[1] for s in sets], dtype=dtype)
    for b, (ga, be) in enumerate(sets):
        zz1, im1, e1 = plan.energy(ga, be, dtype=dtype)
        assert zz1 == zzs[b] and e1 == ens[b]                                   # same arithmetic
        Eref, _ = energy.maxcut_energy(n, g.edges, ga, be)
        assert abs(ens[b] - Eref) < TOL[dtype] * len(g.edges)


@pytest.mark.parametrize("dtype", [T.TN_C64, T.TN_C128])
def test_two_slice_lanes_match_one_lane_and_oracle(dtype):
    """Odd slices on the side stream in window 1 (workspace with two windows) give the same
    partials, bit for bit, as one lane (one window), and match the oracle."""
    n, p = 44, 2
    g = random_regular_graph(n, 3, 23)
    ga, be = qaoa_angles(p, 23)
    plan = T.build_plan(g, p, "amplitude", "min-fill", n_sliced=3, small_log2=6)
    assert plan.info["slices_batchable"] == 0
    outs = []
    for windows in (1, 2):
        ws = plan.workspace(dtype, batch=windows)
        part = torch.zeros(2 * plan.n_slices, dtype=torch.float64, device="cuda")
        B.tn_contract_sliced(plan.handle, dtype, ga, be, 0, plan.n_slices, ws.data_ptr(), ws.numel(),
                             torch.cuda.current_stream().cuda_stream, part.data_ptr())
        torch.cuda.synchronize()
        outs.append(part.cpu())
    assert torch.equal(outs[0], outs[1])
    pre, sl, res, _ = plan.schedule()
    ref = contract.contract_sliced(network.qaoa_amplitude_network(n, g.edges, ga, be), pre, sl, res)
    assert rel(plan.sum_partials(outs[1].tolist()), ref) < TOL[dtype]


def test_slice_lanes_with_fused_pairs_match_one_lane_and_oracle():
    """The producer -> consumer launch (k_gemm_fc) in slice lanes: 4 windows give the same partials,
    bit for bit, as one window, and match the oracle."""
    n, p, k = 36, 3, 3
    g = random_regular_graph(n, 3, 7 * n + p)
    ga, be = qaoa_angles(p, n + 1)
    plan = T.build_plan(g, p, "amplitude", "rgreedy-fill", n_sliced=k, small_log2=0, rg_q=4, rg_tau=0.4)
    outs = []
    for windows in (1, 4):
        ws = plan.workspace(T.TN_C64, batch=windows)
        part = torch.zeros(2 * plan.n_slices, dtype=torch.float64, device="cuda")
        plan.profile(True)
        B.tn_contract_sliced(plan.handle, T.TN_C64, ga, be, 0, plan.n_slices, ws.data_ptr(), ws.numel(),
                             torch.cuda.current_stream().cuda_stream, part.data_ptr())
        torch.cuda.synchronize()
        assert {r["kernel"] for r in plan.profile_records()} & FUSED_PAIR
        plan.profile(False)
        outs.append(part.cpu())
    assert torch.equal(outs[0], outs[1])
    pre, sl, res, _ = plan.schedule()
    ref = contract.contract_sliced(network.qaoa_amplitude_network(n, g.edges, ga, be), pre, sl, res)
    assert rel(plan.sum_partials(outs[1].tolist()), ref) < TOL[T.TN_C64]


# ------------------------------------------------------------------ amplitude batches
def _oracle_batch(n, edges, ga, be, opened, pre, sl, res):
    """Oracle batch with the plan's schedule as data: prefix once, Eq. (1) over the slices, the
    open indices left open; entries summed over slices in the fixed pairwise
    order."""
    p = len(ga)
    tens = network.qaoa_amplitude_network(n, edges, ga, be, open_qubits=opened)
    ol = network.open_labels(n, p, opened)
    rest, ps = contract.partial_eliminate(tens, pre)
    parts = []
    for j in range(1 << len(sl)):
        fixed = network.fix_indices(rest, contract.slice_assignment(sl, j))
        parts.append(ps * contract.contract_open(fixed, ol, order=res))
    return np.array([contract.pairwise_sum([v[x] for v in parts]) for x in range(1 << len(opened))])


@pytest.mark.parametrize("dtype", [T.TN_C64, T.TN_C128])
@pytest.mark.parametrize("n,p,k,opened,small", [(12, 2, 0, (0, 3, 7), 4), (16, 1, 2, (2, 9), 4),
                                                (30, 2, 3, (1, 4, 8, 17), 6), (40, 1, 2, (0, 39), 0),
                                                (24, 3, 2, (5,), 30)])
def test_amplitude_batch_vs_oracle(dtype, n, p, k, opened, small):
    """A batch of 2^a amplitudes (open output indices) vs the oracle; entry 0 vs the
    single-amplitude plan; the state vector where N <= 16."""
    g = random_regular_graph(n, 3, 3 * n + p)
    ga, be = qaoa_angles(p, n + 5)
    plan = T.build_plan(g, p, "amplitude", "min-fill", n_sliced=k, small_log2=small, open_qubits=opened)
    got = np.array(plan.contract(ga, be, dtype=dtype))
    pre, sl, res, _ = plan.schedule()
    ref = _oracle_batch(n, g.edges, ga, be, opened, pre, sl, res)
    scale = np.max(np.abs(ref))
    assert np.max(np.abs(got - ref)) / scale < TOL[dtype]
    single = T.build_plan(g, p, "amplitude", "min-fill", n_sliced=k, small_log2=small)
    assert abs(got[0] - single.contract(ga, be, dtype=dtype)) / scale < TOL[dtype]
    if n <= 16:
        psi = sv.qaoa_state(n, g.edges, ga, be)
        qs = sorted(opened)
        for x in range(1 << len(qs)):
            bits = [0] * n
            for b, q in enumerate(qs):
                bits[q] = (x >> b) & 1
            assert abs(got[x] - sv.amplitude(psi, bits)) / scale < TOL[dtype]


def test_amplitude_batch_sliced_partition_bit_identical():
    n, p = 30, 1
    g = random_regular_graph(n, 3, 77)
    ga, be = qaoa_angles(p, 77)
    plan = T.build_plan(g, p, "amplitude", "min-fill", n_sliced=3, small_log2=6, open_qubits=(3, 11, 20))
    A = plan.batch
    full = torch.zeros(2 * plan.n_slices * A, dtype=torch.float64, device="cuda")
    plan.contract_sliced(ga, be, 0, plan.n_slices, full, dtype=T.TN_C64)
    parts = torch.zeros_like(full)
    for a0, b0 in ((0, 3), (3, 5), (5, 8)):
        plan.contract_sliced(ga, be, a0, b0, parts, dtype=T.TN_C64)
    torch.cuda.synchronize()
    assert torch.equal(full, parts)
    s1 = plan.sum_partials(full.cpu().tolist())
    s2, _ = run_sliced(plan, ga, be, dtype=T.TN_C64)
    assert s1 == s2 and len(s1) == A


def test_graph_replay_matches_direct_bit_for_bit(monkeypatch):
    """tn_contract_sliced replays a captured CUDA graph from the second call with the same
    arguments on (the leaves are materialised outside the graph, so new angles apply): with fresh
    angles at every call, the replayed partials equal the direct path's (TNB_GRAPH=0) bit for bit."""
    plan, g, ga, be, meta = _bench_plan()
    n = plan.n_slices
    part = torch.zeros(2 * n, dtype=torch.float64, device="cuda")
    angles = [qaoa_angles(1, 500 + i) for i in range(4)]
    res = {}
    for mode in ("0", "1"):
        monkeypatch.setenv("TNB_GRAPH", mode)
        res[mode] = []
        for gam, bet in angles:     # call 1 direct, call 2 captures, calls 3-4 replay
            part.zero_()
            plan.contract_sliced(gam, bet, 0, n, part, dtype=T.TN_C64)
            torch.cuda.synchronize()
            res[mode].append(part.cpu().clone())
    for a0, a1 in zip(res["0"], res["1"]):
        assert torch.equal(a0, a1)
    assert not torch.equal(res["1"][2], res["1"][3])   # the angles did change the result
