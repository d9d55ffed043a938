"""Dense 2^N state-vector simulation (oracle pin; test infrastructure only).

The plain definition of what the tensor network computes: sigma =
<0^N| U |0^N> (§5) and <psi| Z_u Z_v |psi>.
Axis q of the (2,)*N state tensor is qubit q.
"""
from __future__ import annotations

from typing import Iterable, List, Sequence, Tuple

import numpy as np

from . import gates


def zero_state(n: int) -> np.ndarray:
    psi = np.zeros((2,) * n, dtype=np.complex128)
    psi[(0,) * n] = 1.0
    return psi


def apply_1q(psi: np.ndarray, m: np.ndarray, q: int) -> np.ndarray:
    """psi'[.., o, ..] = sum_i m[o, i] psi[.., i, ..] on axis q."""
    out = np.tensordot(m, psi, axes=([1], [q]))
    return np.moveaxis(out, 0, q)


def apply_2q(psi: np.ndarray, m4: np.ndarray, a: int, b: int) -> np.ndarray:
    """4x4 matrix on (a, b), a the more significant bit of the pair."""
    m = m4.reshape(2, 2, 2, 2)  # [oa, ob, ia, ib]
    out = np.tensordot(m, psi, axes=([2, 3], [a, b]))
    return np.moveaxis(out, [0, 1], [a, b])


def apply_diag_1q(psi: np.ndarray, d: np.ndarray, q: int) -> np.ndarray:
    shape = [1] * psi.ndim
    shape[q] = 2
    return psi * d.reshape(shape)


# ---------------------------------------------------------------- gate lists
# gate = (kind, params, qubits): kind in {"h", "x", "zpow", "cnot", "cz"}
Gate = Tuple[str, float, Tuple[int, ...]]


def run_gates(n: int, gate_list: Iterable[Gate], psi: np.ndarray | None = None) -> np.ndarray:
    psi = zero_state(n) if psi is None else psi.copy()
    for kind, t, qs in gate_list:
        if kind == "h":
            psi = apply_1q(psi, gates.H, qs[0])
        elif kind == "x":
            psi = apply_1q(psi, gates.X, qs[0])
        elif kind == "zpow":
            psi = apply_diag_1q(psi, gates.zpow_diag(t), qs[0])
        elif kind == "cnot":
            psi = apply_2q(psi, gates.cnot_matrix(), qs[0], qs[1])
        elif kind == "cz":
            psi = apply_2q(psi, np.diag([1, 1, 1, -1]).astype(np.complex128), qs[0], qs[1])
        else:
            raise ValueError(kind)
    return psi


def fig1_circuit(n: int, edges: Sequence[Tuple[int, int]], gammas, betas) -> List[Gate]:
    """The literal Fig. 1 gate list.

    H on every qubit; per layer k: per edge (i, j): CNOT(i, j), Z^{2 gamma_k / pi}
    on j, CNOT(i, j); per qubit: H, Z^{2 beta_k / pi}, H.
    """
    g: List[Gate] = [("h", 0.0, (q,)) for q in range(n)]
    for gam, bet in zip(gammas, betas):
        for i, j in edges:
            g.append(("cnot", 0.0, (i, j)))
            g.append(("zpow", 2.0 * gam / np.pi, (j,)))
            g.append(("cnot", 0.0, (i, j)))
        for q in range(n):
            g.append(("h", 0.0, (q,)))
            g.append(("zpow", 2.0 * bet / np.pi, (q,)))
            g.append(("h", 0.0, (q,)))
    return g


# ---------------------------------------------------------------- QAOA (fused)
def cut_values(n: int, edges: Sequence[Tuple[int, int]]) -> np.ndarray:
    """C(z) = number of cut edges for every basis state z (shape (2,)*n)."""
    idx = np.indices((2,) * n).reshape(n, -1)
    c = np.zeros(idx.shape[1], dtype=np.float64)
    for i, j in edges:
        c += (idx[i] != idx[j])
    return c.reshape((2,) * n)


def qaoa_state(n: int, edges, gammas, betas) -> np.ndarray:
    """|psi_p> = prod_k e^{-i beta_k H_B} e^{-i gamma_k C} H^{(x)N}|0^N>."""
    psi = np.full((2,) * n, 2.0 ** (-n / 2.0), dtype=np.complex128)
    cz = cut_values(n, edges)
    for gam, bet in zip(gammas, betas):
        psi = psi * np.exp(-1j * gam * cz)
        m = gates.rx(bet)
        for q in range(n):
            psi = apply_1q(psi, m, q)
    return psi


def amplitude(psi: np.ndarray, bits: Sequence[int] | None = None) -> complex:
    n = psi.ndim
    bits = (0,) * n if bits is None else tuple(bits)
    return complex(psi[bits])


def zz_expectation(psi: np.ndarray, u: int, v: int) -> float:
    n = psi.ndim
    idx = np.indices((2,) * n)
    zu = 1 - 2 * idx[u]
    zv = 1 - 2 * idx[v]
    return float(np.sum(np.abs(psi) ** 2 * zu * zv))


def maxcut_energy(psi: np.ndarray, edges) -> float:
    """<psi| sum_e (1 - Z_u Z_v)/2 |psi>."""
    return float(sum((1.0 - zz_expectation(psi, u, v)) / 2.0 for u, v in edges))
