"""Circuit -> tensor expression (oracle; test infrastructure only).

PAPER.md:199-235 (§4.1): a gate is a tensor with input and output indices per
qubit; the input index of a gate is the output index of the previous one;
repeated indices are summed.  PAPER.md:350-359 (§4.2): a gate that is diagonal
on a qubit uses ONE index for its input and output on that wire (Fig. 2,
"gadgets").  Fixed boundary indices are sliced away.

A network is a list of (array, labels): `array.ndim == len(labels)`, axis a of
the array is index labels[a], every index has dimension 2.

Index labels of the fused single-amplitude network (reading A6):
   live wire w(q, l), l = 0..p-1 (the wire of qubit q before the layer-(l+1)
   mixer)  ->  label l*N + q;   output wire w(q, p) -> p*N + q (fixed to 0);
   input wire (before H) -> (p+1)*N + q (fixed to 0).
"""
from __future__ import annotations

from typing import Dict, List, Sequence, Tuple

import numpy as np

from . import gates

Tensor = Tuple[np.ndarray, Tuple[int, ...]]


# ------------------------------------------------------------------ fixing
def fix_indices(tensors: Sequence[Tensor], fixed: Dict[int, int]) -> List[Tensor]:
    """Replace every tensor containing a fixed label by its sub-array.

    Also Eq. (1)'s slice operation ("slicing any tensor with those indices").
    """
    out: List[Tensor] = []
    for arr, labs in tensors:
        idx = tuple(fixed[l] if l in fixed else slice(None) for l in labs)
        new_labs = tuple(l for l in labs if l not in fixed)
        out.append((np.asarray(arr[idx]), new_labs))
    return out


# ------------------------------------------------------------------ QAOA, fused gates
def qaoa_amplitude_network(n: int, edges: Sequence[Tuple[int, int]], gammas, betas,
                           out_bits: Sequence[int] | None = None,
                           open_qubits: Sequence[int] = ()) -> List[Tensor]:
    """Tensor expression of sigma = <out| U |0^N>, boundary fixed.

    U = prod_l [RX(2 beta_l)^{(x)N} prod_e ZZ(gamma_l)] H^{(x)N}  (Fig. 1 with the
    CNOT-Z-CNOT gadget fused into the diagonal ZZ(gamma); reading A1).

    open_qubits: output wires w(q, p) = p*N + q left OPEN instead of fixed (PAPER.md:599-603,
    §6 "if we decide to leave out some indices, the result will be a tensor indexed by those
    indices"): the network then evaluates the batch of 2^a amplitudes <x_open 0_rest|U|0^N>.
    """
    p = len(gammas)
    assert len(betas) == p and p >= 1

    def w(q, l):
        return l * n + q

    def inp(q):
        return (p + 1) * n + q

    tens: List[Tensor] = []
    for q in range(n):
        tens.append((gates.H.copy(), (w(q, 0), inp(q))))          # H[out, in]
    for l in range(1, p + 1):
        zz = gates.zz_phase(gammas[l - 1])
        for i, j in edges:
            tens.append((zz, (w(i, l - 1), w(j, l - 1))))           # diagonal: 1 index per wire
        m = gates.rx(betas[l - 1])
        for q in range(n):
            tens.append((m, (w(q, l), w(q, l - 1))))               # RX[out, in]
    out_bits = [0] * n if out_bits is None else list(out_bits)
    fixed = {inp(q): 0 for q in range(n)}
    opened = set(open_qubits)
    fixed.update({w(q, p): out_bits[q] for q in range(n) if q not in opened})
    return fix_indices(tens, fixed)


def open_labels(n: int, p: int, open_qubits: Sequence[int]) -> List[int]:
    """Labels of the open output wires, in ascending qubit order: bit b of a batch index is the
    output bit of the b-th open qubit (ascending)."""
    return [p * n + q for q in sorted(open_qubits)]


def live_labels(tensors: Sequence[Tensor]) -> List[int]:
    s = set()
    for _, labs in tensors:
        s.update(labs)
    return sorted(s)


# ------------------------------------------------------------------ light cones
def light_cone(n: int, edges: Sequence[Tuple[int, int]], p: int, u: int, v: int):
    """Reverse light cone of Z_u Z_v through p QAOA layers (reading A17).

    L_p = {u, v};  E_l = edges touching L_l;  L_{l-1} = L_l U endpoints(E_l).
    Returns (L, E, m) with L[l] (l = 0..p), E[l] (l = 1..p) and
    m[q] = max{ l : q in L_l } for q in L_0.
    """
    L = {p: {u, v}}
    E = {}
    for l in range(p, 0, -1):
        E[l] = [(i, j) for (i, j) in edges if i in L[l] or j in L[l]]
        L[l - 1] = set(L[l])
        for i, j in E[l]:
            L[l - 1].update((i, j))
    m = {q: max(l for l in range(p + 1) if q in L[l]) for q in L[0]}
    return L, E, m


def zz_cone_network(n: int, edges, gammas, betas, u: int, v: int) -> List[Tensor]:
    """<psi| Z_u Z_v |psi> restricted to the reverse light cone.

    Ket wire of qubit q at level a (a = 0..m_q): k(q, a); bra wire b(q, a); the top
    level a = m_q is one shared index t_q (between the ket and the bra there is
    only Z_u Z_v).  Ket tensors: |+> on k(q,0); ZZ(gamma_l) on (k(i,l-1), k(j,l-1))
    for (i, j) in E_l; RX(2 beta_l) from k(q,l-1) to k(q,l) for l <= m_q.  The bra
    tensors are their complex conjugates on the b wires.  Z on t_u and t_v.
    """
    p = len(gammas)
    L, E, m = light_cone(n, edges, p, u, v)
    labels: Dict[Tuple[str, int, int], int] = {}

    def lab(key):
        if key not in labels:
            labels[key] = len(labels)
        return labels[key]

    def k(q, a):
        return lab(("t", q, 0)) if a == m[q] else lab(("k", q, a))

    def b(q, a):
        return lab(("t", q, 0)) if a == m[q] else lab(("b", q, a))

    plus = np.array([1.0, 1.0], dtype=np.complex128) * gates.SQRT1_2
    tens: List[Tensor] = []
    for q in sorted(L[0]):
        tens.append((plus, (k(q, 0),)))
        tens.append((plus.conj(), (b(q, 0),)))
    for l in range(1, p + 1):
        zz = gates.zz_phase(gammas[l - 1])
        for i, j in E[l]:
            tens.append((zz, (k(i, l - 1), k(j, l - 1))))
            tens.append((zz.conj(), (b(i, l - 1), b(j, l - 1))))
        m_rx = gates.rx(betas[l - 1])
        for q in sorted(L[0]):
            if m[q] >= l:
                tens.append((m_rx, (k(q, l), k(q, l - 1))))
                tens.append((m_rx.conj(), (b(q, l), b(q, l - 1))))
    zd = np.array([1.0, -1.0], dtype=np.complex128)
    tens.append((zd, (lab(("t", u, 0)),)))
    tens.append((zd, (lab(("t", v, 0)),)))
    return tens


# ------------------------------------------------------------------ generic gate lists
def circuit_network(n: int, gate_list, in_bits: Sequence[int], out_bits: Sequence[int]) -> List[Tensor]:
    """SPEC.md:127-135 circuit_to_network for {h, x, zpow, cnot, cz}, boundary fixed.

    A fresh label is created only where a gate is non-diagonal on a wire; ZPow and
    CZ are diagonal on their qubits, CNOT on its control.
    """
    cur = list(range(n))          # current label of each wire
    nxt = n
    tens: List[Tensor] = []
    for kind, t, qs in gate_list:
        if kind in ("h", "x"):
            m = gates.H if kind == "h" else gates.X
            q = qs[0]
            tens.append((m, (nxt, cur[q])))
            cur[q] = nxt
            nxt += 1
        elif kind == "zpow":
            tens.append((gates.zpow_diag(t), (cur[qs[0]],)))
        elif kind == "cz":
            tens.append((np.array([[1, 1], [1, -1]], dtype=np.complex128), (cur[qs[0]], cur[qs[1]])))
        elif kind == "cnot":
            c, tq = qs
            tens.append((gates.cnot_tensor(), (cur[c], cur[tq], nxt)))  # [c, t_in, t_out]
            cur[tq] = nxt
            nxt += 1
        else:
            raise ValueError(kind)
    fixed = {q: in_bits[q] for q in range(n)}
    for q in range(n):
        fixed[cur[q]] = out_bits[q] if cur[q] != q else fixed[q]
        if cur[q] == q and out_bits[q] != in_bits[q]:
            return [(np.zeros(()), ())]   # identity wire with different boundary bits
    return fix_indices(tens, fixed)
