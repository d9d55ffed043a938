"""Gate matrices (oracle; test infrastructure only).

PAPER.md:69-83 (Fig. 1: H, CNOT, Z^{2gamma}, Z^{2beta}) and the QAOA ansatz
PAPER.md:161-163 (|psi_p> = prod_k e^{-i beta_k H_B} e^{-i gamma_k H_C}|psi_0>,
H_B = sum_j sigma_x^j).  Conventions (reading A1):
  * Z^t = diag(1, e^{i pi t})
  * MaxCut cost C_ij = (1 - Z_i Z_j)/2, U_C(gamma) = e^{-i gamma C}
    -> on the computational-basis bits (a, b) of an edge, the diagonal
       factor is 1 if a == b else e^{-i gamma}                  ("ZZ(gamma)")
  * U_B(beta) = e^{-i beta X} = [[cos b, -i sin b], [-i sin b, cos b]]  ("RX(2 beta)")
"""
from __future__ import annotations

import numpy as np

SQRT1_2 = 1.0 / np.sqrt(2.0)

H = np.array([[1.0, 1.0], [1.0, -1.0]], dtype=np.complex128) * SQRT1_2
X = np.array([[0.0, 1.0], [1.0, 0.0]], dtype=np.complex128)
Z = np.array([[1.0, 0.0], [0.0, -1.0]], dtype=np.complex128)
I2 = np.eye(2, dtype=np.complex128)


def zpow_diag(t: float) -> np.ndarray:
    """Diagonal of Z^t = diag(1, e^{i pi t}) (ZPow(1) = [1, -1])."""
    return np.array([1.0, np.exp(1j * np.pi * t)], dtype=np.complex128)


def cnot_tensor() -> np.ndarray:
    """CNOT as values[c, t_in, t_out] (SPEC.md:84 truth table)."""
    t = np.zeros((2, 2, 2), dtype=np.complex128)
    for c in range(2):
        for i in range(2):
            o = i ^ c
            t[c, i, o] = 1.0
    return t


def cnot_matrix() -> np.ndarray:
    """4x4 CNOT on |c t> (c most significant)."""
    m = np.zeros((4, 4), dtype=np.complex128)
    for c in range(2):
        for t in range(2):
            m[(c << 1) | (t ^ c), (c << 1) | t] = 1.0
    return m


def zz_phase(gamma: float) -> np.ndarray:
    """e^{-i gamma (1 - z_a z_b)/2} on the bits (a, b) of one edge, as a 2x2 array."""
    ph = np.exp(-1j * gamma)
    return np.array([[1.0, ph], [ph, 1.0]], dtype=np.complex128)


def rx(beta: float) -> np.ndarray:
    """e^{-i beta X}: the per-qubit mixer of U_B(beta) (matrix [out, in])."""
    c, s = np.cos(beta), np.sin(beta)
    return np.array([[c, -1j * s], [-1j * s, c]], dtype=np.complex128)


def expm_hermitian(hmat: np.ndarray, t: float) -> np.ndarray:
    """e^{-i t H} by eigendecomposition (used only to pin rx / zz_phase)."""
    w, v = np.linalg.eigh(hmat)
    return (v * np.exp(-1j * t * w)) @ v.conj().T
