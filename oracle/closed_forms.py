"""Closed forms that pin the oracle at any N (test infrastructure only).

Derivations (conventions of oracle/gates.py):

  gamma = 0 : U_C = I, e^{-i b X}|+> = e^{-i b}|+>  ->  sigma = 2^{-N/2} e^{-i N sum_l b_l}
  beta  = 0 : U_B = I, <0^N| diag phases |+>^N picks z = 0, C(0) = 0  ->  sigma = 2^{-N/2}
  gamma = pi, every degree odd : e^{-i pi C(z)} = prod_q (-1)^{deg(q) z_q} = Z^{(x)N},
      Z|+> = |->, e^{-i b X}|-> = e^{+i b}|->, Z|-> = |+>, ...
      ->  sigma = 2^{-N/2} exp(i N sum_l (-1)^{l-1} b_l)

  p = 1 edge expectation (Wang, Hadfield, Jiang, Rieffel 2018 -- cited at
  PAPER.md:173), d_u = deg(u)-1, d_v = deg(v)-1, lam = #common neighbours:
     <C_uv> = 1/2 + 1/4 sin(4b) sin(g) (cos^{d_u} g + cos^{d_v} g)
                  - 1/4 sin^2(2b) cos^{d_u+d_v-2 lam}(g) (1 - cos^{lam}(2g))
     <Z_u Z_v> = 1 - 2 <C_uv>
"""
from __future__ import annotations

import math
from typing import Sequence, Tuple


def amp_gamma0(n: int, betas: Sequence[float]) -> complex:
    return 2.0 ** (-n / 2.0) * complex(math.cos(-n * sum(betas)), math.sin(-n * sum(betas)))


def amp_beta0(n: int) -> complex:
    return complex(2.0 ** (-n / 2.0), 0.0)


def amp_gamma_pi(n: int, betas: Sequence[float]) -> complex:
    ph = n * sum(((-1) ** l) * b for l, b in enumerate(betas))  # l = 0 is layer 1
    return 2.0 ** (-n / 2.0) * complex(math.cos(ph), math.sin(ph))


def wang_p1_zz(edges: Sequence[Tuple[int, int]], u: int, v: int, gamma: float, beta: float) -> float:
    nbr = {}
    for a, b in edges:
        nbr.setdefault(a, set()).add(b)
        nbr.setdefault(b, set()).add(a)
    du = len(nbr[u]) - 1
    dv = len(nbr[v]) - 1
    lam = len((nbr[u] - {v}) & (nbr[v] - {u}))
    c = (0.5 + 0.25 * math.sin(4 * beta) * math.sin(gamma) * (math.cos(gamma) ** du + math.cos(gamma) ** dv)
         - 0.25 * math.sin(2 * beta) ** 2 * math.cos(gamma) ** (du + dv - 2 * lam)
         * (1.0 - math.cos(2 * gamma) ** lam))
    return 1.0 - 2.0 * c
