"""MaxCut energy via per-edge light-cone networks (oracle; test infrastructure only).

PAPER.md:184-188: the energy <gamma beta| C |gamma beta> is a "duplicated" tensor
expression (ket, bra and the gates of C); its cost depends on p,
not on the graph size (light cones).  Per edge: <Z_u Z_v> = contraction of
network.zz_cone_network (real up to rounding); E = sum_e (1 - <Z_u Z_v>)/2
(reading A3).
"""
from __future__ import annotations

from typing import List, Sequence, Tuple

from . import contract, network


def zz_values(n: int, edges: Sequence[Tuple[int, int]], gammas, betas) -> List[complex]:
    out = []
    for u, v in edges:
        tens = network.zz_cone_network(n, edges, gammas, betas, u, v)
        out.append(contract.contract(tens))
    return out


def maxcut_energy(n: int, edges, gammas, betas) -> Tuple[float, List[complex]]:
    zz = zz_values(n, edges, gammas, betas)
    return float(sum((1.0 - z.real) / 2.0 for z in zz)), zz
