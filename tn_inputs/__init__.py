"""Seeded synthetic inputs shared by the product path, the oracle and the tests.

This module holds NONE of the method's arithmetic: it only draws the problem
instance the paper benchmarks on -- a random 3-regular MaxCut graph
(§3.2 "random 3-regular graphs") and the 2p QAOA angles
(§3.1 "parametrized by 2p variational parameters").

Generator (reading A16):
  * a splitmix64-seeded PCG32 (XSH-RR) stream, one per (seed, stream-tag);
  * configuration-model pairing with full resample on a self-loop or a
    multi-edge, at most 10,000 attempts;
  * gamma_1..gamma_p then beta_1..beta_p ~ U(0, pi) from their own stream.

Both the CUDA path (through `bench.py` / the binding) and `oracle/` consume
these values; neither side generates its own instances.
"""
from __future__ import annotations

import math
from dataclasses import dataclass
from typing import List, Sequence, Tuple

_M64 = (1 << 64) - 1


def splitmix64(x: int) -> int:
    """One splitmix64 output for state x (used only to seed PCG32)."""
    x = (x + 0x9E3779B97F4A7C15) & _M64
    z = x
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
    return z ^ (z >> 31)


class PCG32:
    """Minimal PCG32 (XSH-RR, 64-bit LCG state)."""

    _MULT = 6364136223846793005

    def __init__(self, seed: int, stream: int = 0):
        self.state = 0
        self.inc = ((splitmix64(stream ^ 0xDA3E39CB94B95BDB) << 1) | 1) & _M64
        self.next_u32()
        self.state = (self.state + splitmix64(seed & _M64)) & _M64
        self.next_u32()

    def next_u32(self) -> int:
        old = self.state
        self.state = (old * self._MULT + self.inc) & _M64
        xorshifted = (((old >> 18) ^ old) >> 27) & 0xFFFFFFFF
        rot = old >> 59
        return ((xorshifted >> rot) | (xorshifted << ((-rot) & 31))) & 0xFFFFFFFF

    def bounded(self, n: int) -> int:
        """Uniform integer in [0, n) by rejection (no modulo bias)."""
        if n <= 0:
            raise ValueError("bounded(n) needs n > 0")
        threshold = ((1 << 32) - n) % n
        while True:
            r = self.next_u32()
            if r >= threshold:
                return r % n

    def uniform(self) -> float:
        """Uniform double in [0, 1) with 53 random bits."""
        a = self.next_u32() >> 5
        b = self.next_u32() >> 6
        return (a * 67108864.0 + b) / 9007199254740992.0


# stream tags (fixed; changing them changes every instance)
STREAM_GRAPH = 1
STREAM_ANGLES = 2


@dataclass(frozen=True)
class Graph:
    n: int
    edges: Tuple[Tuple[int, int], ...]  # sorted, i < j

    def degree(self, q: int) -> int:
        return sum(1 for e in self.edges if q in e)


def random_regular_graph(n: int, d: int, seed: int, max_tries: int = 10000) -> Graph:
    """Simple d-regular graph on n nodes (configuration model, full resample).

    SPEC.md:49-57 (random_regular_graph): n*d even, d < n; deterministic for a seed.
    Edges are returned sorted with i < j (the builder's stored edge order).
    """
    if n <= 0 or d < 0:
        raise ValueError("need n > 0, d >= 0")
    if (n * d) % 2 != 0 or d >= n:
        raise ValueError(f"infeasible regular graph n={n} d={d}")
    rng = PCG32(seed, STREAM_GRAPH)
    stubs0 = [q for q in range(n) for _ in range(d)]
    for _ in range(max_tries):
        stubs = list(stubs0)
        for i in range(len(stubs) - 1, 0, -1):  # Fisher-Yates
            j = rng.bounded(i + 1)
            stubs[i], stubs[j] = stubs[j], stubs[i]
        seen = set()
        ok = True
        for k in range(0, len(stubs), 2):
            a, b = stubs[k], stubs[k + 1]
            if a == b:
                ok = False
                break
            e = (a, b) if a < b else (b, a)
            if e in seen:
                ok = False
                break
            seen.add(e)
        if ok:
            return Graph(n, tuple(sorted(seen)))
    raise RuntimeError(f"no simple {d}-regular graph on {n} nodes in {max_tries} tries")


def qaoa_angles(p: int, seed: int) -> Tuple[List[float], List[float]]:
    """gamma_1..gamma_p then beta_1..beta_p, each ~ U(0, pi)."""
    rng = PCG32(seed, STREAM_ANGLES)
    gammas = [math.pi * rng.uniform() for _ in range(p)]
    betas = [math.pi * rng.uniform() for _ in range(p)]
    return gammas, betas


def edges_array(g: Graph) -> List[int]:
    """Flat [i0, j0, i1, j1, ...] edge list for C-ABI marshalling."""
    out: List[int] = []
    for i, j in g.edges:
        out.extend((i, j))
    return out


# ---------------------------------------------------------------------------
# Named workloads (BASELINE.json configs; readings in SURVEY.md §0 F3, §8)
# ---------------------------------------------------------------------------
@dataclass(frozen=True)
class Workload:
    name: str
    n: int
    p: int
    kind: str          # "amplitude" | "energy"
    seed: int = 0
    note: str = ""


WORKLOADS = {
    "C1": Workload("C1", 16, 1, "energy", note="24 light-cone <ZiZj> networks, c128"),
    "C2": Workload("C2", 56, 2, "amplitude", note="single amplitude, c64, min-fill, unsliced"),
    "C3": Workload("C3", 100, 3, "energy", note="150 light-cone networks, c64 and c128"),
    "C4a": Workload("C4a", 150, 1, "amplitude", note="sliced, width<=30"),
    "C4b": Workload("C4b", 64, 3, "amplitude", note="sliced, width<=30 (p=3 companion)"),
    "C5a": Workload("C5a", 210, 1, "amplitude", note="paper's 210-qubit 1,785-gate circuit, width<=32"),
    "C5b": Workload("C5b", 70, 3, "amplitude", note="p=3 companion with 210 live indices, width<=32"),
    # the paper's own plan for the 210-qubit circuit (greedy min-degree, r = n):
    # k = 9 (width 30 on this instance) and k = 6 (width 33: over the 2^32 cap, reported only)
    "C5r": Workload("C5r", 210, 1, "amplitude", note="paper-replica plan: min-degree, k=9, r=n"),
    "C5r6": Workload("C5r6", 210, 1, "amplitude", note="paper-replica plan: min-degree, k=6, r=n"),
}


def workload_instance(name: str, seed: int | None = None):
    w = WORKLOADS[name]
    s = w.seed if seed is None else seed
    g = random_regular_graph(w.n, 3, s)
    gammas, betas = qaoa_angles(w.p, s)
    return w, g, gammas, betas


def random_complex(shape: Sequence[int], seed: int):
    """Seeded complex128 test tensor, entries uniform in the unit square (numpy)."""
    import numpy as np

    rng = np.random.default_rng(seed)
    return rng.uniform(-1, 1, size=tuple(shape)) + 1j * rng.uniform(-1, 1, size=tuple(shape))
