"""ORACLE -- TEST INFRASTRUCTURE ONLY.

A plain, slow, obviously-correct CPU implementation (numpy, complex128) of what
the hot path computes, written from the paper and checked against
values the paper and the mathematics fix (tests/test_oracle_*.py, -m "not gpu").

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s `cpu_baseline` /
`--impl reference` leg may import anything under `oracle/`.  The product path
(`paper_2012_02430_b200`, `include/`, the CUDA library) never imports, links or
executes it, and the oracle imports nothing from the product path: the two
share no code.  The only common module is `tn_inputs` (seeded graph and angle
draws, none of the method's arithmetic).

Modules
  gates        textbook gate matrices (Fig. 1)
  statevector  2^N state-vector simulation (pins; N <= ~20)
  closed_forms special-angle amplitudes and Wang et al.'s p=1 <ZZ> (pins)
  network      circuit -> tensor expression (§4.1-4.2), fixing, cones
  contract     bucket elimination, Eq. (1) slicing, greedy
  energy       per-edge light-cone <Z_u Z_v> and MaxCut energy

Parity status: every function above is pinned;
none is "parity unpinned".
"""
