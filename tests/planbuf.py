"""Test helper: parse a plan buffer (csrc/plan_format.h layout) with ctypes structures, so host
tests can check the lowered program (arena offsets, ops) without any device code.

Layout: PlanHeader | ProgramRec[n_programs] | LeafRec[n_leaves] | StepRec[n_steps] | OpRec[n_ops]
| ScalarRec[n_scalars] | int32 prefix | int32 sliced | int32 residual | int32 degrees.
"""
from __future__ import annotations

import ctypes as C

OP_BIG, OP_RUN, OP_CHAIN, OP_GROUP, OP_PRUN, OP_GROUP_FEED = range(6)
F_REL = 4
ALIGN = 32


class PlanHeader(C.Structure):
    _fields_ = [("magic", C.c_uint32), ("version", C.c_uint32),
                ("kind", C.c_int32), ("n_qubits", C.c_int32), ("p", C.c_int32), ("n_edges", C.c_int32),
                ("width", C.c_int32), ("unsliced_width", C.c_int32), ("k", C.c_int32), ("slice_step", C.c_int32),
                ("orderer", C.c_int32), ("r", C.c_int32), ("small_log2", C.c_int32), ("n_labels", C.c_int32),
                ("n_programs", C.c_int32), ("n_leaves", C.c_int32), ("n_steps", C.c_int32), ("n_ops", C.c_int32),
                ("n_scalars", C.c_int32),
                ("n_prefix", C.c_int32), ("n_residual", C.c_int32), ("n_degrees", C.c_int32),
                ("arena_elems", C.c_uint64), ("persistent_elems", C.c_uint64),
                ("pred_elems_slice", C.c_double), ("pred_elems_prefix", C.c_double),
                ("pred_elems_big_slice", C.c_double), ("big_launches_slice", C.c_uint64),
                ("launches_prefix", C.c_uint64), ("launches_slice", C.c_uint64),
                ("n_open", C.c_int32), ("pad0", C.c_int32), ("reserved", C.c_uint64 * 3)]


class ProgramRec(C.Structure):
    _fields_ = [("stepA_begin", C.c_int32), ("stepA_end", C.c_int32), ("opA_begin", C.c_int32),
                ("opA_end", C.c_int32), ("stepB_begin", C.c_int32), ("stepB_end", C.c_int32),
                ("opB_begin", C.c_int32), ("opB_end", C.c_int32), ("scal_begin", C.c_int32),
                ("scal_end", C.c_int32), ("edge_u", C.c_int32), ("edge_v", C.c_int32),
                ("log2_scale", C.c_double), ("arena_begin", C.c_uint64), ("arena_end", C.c_uint64)]


class LeafRec(C.Structure):
    _fields_ = [("off", C.c_uint64), ("rank", C.c_int32), ("nfact", C.c_int32), ("code", C.c_uint8 * 4),
                ("layer", C.c_uint8 * 4), ("conj", C.c_uint8 * 4), ("pad", C.c_uint8 * 4)]


class InRec(C.Structure):
    _fields_ = [("off", C.c_uint64), ("out_mask", C.c_uint64), ("rank", C.c_uint32),
                ("slice_mask", C.c_uint32), ("pv", C.c_uint32), ("flags", C.c_uint32)]


class StepRec(C.Structure):
    _fields_ = [("out_off", C.c_uint64), ("out_rank", C.c_int32), ("n_in", C.c_int32), ("inplace", C.c_int32),
                ("phase", C.c_int32), ("label", C.c_int32), ("degree", C.c_int32), ("in_", InRec * 8)]


class OpRec(C.Structure):
    _fields_ = [("type", C.c_int32), ("begin", C.c_int32), ("end", C.c_int32), ("phase", C.c_int32)]


def _arr(buf: bytes, off: int, typ, n: int):
    sz = C.sizeof(typ)
    return [typ.from_buffer_copy(buf, off + i * sz) for i in range(n)], off + n * sz


def parse(buf: bytes) -> dict:
    h = PlanHeader.from_buffer_copy(buf, 0)
    off = C.sizeof(PlanHeader)
    progs, off = _arr(buf, off, ProgramRec, h.n_programs)
    leaves, off = _arr(buf, off, LeafRec, h.n_leaves)
    steps, off = _arr(buf, off, StepRec, h.n_steps)
    ops, off = _arr(buf, off, OpRec, h.n_ops)
    return {"header": h, "programs": progs, "leaves": leaves, "steps": steps, "ops": ops}


def span(rank: int, slice_bits: int = 0) -> int:
    """Arena elements a tensor of `rank` phase bits and `slice_bits` sliced bits occupies."""
    n = 1 << (rank + slice_bits)
    return (n + ALIGN - 1) // ALIGN * ALIGN


def feed_overlaps(buf: bytes):
    """Every OP_GROUP_FEED pair whose consumer output range intersects an input of the producer
    group (the fused launch would write over memory other CTAs still read)."""
    P = parse(buf)
    steps, ops = P["steps"], P["ops"]
    bad = []
    for oi, a in enumerate(ops):
        if a.type != OP_GROUP_FEED or oi + 1 >= len(ops):
            continue
        b = ops[oi + 1]
        head = steps[b.begin]
        lo, hi = head.out_off, head.out_off + span(head.out_rank)
        for si in range(a.begin, a.end):
            st = steps[si]
            for t in range(st.n_in):
                if si > a.begin and t == 0 and st.inplace:
                    continue  # the in-place chain intermediate (never written by the fused launch)
                i = st.in_[t]
                ilo, ihi = i.off, i.off + span(i.rank, bin(i.slice_mask).count("1"))
                if ilo < hi and lo < ihi:
                    bad.append((oi, si, t, (ilo, ihi), (lo, hi)))
    return bad
