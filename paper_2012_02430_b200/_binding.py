"""Thin ctypes binding of libtnb200.so (include/tn_b200.h) -- argument marshalling only.

The function names are the C names.  Every numeric step runs in the library's CUDA
kernels; there is no Python or CPU fallback: importing this module without the built
library raises ImportError (build it with `python -m paper_2012_02430_b200.build`).
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libtnb200.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: build it with `python -m paper_2012_02430_b200.build` "
                      "(there is no CPU fallback)")
_lib = C.CDLL(LIB_PATH)

TN_C64, TN_C128 = 0, 1
TN_KIND_AMPLITUDE, TN_KIND_ENERGY = 0, 1
TN_ORDER_MIN_FILL, TN_ORDER_MIN_DEGREE, TN_ORDER_RGREEDY, TN_ORDER_RGREEDY_FILL = 0, 1, 2, 3
STATUS = {0: "TN_OK", -1: "TN_E_INVAL", -2: "TN_E_PLAN", -3: "TN_E_TOO_WIDE", -4: "TN_E_NOMEM",
          -5: "TN_E_CUDA", -6: "TN_E_DTYPE"}

SYMBOLS = ["tn_plan_build", "tn_buffer_free", "tn_slice_scan", "tn_plan_load", "tn_plan_free", "tn_plan_info",
           "tn_plan_schedule", "tn_plan_steps", "tn_contract", "tn_contract_sliced", "tn_sum_partials", "tn_energy", "tn_energy_batch",
           "tn_workspace_bytes",
           "tn_eliminate", "tn_eliminate_group", "tn_profile_enable", "tn_profile_read", "tn_profile_records", "tn_last_error", "tn_version"]


class TnError(RuntimeError):
    def __init__(self, status: int, where: str):
        self.status = status
        self.name = STATUS.get(status, str(status))
        super().__init__(f"{where}: {self.name}: {last_error()}")


class tn_build_opts(C.Structure):
    _fields_ = [("kind", C.c_int32), ("orderer", C.c_int32), ("n_sliced", C.c_int32), ("r", C.c_int32),
                ("max_width", C.c_int32), ("small_log2", C.c_int32), ("rg_q", C.c_int32),
                ("rg_tau_milli", C.c_int32), ("rg_seed", C.c_uint32), ("n_open", C.c_int32),
                ("open_qubits", C.POINTER(C.c_int32))]


class tn_plan_info_t(C.Structure):
    _fields_ = [("kind", C.c_int32), ("n_qubits", C.c_int32), ("p", C.c_int32), ("n_edges", C.c_int32),
                ("width", C.c_int32), ("unsliced_width", C.c_int32), ("k", C.c_int32),
                ("slice_step", C.c_int32), ("n_programs", C.c_int32), ("n_labels", C.c_int32),
                ("n_slices", C.c_uint64), ("prefix_steps", C.c_uint64), ("steps_per_slice", C.c_uint64),
                ("launches_prefix", C.c_uint64), ("launches_per_slice", C.c_uint64),
                ("workspace_bytes", C.c_size_t * 2), ("pred_bytes_per_slice", C.c_double * 2),
                ("pred_bytes_prefix", C.c_double * 2), ("pred_bytes_big_per_slice", C.c_double * 2),
                ("big_launches_per_slice", C.c_uint64), ("slices_batchable", C.c_int32),
                ("n_open", C.c_int32)]

    def as_dict(self):
        d = {}
        for name, _ in self._fields_:
            v = getattr(self, name)
            d[name] = list(v) if hasattr(v, "__len__") else v
        return d


class tn_step_info_t(C.Structure):
    _fields_ = [("phase", C.c_int32), ("label", C.c_int32), ("out_rank", C.c_int32), ("degree", C.c_int32),
                ("n_in", C.c_int32), ("inplace", C.c_int32), ("standalone", C.c_int32),
                ("in_rank", C.c_int32 * 8), ("in_out_mask", C.c_uint64 * 8), ("in_pv", C.c_int32 * 8),
                ("bytes_c64", C.c_double)]


class tn_prof_record_t(C.Structure):
    _fields_ = [("step_begin", C.c_int32), ("step_end", C.c_int32), ("kind", C.c_int32),
                ("out_rank", C.c_int32), ("ms", C.c_double), ("bytes", C.c_double),
                ("kernel", C.c_int32), ("pad", C.c_int32), ("flops", C.c_double)]


KERNEL_NAMES = {0: "?", 1: "k_bucket", 2: "k_chain", 3: "k_group_t", 4: "k_pair", 5: "k_gemm",
                6: "k_chain_split", 7: "k_program", 8: "k_gemm_tc", 9: "k_gemm_fc", 10: "k_fc_tc", 11: "k_gemm_hm", 12: "k_fc_hm"}


_P = C.c_void_p
_D = C.POINTER(C.c_double)
_lib.tn_plan_build.argtypes = [C.c_int32, C.c_int32, C.POINTER(C.c_int32), C.c_int32,
                               C.POINTER(tn_build_opts), C.POINTER(_P), C.POINTER(C.c_size_t)]
_lib.tn_slice_scan.argtypes = [C.c_int32, C.c_int32, C.POINTER(C.c_int32), C.c_int32, C.POINTER(tn_build_opts),
                               C.POINTER(C.c_int32), C.POINTER(C.c_int32), C.POINTER(C.c_double), C.c_int32,
                               C.POINTER(C.c_int32), C.POINTER(C.c_int32)]
_lib.tn_buffer_free.argtypes = [_P]
_lib.tn_buffer_free.restype = None
_lib.tn_plan_load.argtypes = [_P, C.c_size_t, C.POINTER(_P)]
_lib.tn_plan_free.argtypes = [_P]
_lib.tn_plan_free.restype = None
_lib.tn_plan_info.argtypes = [_P, C.POINTER(tn_plan_info_t)]
_I32P = C.POINTER(C.c_int32)
_lib.tn_plan_schedule.argtypes = [_P, _I32P, _I32P, _I32P, _I32P]
_lib.tn_plan_steps.argtypes = [_P, C.POINTER(tn_step_info_t), C.c_int64, C.POINTER(C.c_int64)]
_lib.tn_contract.argtypes = [_P, C.c_int, _D, _D, C.c_int32, _P, C.c_size_t, _P, _D]
_lib.tn_contract_sliced.argtypes = [_P, C.c_int, _D, _D, C.c_int32, C.c_uint64, C.c_uint64, _P,
                                    C.c_size_t, _P, _P]
_lib.tn_sum_partials.argtypes = [_P, _D, _D]
_lib.tn_energy.argtypes = [_P, C.c_int, _D, _D, C.c_int32, _P, C.c_size_t, _P, _D, _D, _D]
_lib.tn_energy_batch.argtypes = [_P, C.c_int, _D, _D, C.c_int32, C.c_uint64, _P, C.c_size_t, _P, _D, _D, _D]
_lib.tn_workspace_bytes.argtypes = [_P, C.c_int, C.c_uint64]
_lib.tn_eliminate.argtypes = [C.c_int, C.c_int32, C.POINTER(_P), C.POINTER(C.c_uint64), _I32P, _P,
                              C.c_int32, _P]
_lib.tn_profile_enable.argtypes = [_P, C.c_int32]
_lib.tn_profile_read.argtypes = [_P, C.POINTER(C.c_uint64), _D, _D, C.POINTER(C.c_uint64)]
_lib.tn_profile_records.argtypes = [_P, C.POINTER(tn_prof_record_t), C.c_int64, C.POINTER(C.c_int64)]
_lib.tn_last_error.restype = C.c_char_p
_lib.tn_eliminate_group.argtypes = [C.c_int, C.c_int32, C.c_int32, C.POINTER(_P), C.POINTER(C.c_uint64),
                                    C.POINTER(C.c_uint32), _P, C.c_int32, C.c_int32, _P]
_lib.tn_version.restype = C.c_int32
for _n in SYMBOLS:
    if _n not in ("tn_buffer_free", "tn_plan_free", "tn_last_error", "tn_version", "tn_workspace_bytes"):
        getattr(_lib, _n).restype = C.c_int
_lib.tn_workspace_bytes.restype = C.c_size_t


def last_error() -> str:
    return (_lib.tn_last_error() or b"").decode()


def _check(st: int, where: str):
    if st != 0:
        raise TnError(st, where)


def _dbl(xs):
    return (C.c_double * len(xs))(*[float(x) for x in xs])


# ---------------------------------------------------------------- 1:1 wrappers
def tn_version() -> int:
    return int(_lib.tn_version())


def tn_plan_build(n_qubits: int, edges, p: int, kind: int = TN_KIND_AMPLITUDE,
                  orderer: int = TN_ORDER_MIN_FILL, n_sliced: int = 0, r: int = 0,
                  max_width: int = 0, small_log2: int = -1, rg_q: int = 0, rg_tau: float = 0.0,
                  rg_seed: int = 0, open_qubits=()) -> bytes:
    flat = []
    for e in edges:
        flat.extend((int(e[0]), int(e[1])))
    arr = (C.c_int32 * max(1, len(flat)))(*flat)
    oq = [int(q) for q in open_qubits]
    oarr = (C.c_int32 * max(1, len(oq)))(*oq)
    opts = tn_build_opts(kind, orderer, n_sliced, r, max_width, small_log2, rg_q, int(round(rg_tau * 1000)),
                         rg_seed, len(oq), C.cast(oarr, C.POINTER(C.c_int32)))
    buf, ln = _P(), C.c_size_t()
    _check(_lib.tn_plan_build(n_qubits, len(flat) // 2, arr, p, C.byref(opts), C.byref(buf), C.byref(ln)),
           "tn_plan_build")
    try:
        return C.string_at(buf, ln.value)
    finally:
        _lib.tn_buffer_free(buf)


def tn_slice_scan(n_qubits: int, edges, p: int, n_sliced: int, orderer: int = TN_ORDER_MIN_FILL, r: int = 0,
                  rg_q: int = 0, rg_tau: float = 0.0, rg_seed: int = 0):
    """First-round candidates of step-dependent slicing: (list of (s, width, cost), peak)."""
    flat = []
    for e in edges:
        flat.extend((int(e[0]), int(e[1])))
    arr = (C.c_int32 * max(1, len(flat)))(*flat)
    oarr = (C.c_int32 * 1)()
    opts = tn_build_opts(TN_KIND_AMPLITUDE, orderer, n_sliced, r, 0, -1, rg_q, int(round(rg_tau * 1000)),
                         rg_seed, 0, C.cast(oarr, C.POINTER(C.c_int32)))
    n, peak = C.c_int32(), C.c_int32()
    _check(_lib.tn_slice_scan(n_qubits, len(flat) // 2, arr, p, C.byref(opts), None, None, None, 0, C.byref(n),
                              C.byref(peak)), "tn_slice_scan")
    cap = max(1, n.value)
    so, wo, co = (C.c_int32 * cap)(), (C.c_int32 * cap)(), (C.c_double * cap)()
    _check(_lib.tn_slice_scan(n_qubits, len(flat) // 2, arr, p, C.byref(opts), so, wo, co, cap, C.byref(n),
                              C.byref(peak)), "tn_slice_scan")
    return [(so[i], wo[i], co[i]) for i in range(n.value)], peak.value


def tn_plan_load(buf: bytes) -> int:
    h = _P()
    _check(_lib.tn_plan_load(buf, len(buf), C.byref(h)), "tn_plan_load")
    return h.value


def tn_plan_free(h: int) -> None:
    _lib.tn_plan_free(h)


def tn_plan_info(h: int) -> dict:
    info = tn_plan_info_t()
    _check(_lib.tn_plan_info(h, C.byref(info)), "tn_plan_info")
    return info.as_dict()


def tn_plan_schedule(h: int):
    info = tn_plan_info(h)
    s, k, L = info["slice_step"], info["k"], info["n_labels"] - info["n_open"]
    pre = (C.c_int32 * max(1, s))()
    sl = (C.c_int32 * max(1, k))()
    res = (C.c_int32 * max(1, L - s - k))()
    nd = info["prefix_steps"] + info["steps_per_slice"]
    deg = (C.c_int32 * max(1, nd))()
    _check(_lib.tn_plan_schedule(h, pre, sl, res, deg), "tn_plan_schedule")
    return list(pre)[:s], list(sl)[:k], list(res)[:L - s - k], list(deg)[:nd]


def tn_plan_steps(h: int):
    n = C.c_int64()
    _check(_lib.tn_plan_steps(h, None, 0, C.byref(n)), "tn_plan_steps")
    arr = (tn_step_info_t * max(1, n.value))()
    _check(_lib.tn_plan_steps(h, arr, n.value, C.byref(n)), "tn_plan_steps")
    out = []
    for i in range(n.value):
        s = arr[i]
        k = s.n_in
        out.append({"phase": s.phase, "label": s.label, "out_rank": s.out_rank, "degree": s.degree,
                    "n_in": k, "inplace": s.inplace, "standalone": s.standalone,
                    "in_rank": list(s.in_rank)[:k], "in_out_mask": list(s.in_out_mask)[:k],
                    "in_pv": list(s.in_pv)[:k], "bytes_c64": s.bytes_c64})
    return out


def _unpack(out, A: int):
    vals = [complex(out[2 * x], out[2 * x + 1]) for x in range(A)]
    return vals[0] if A == 1 else vals


def tn_contract(h: int, dtype: int, gammas, betas, ws_ptr: int, ws_bytes: int, stream: int):
    """sigma (complex) for a single-amplitude plan; the list of 2^a batch entries when n_open = a > 0."""
    A = 1 << tn_plan_info(h)["n_open"]
    out = (C.c_double * (2 * A))()
    _check(_lib.tn_contract(h, dtype, _dbl(gammas), _dbl(betas), len(gammas), ws_ptr, ws_bytes,
                            stream, out), "tn_contract")
    return _unpack(out, A)


def tn_contract_sliced(h: int, dtype: int, gammas, betas, begin: int, end: int, ws_ptr: int,
                       ws_bytes: int, stream: int, partials_ptr: int) -> None:
    _check(_lib.tn_contract_sliced(h, dtype, _dbl(gammas), _dbl(betas), len(gammas), begin, end,
                                   ws_ptr, ws_bytes, stream, partials_ptr), "tn_contract_sliced")


def tn_sum_partials(h: int, partials):
    """partials: flat float64 sequence [re, im] per (slice j, batch entry x) at 2 (j 2^a + x)
    (host).  Returns a complex (a = 0) or the list of 2^a batch entries."""
    A = 1 << tn_plan_info(h)["n_open"]
    arr = _dbl(list(partials))
    out = (C.c_double * (2 * A))()
    _check(_lib.tn_sum_partials(h, arr, out), "tn_sum_partials")
    return _unpack(out, A)


def tn_energy(h: int, dtype: int, gammas, betas, ws_ptr: int, ws_bytes: int, stream: int):
    E = tn_plan_info(h)["n_programs"]
    zz = (C.c_double * E)()
    im, en = C.c_double(), C.c_double()
    _check(_lib.tn_energy(h, dtype, _dbl(gammas), _dbl(betas), len(gammas), ws_ptr, ws_bytes, stream,
                          zz, C.byref(im), C.byref(en)), "tn_energy")
    return list(zz), im.value, en.value


def tn_workspace_bytes(h: int, dtype: int, batch: int) -> int:
    return int(_lib.tn_workspace_bytes(h, dtype, batch))


def tn_energy_batch(h: int, dtype: int, gammas_sets, betas_sets, ws_ptr: int, ws_bytes: int, stream: int):
    """gammas_sets / betas_sets: B sequences of p angles each."""
    B = len(gammas_sets)
    p = len(gammas_sets[0])
    E = tn_plan_info(h)["n_programs"]
    zz = (C.c_double * (E * B))()
    im = (C.c_double * B)()
    en = (C.c_double * B)()
    _check(_lib.tn_energy_batch(h, dtype, _dbl([x for g in gammas_sets for x in g]),
                                _dbl([x for b in betas_sets for x in b]), p, B, ws_ptr, ws_bytes, stream,
                                zz, im, en), "tn_energy_batch")
    return [list(zz[b * E:(b + 1) * E]) for b in range(B)], list(im), list(en)


def tn_eliminate(dtype: int, in_ptrs, out_masks, pvs, out_ptr: int, out_rank: int, stream: int) -> None:
    n = len(in_ptrs)
    ins = (_P * n)(*in_ptrs)
    masks = (C.c_uint64 * n)(*out_masks)
    pv = (C.c_int32 * n)(*pvs)
    _check(_lib.tn_eliminate(dtype, n, ins, masks, pv, out_ptr, out_rank, stream), "tn_eliminate")


def tn_eliminate_group(dtype: int, M: int, in_ptrs, out_masks, x_masks, out_ptr: int, out_rank: int,
                       kernel: int, stream: int) -> None:
    n = len(in_ptrs)
    ins = (_P * n)(*in_ptrs)
    masks = (C.c_uint64 * n)(*out_masks)
    xm = (C.c_uint32 * n)(*x_masks)
    _check(_lib.tn_eliminate_group(dtype, M, n, ins, masks, xm, out_ptr, out_rank, kernel, stream),
           "tn_eliminate_group")


def tn_profile_enable(h: int, enable: bool) -> None:
    _check(_lib.tn_profile_enable(h, 1 if enable else 0), "tn_profile_enable")


def tn_profile_read(h: int):
    n, alln = C.c_uint64(), C.c_uint64()
    ms, by = C.c_double(), C.c_double()
    _check(_lib.tn_profile_read(h, C.byref(n), C.byref(ms), C.byref(by), C.byref(alln)), "tn_profile_read")
    return {"launches": n.value, "ms": ms.value, "bytes": by.value, "all_launches": alln.value}


def tn_profile_records(h: int):
    n = C.c_int64()
    _check(_lib.tn_profile_records(h, None, 0, C.byref(n)), "tn_profile_records")
    arr = (tn_prof_record_t * max(1, n.value))()
    _check(_lib.tn_profile_records(h, arr, n.value, C.byref(n)), "tn_profile_records")
    return [{"step_begin": r.step_begin, "step_end": r.step_end, "kind": ("step", "chain", "group", "run")[r.kind - 1],
             "kernel": KERNEL_NAMES.get(r.kernel, "?"), "out_rank": r.out_rank, "ms": r.ms, "bytes": r.bytes,
             "flops": r.flops} for r in arr[:n.value]]
