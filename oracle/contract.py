"""Bucket elimination and Eq. (1) slicing (oracle; test infrastructure only).

PAPER.md:361-368 (§4.2): the network is contracted by sequential elimination of
its indices; the tensor produced by eliminating index i is indexed by the union
of the index sets of the tensors containing i, minus i.  Buckets are keyed by
the earliest index in the elimination order.  Each
bucket is ONE numpy.einsum call (a library primitive serving as one step, in
complex128); scalars are multiplied into a running accumulator.

PAPER.md:519-524, Eq. (1):  sum_{m_1..m_n} ( sum_{V \\ {m_i}} T^1 ... T^N ).
Step-dependent slicing: the prefix of the order is
contracted once with the sliced indices still present, then every slice fixes
the sliced indices in the remaining tensors and contracts the residual order.
Slice results are summed in a fixed pairwise tree over the slice id j, bit b of
j being the value of the b-th sliced label in ascending label order (A13, A14).

`greedy_min_degree` is the oracle's OWN orderer (ties to the
smallest label), independent of the product planner.
"""
from __future__ import annotations

from typing import Dict, Iterable, List, Sequence, Tuple

import numpy as np

from .network import Tensor, fix_indices


def _einsum_bucket(ts: Sequence[Tensor], v: int) -> Tensor:
    union = sorted(set().union(*[set(l) for _, l in ts]) - {v})
    local = {lab: i for i, lab in enumerate(union + [v])}
    if len(local) > 52:
        raise ValueError("bucket too wide for numpy.einsum sublists")
    args = []
    for arr, labs in ts:
        args.append(arr)
        args.append([local[l] for l in labs])
    args.append([local[l] for l in union])
    out = np.einsum(*args, optimize=False)
    return np.asarray(out, dtype=np.complex128), tuple(union)


def partial_eliminate(tensors: Sequence[Tensor], order: Sequence[int]):
    """Eliminate the indices of `order` (in order); return (remaining tensors, scalar).

    Tensors touching no index of `order` pass through unchanged.
    """
    pos = {lab: i for i, lab in enumerate(order)}
    buckets: Dict[int, List[Tensor]] = {v: [] for v in order}
    rest: List[Tensor] = []
    scalar = complex(1.0)
    for arr, labs in tensors:
        if len(labs) == 0:
            scalar *= complex(arr)
            continue
        ins = [l for l in labs if l in pos]
        if ins:
            buckets[min(ins, key=pos.__getitem__)].append((arr, tuple(labs)))
        else:
            rest.append((arr, tuple(labs)))
    for v in order:
        ts = buckets[v]
        if not ts:
            continue
        arr, labs = _einsum_bucket(ts, v)
        if len(labs) == 0:
            scalar *= complex(arr)
            continue
        ins = [l for l in labs if l in pos]
        if ins:
            buckets[min(ins, key=pos.__getitem__)].append((arr, labs))
        else:
            rest.append((arr, labs))
    return rest, scalar


def bucket_eliminate(tensors: Sequence[Tensor], order: Sequence[int]) -> complex:
    """Full contraction to a scalar along `order` (must cover every label)."""
    rest, scalar = partial_eliminate(tensors, order)
    if rest:
        missing = sorted(set().union(*[set(l) for _, l in rest]))
        raise ValueError(f"order misses live labels {missing[:8]}")
    return scalar


def contract_open(tensors: Sequence[Tensor], open_labels: Sequence[int], order: Sequence[int] | None = None,
                  ) -> np.ndarray:
    """Batch of amplitudes (§6): eliminate every label except `open_labels`
    (bucket elimination along `order`, or the oracle's own min-degree order with the open labels
    excluded) and multiply the remaining tensors -- which hold open labels only -- into one
    tensor.  Returns the flat vector v[i], bit b of i = the value of open_labels[b]."""
    opened = list(open_labels)
    if order is None:
        order, _ = greedy_min_degree(tensors, exclude=opened)
    rest, scalar = partial_eliminate(tensors, order)
    a = len(opened)
    # rest tensors hold open labels only: one einsum over them (a library primitive), axes in
    # the order opened[a-1] .. opened[0] so that the C-order flattening has bit b = opened[b]
    local = {lab: i for i, lab in enumerate(opened)}
    args = []
    for arr, labs in rest:
        if any(l not in local for l in labs):
            raise ValueError("order misses live labels")
        args.append(arr)
        args.append([local[l] for l in labs])
    args.append([local[l] for l in reversed(opened)])
    if rest:
        out = np.einsum(*args, optimize=False)
    else:
        out = np.ones((2,) * a, dtype=np.complex128)
    # an open label held by no remaining tensor (cannot happen for a connected network)
    return (np.asarray(out, dtype=np.complex128) * scalar).reshape(-1)


def pairwise_sum(vals: Sequence[complex]) -> complex:
    """Fixed-order pairwise tree over the list index."""
    vals = list(vals)
    if not vals:
        return complex(0.0)
    while len(vals) > 1:
        nxt = [vals[i] + vals[i + 1] for i in range(0, len(vals) - 1, 2)]
        if len(vals) % 2:
            nxt.append(vals[-1])
        vals = nxt
    return vals[0]


def slice_assignment(sliced: Sequence[int], j: int) -> Dict[int, int]:
    s = sorted(sliced)
    return {lab: (j >> b) & 1 for b, lab in enumerate(s)}


def contract_sliced(tensors: Sequence[Tensor], prefix: Sequence[int], sliced: Sequence[int],
                    residual: Sequence[int], slices: Iterable[int] | None = None,
                    return_parts: bool = False):
    """Step-dependent sliced contraction, Eq. (1) with a shared prefix."""
    rest, pscalar = partial_eliminate(tensors, prefix)
    k = len(sliced)
    js = range(1 << k) if slices is None else list(slices)
    parts = []
    for j in js:
        sl = fix_indices(rest, slice_assignment(sliced, j))
        parts.append(pscalar * bucket_eliminate(sl, residual))
    total = pairwise_sum(parts)
    return (total, parts) if return_parts else total


# ------------------------------------------------------------------ line graph + own greedy
def line_graph(tensors: Sequence[Tensor]) -> Dict[int, set]:
    """Vertices = indices, one clique per tensor."""
    adj: Dict[int, set] = {}
    for _, labs in tensors:
        for a in labs:
            adj.setdefault(a, set())
            for b in labs:
                if a != b:
                    adj[a].add(b)
    return adj


def eliminate_vertex(adj: Dict[int, set], v: int) -> None:
    """Remove v and make its neighbourhood a clique."""
    nb = adj.pop(v)
    for a in nb:
        adj[a].discard(v)
        adj[a].update(nb - {a})


def greedy_min_degree(tensors: Sequence[Tensor], exclude: Iterable[int] = ()) -> Tuple[List[int], List[int]]:
    """Eliminate a lowest-degree vertex, ties -> smallest label."""
    adj = line_graph(tensors)
    ex = set(exclude)
    order, degs = [], []
    while True:
        cand = [v for v in adj if v not in ex]
        if not cand:
            break
        v = min(cand, key=lambda x: (len(adj[x]), x))
        degs.append(len(adj[v]))
        order.append(v)
        eliminate_vertex(adj, v)
    return order, degs


def width_of_order(tensors: Sequence[Tensor], order: Sequence[int]) -> List[int]:
    adj = line_graph(tensors)
    degs = []
    for v in order:
        degs.append(len(adj[v]))
        eliminate_vertex(adj, v)
    return degs


def contract(tensors: Sequence[Tensor], order: Sequence[int] | None = None) -> complex:
    """sigma by bucket elimination; own greedy min-degree order unless given."""
    if order is None:
        order, _ = greedy_min_degree(tensors)
    return bucket_eliminate(tensors, order)


def brute_force(tensors: Sequence[Tensor]) -> complex:
    """Sum over all assignments of all labels of the product (the plain definition;
    PAPER.md:214, 233-234).  Only for <= ~22 labels."""
    labs = sorted(set().union(*[set(l) for _, l in tensors])) if tensors else []
    if len(labs) > 52:
        raise ValueError("too many labels")
    local = {l: i for i, l in enumerate(labs)}
    args = []
    for arr, ls in tensors:
        args.append(arr)
        args.append([local[l] for l in ls])
    args.append([])
    return complex(np.einsum(*args, optimize=False))


# ------------------------------------------------------------------ sub-slicing (host RAM bound)
def subslice_labels(tensors: Sequence[Tensor], order: Sequence[int], max_width: int) -> List[int]:
    """Labels to fix in addition, so that bucket elimination of `tensors` along `order` (minus
    the fixed labels) has width <= max_width -- Eq. (1) applied once more, which is exact
    ("when host RAM is short it sub-slices further").
    Greedy, the oracle's own rule: while too wide, fix the label that occurs in the neighbourhoods
    of the widest steps with the largest total weight sum 2^degree (ties -> smaller label)."""
    extra: List[int] = []
    while True:
        fixed = fix_indices(tensors, {l: 0 for l in extra})
        adj = line_graph(fixed)
        steps = []
        for v in order:
            if v in extra or v not in adj:
                continue
            steps.append((len(adj[v]), set(adj[v])))
            eliminate_vertex(adj, v)
        w = max((d for d, _ in steps), default=0)
        if w <= max_width:
            return extra
        cnt: Dict[int, float] = {}
        for d, nb in steps:
            if d >= w - 1:
                for u in nb:
                    cnt[u] = cnt.get(u, 0.0) + 2.0 ** d
        extra.append(max(cnt, key=lambda u: (cnt[u], -u)))


def subslice_value(tensors: Sequence[Tensor], order: Sequence[int], extra: Sequence[int], i: int) -> complex:
    """Sub-slice i: the labels of `extra` fixed to the bits of i (bit b = b-th label ascending),
    then bucket elimination along `order` without them."""
    fixed = fix_indices(tensors, slice_assignment(extra, i))
    ex = set(extra)
    return bucket_eliminate(fixed, [l for l in order if l not in ex])


def contract_subsliced(tensors: Sequence[Tensor], order: Sequence[int], extra: Sequence[int],
                       workers: int = 1, ids: Sequence[int] | None = None) -> complex:
    """sum over the 2^m sub-slices (fixed pairwise tree over the sub-slice id), each evaluated by
    subslice_value -- in `workers` forked processes (independent sums; the value and its rounding
    do not depend on the worker count).  `ids`: a subset (the caller sums it)."""
    ids = list(range(1 << len(extra))) if ids is None else list(ids)
    return pairwise_sum(map_subslices(tensors, order, extra, ids, workers))


_POOL_STATE = None


def _pool_eval(i):
    t, o, e = _POOL_STATE
    return subslice_value(t, o, e, i)


def map_subslices(tensors, order, extra, ids, workers: int = 1) -> List[complex]:
    """[subslice_value(i) for i in ids], optionally over a fork-based process pool (the tensors are
    inherited by the workers, not pickled)."""
    global _POOL_STATE
    ids = list(ids)
    if workers <= 1 or len(ids) <= 1:
        return [subslice_value(tensors, order, extra, i) for i in ids]
    import multiprocessing as mp

    _POOL_STATE = (tensors, order, list(extra))
    try:
        with mp.get_context("fork").Pool(min(workers, len(ids))) as pool:
            return pool.map(_pool_eval, ids, chunksize=1)
    finally:
        _POOL_STATE = None


def _pool_slice_task(task):
    rest, sliced, residual, extra = _POOL_STATE
    j, i = task
    return subslice_value(fix_indices(rest, slice_assignment(sliced, j)), residual, extra, i)


def slice_values(tensors: Sequence[Tensor], prefix: Sequence[int], sliced: Sequence[int],
                 residual: Sequence[int], slices: Iterable[int], max_width: int | None = None,
                 workers: int = 1):
    """Per-slice results of Eq. (1) with a shared prefix (as contract_sliced), each slice
    optionally sub-sliced to max_width (subslice_labels on slice 0's network; every slice has the
    same structure) and the (slice, sub-slice) evaluations spread over `workers` forked processes.
    Returns (values in the order of `slices`, extra labels)."""
    global _POOL_STATE
    rest, pscalar = partial_eliminate(tensors, prefix)
    js = list(slices)
    extra: List[int] = []
    if max_width is not None and js:
        extra = subslice_labels(fix_indices(rest, slice_assignment(sliced, js[0])), residual, max_width)
    m = len(extra)
    tasks = [(j, i) for j in js for i in range(1 << m)]
    _POOL_STATE = (rest, list(sliced), list(residual), extra)
    try:
        if workers <= 1 or len(tasks) <= 1:
            flat = [_pool_slice_task(t) for t in tasks]
        else:
            import multiprocessing as mp

            with mp.get_context("fork").Pool(min(workers, len(tasks))) as pool:
                flat = pool.map(_pool_slice_task, tasks, chunksize=1)
    finally:
        _POOL_STATE = None
    vals = [pscalar * pairwise_sum(flat[a << m:(a + 1) << m]) for a in range(len(js))]
    return vals, extra
