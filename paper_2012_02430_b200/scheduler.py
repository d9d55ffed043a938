"""Slice scheduler: one process per GPU (torch.distributed), Eq. (1)'s 2^k slices split into
contiguous blocks, one all-reduce of the per-slice partials, fixed-order sum.

PAPER.md:519-524 (Eq. 1): the sliced networks are independent; their results are summed.
PAPER.md:650-651: the steps before the slice step s are contracted first -- here every rank
recomputes that (cheap) prefix instead of broadcasting it (SURVEY.md §8 e).
The collective is a single all_reduce(SUM) over a zero-padded float64 vector of 2*2^k values;
adding zeros is exact, so the fixed pairwise sum (tn_sum_partials) is bit-identical for any
number of ranks.
"""
from __future__ import annotations

from typing import Callable, Optional, Tuple


def slice_block(n_slices: int, rank: int, world: int) -> Tuple[int, int]:
    """Contiguous block [begin, end) of rank `rank` out of `world` (balanced to +-1)."""
    if world <= 0 or not (0 <= rank < world):
        raise ValueError("bad rank/world")
    return (rank * n_slices) // world, ((rank + 1) * n_slices) // world


def run_sliced(plan, gammas, betas, dtype: int = 0, group=None, device=None,
               compute: Optional[Callable] = None, stream=None):
    """Whole-job sliced amplitude; returns (sigma, partials_host).

    compute(begin, end, partials) fills partials[2(j A + x) : 2(j A + x) + 2] for j in [begin, end)
    and batch entries x < A = plan.batch (A = 1: a single amplitude); the default is
    the CUDA path (tn_contract_sliced).  Tests on CPU inject their own compute (gloo backend).
    """
    import torch
    import torch.distributed as dist

    n = plan.n_slices
    if dist.is_available() and dist.is_initialized():
        rank, world = dist.get_rank(group), dist.get_world_size(group)
    else:
        rank, world = 0, 1
    begin, end = slice_block(n, rank, world)
    if compute is None:
        dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
        cur = torch.cuda.current_stream(dev)
        s = cur if stream is None else stream
        if s != cur:
            s.wait_stream(cur)          # inputs / earlier work of the caller's stream come first
        with torch.cuda.stream(s):      # zero-fill and contraction on the same stream
            partials = torch.zeros(2 * n * getattr(plan, "batch", 1), dtype=torch.float64, device=dev)
            if end > begin:
                plan.contract_sliced(gammas, betas, begin, end, partials, dtype=dtype, stream=s)
        if s != cur:
            cur.wait_stream(s)          # the all-reduce and the host copy run on the current stream
            partials.record_stream(cur)
    else:
        dev = torch.device("cpu") if device is None else torch.device(device)
        partials = torch.zeros(2 * n * getattr(plan, "batch", 1), dtype=torch.float64, device=dev)
        if end > begin:
            compute(begin, end, partials)
    if world > 1:
        dist.all_reduce(partials, op=dist.ReduceOp.SUM, group=group)
    host = partials.cpu()
    return plan.sum_partials(host.tolist()), host
