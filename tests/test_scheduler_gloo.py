"""Multi-rank slice scheduler on CPU (gloo, world_size 2): the partition, the single all-reduce
and the fixed-order sum give a result bit-identical to world_size 1.  The per-slice compute is
injected (the oracle, test infrastructure) since this host has no GPU."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2012_02430_b200.scheduler import run_sliced, slice_block


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _instance():
    import paper_2012_02430_b200 as T
    from tn_inputs import qaoa_angles, random_regular_graph

    g = random_regular_graph(30, 3, 4)
    ga, be = qaoa_angles(1, 4)
    plan = T.build_plan(g, 1, "amplitude", "min-fill", n_sliced=3)
    return plan, g, ga, be


def _oracle_compute(plan, g, ga, be):
    from oracle import contract, network

    pre, sl, res, _ = plan.schedule()
    tens = network.qaoa_amplitude_network(g.n, g.edges, ga, be)

    def compute(begin, end, partials):
        _, parts = contract.contract_sliced(tens, pre, sl, res, slices=range(begin, end), return_parts=True)
        for j, v in zip(range(begin, end), parts):
            partials[2 * j] = v.real * 1.0
            partials[2 * j + 1] = v.imag * 1.0
    return compute


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    plan, g, ga, be = _instance()
    sigma, host = run_sliced(plan, ga, be, compute=_oracle_compute(plan, g, ga, be))
    q.put((rank, sigma, host.tolist()))
    dist.destroy_process_group()


def test_slice_block_partition():
    for n in (1, 8, 64, 4096):
        for w in (1, 2, 3, 4, 8):
            blocks = [slice_block(n, r, w) for r in range(w)]
            assert blocks[0][0] == 0 and blocks[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(blocks, blocks[1:]))
            assert max(b - a for a, b in blocks) - min(b - a for a, b in blocks) <= 1


def test_two_rank_gloo_matches_single_rank():
    from oracle import contract, network

    plan, g, ga, be = _instance()
    ref1, host1 = run_sliced(plan, ga, be, compute=_oracle_compute(plan, g, ga, be))
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, sigma, host in res:
        assert sigma == ref1                      # bit-identical for any world size
        assert host == host1.tolist()
    unsliced = contract.contract(network.qaoa_amplitude_network(g.n, g.edges, ga, be))
    assert abs(ref1 - unsliced) < 1e-12 * max(1.0, abs(unsliced)) + 1e-15
