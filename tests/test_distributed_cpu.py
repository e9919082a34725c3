"""Multi-process (world_size 2, gloo, CPU) test of the sharding + exchange logic
of DESIGN.md §6: ranks evaluate disjoint seed blocks, the int64 met counts are
all-reduced, goodput summed in rank order, and the argmax over the reduced
counts equals a single-process evaluation over all seeds.  The per-rank
compute stand-in is the CPU oracle (tests may call it; the product never does)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from workloads import DEFAULT_MODEL, DEFAULT_SLO, make_trace, policy, static_candidates

XPD = [(2, 700, 550), (3, 675, 525), (4, 600, 600), (4, 750, 450), (5, 600, 600), (6, 500, 650)]
QPS = [0.5, 1.5, 2.5]
S_PER_RANK = 2
R = 150


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _argmax(met, capsum):
    out = []
    for q in range(met.shape[1]):
        key = np.lexsort((np.arange(met.shape[0]), capsum, -met[:, q]))
        out.append(int(key[0]))
    return out


def _worker(rank, world, port, outq):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    from paper_2601_12241_b200.distributed import (allreduce_met, max_over_ranks, rank_seeds,
                                                   sum_goodput_rank_order)
    role, cap = static_candidates(8, XPD)
    pols = [policy("static")] * len(XPD)
    traces = [make_trace("lb", s, R) for s in rank_seeds(rank, S_PER_RANK)]
    ev = oracle.evaluate(DEFAULT_MODEL, role, cap, pols, 4800, DEFAULT_SLO, traces, QPS)
    met = allreduce_met(torch.from_numpy(ev["met"].ravel().copy()))
    good = sum_goodput_rank_order(torch.from_numpy(ev["goodput"].ravel().copy()))
    t = max_over_ranks(float(rank + 1))
    if rank == 0:
        outq.put((met.numpy().reshape(len(XPD), len(QPS)), good.numpy().reshape(len(XPD), len(QPS)), t))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_sharded_argmax_matches_single_process(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    met, good, tmax = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    import oracle
    role, cap = static_candidates(8, XPD)
    pols = [policy("static")] * len(XPD)
    traces = [make_trace("lb", s, R) for s in range(world * S_PER_RANK)]
    ref = oracle.evaluate(DEFAULT_MODEL, role, cap, pols, 4800, DEFAULT_SLO, traces, QPS)
    assert np.array_equal(met, ref["met"])
    assert _argmax(met, cap.sum(axis=1)) == list(ref["argmax"])
    # rank-order goodput sum equals the per-rank partial sums added in order
    assert np.allclose(good, ref["goodput"], rtol=1e-12, atol=0)
    assert tmax == float(world)
