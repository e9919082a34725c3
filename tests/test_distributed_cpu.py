"""Multi-process (gloo, CPU, world 2 and 4) test of the product's north-star
sharding (paper_2601_12241_b200/distributed.py): one fixed
(candidate × QPS × seed) grid is split across ranks — QPS striped when
n_qps >= world, whole-prefill-group candidate blocks otherwise, seeds never
split — and the per-rank met (int64) / goodput (FP64) blocks are all-gathered.
The gathered arrays must be byte-identical to a single-process evaluation of
the whole grid, and so must the argmax over them.  The per-rank compute
stand-in is the CPU oracle (tests may call it; the product never does)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from workloads import DEFAULT_MODEL, DEFAULT_SLO, PHASE_SLO, make_trace, policy, static_candidates

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


def _case(name):
    if name == "qps-stripe":            # cfg 2/4 shape: n_qps >= world
        xpd = [(2, 700, 550), (3, 675, 525), (4, 600, 600), (4, 750, 450), (5, 600, 600), (6, 500, 650)]
        role, cap = static_candidates(8, xpd)
        pols = [policy("static")] * len(xpd)
        return role, cap, pols, [make_trace("lb", s, R) for s in range(3)], [0.5, 1.0, 1.5, 2.0, 2.5], DEFAULT_SLO
    # cfg 1/3 shape: n_qps < world -> candidate blocks (static groups kept whole, dynamic cut anywhere)
    xpd = [(4, 600, 600), (4, 600, 550), (4, 700, 500), (4, 700, 450), (5, 600, 600)] + [(4, 600, 600)] * 4
    role, cap = static_candidates(8, xpd)
    pols = [policy("static")] * 5 + [policy("dyn-power", cooldown_s=2.0), policy("dyn-gpu"),
                                     policy("dyn-both", window_s=2.5), policy("dyn-both", step_w=100)]
    return role, cap, pols, [make_trace("phase", s, 300) for s in range(2)], [1.5], PHASE_SLO


def _worker(rank, world, port, case, outq):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    from paper_2601_12241_b200.distributed import all_shards, gather_results, max_over_ranks
    role, cap, pols, traces, qps, slo = _case(case)
    C, Q = role.shape[0], len(qps)
    static = np.array([p["kind"] == 0 for p in pols])
    shards = all_shards(world, role, cap, Q, static)
    sh = shards[rank]
    if len(sh.cand):
        ev = oracle.evaluate(DEFAULT_MODEL, role[sh.cand], cap[sh.cand], [pols[c] for c in sh.cand], 4800, slo,
                             traces, [qps[q] for q in sh.qps])
        met_l, good_l = torch.from_numpy(ev["met"].copy()), torch.from_numpy(ev["goodput"].copy())
    else:
        met_l, good_l = torch.zeros(0, dtype=torch.int64), torch.zeros(0, dtype=torch.float64)
    met, good = gather_results(met_l, good_l, shards, C, Q)
    t = max_over_ranks(float(rank + 1))
    outq.put((rank, met.numpy(), good.numpy(), t, [(list(s.cand), list(s.qps), s.mode) for s in shards]))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("case", ["qps-stripe", "cand-block"])
@pytest.mark.parametrize("world", [2, 4])
def test_sharded_grid_matches_single_process(world, case):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, case, q)) for r in range(world)]
    for p in procs:
        p.start()
    outs = [q.get(timeout=600) for _ in range(world)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    import oracle
    role, cap, pols, traces, qps, slo = _case(case)
    ref = oracle.evaluate(DEFAULT_MODEL, role, cap, pols, 4800, slo, traces, qps)
    shards = outs[0][4]
    # every (candidate, QPS) cell is owned by exactly one rank; seeds are never split
    owned = np.zeros((role.shape[0], len(qps)), int)
    for cand, qq, mode in shards:
        owned[np.ix_(cand, qq)] += 1
        assert mode == case
    assert (owned == 1).all()
    for rank, met, good, tmax, _ in outs:          # every rank holds the same global arrays
        assert np.array_equal(met, ref["met"])
        assert np.array_equal(good, ref["goodput"])       # byte-identical FP64 (one rank per Σ)
        assert _argmax(met, cap.sum(axis=1)) == list(ref["argmax"])
        assert tmax == float(world)


def test_candidate_blocks_keep_prefill_groups_whole():
    from paper_2601_12241_b200.distributed import all_shards
    role, cap = static_candidates(8, [(x, p, d) for x in (2, 4) for p in (500, 600) for d in (400, 450, 500)])
    for world in (2, 3, 4, 8):
        shards = all_shards(world, role, cap, 1)
        seen = {}
        for r, s in enumerate(shards):
            for c in s.cand:
                key = tuple(cap[c][role[c] == 0])
                assert seen.setdefault(key, r) == r          # a prefill group on one rank only
        assert sum(len(s.cand) for s in shards) == role.shape[0]
