"""Multi-GPU plumbing for the evaluation.

BASELINE.json north_star: "the candidate grid is sharded across the GPUs of one
8×B200 box, with NCCL over NVLink used only for the small allgather of
per-candidate scores and the global argmax".  Every (candidate, QPS, trace)
replay is independent, so one fixed grid is split across ranks (strong
scaling) with no data-path collective:

* n_qps >= world: QPS points are striped (q mod world == rank) — light and
  heavy load points alternate, and every (prefill group, QPS, trace) stage-A
  replay and all its decode candidates stay on one GPU;
* n_qps < world: contiguous candidate blocks, cut only between candidates of
  different prefill groups (the factorized path replays a group once);
* seeds (traces) are never split, so each Σ over traces — the FP64 goodput
  included — is formed on one rank in ascending trace order and the gathered
  results are byte-identical for any world size.

The one exchange: ``all_gather_into_tensor`` of each rank's met (int64) and
goodput (FP64) block, then the argmax kernel on the gathered met
(``Context.argmax_device``).  NCCL on GPUs, gloo for the CPU tests.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch
import torch.distributed as dist


@dataclass
class Shard:
    """This rank's part of the (candidate, QPS) grid: index arrays into the
    global candidate and QPS lists (every trace seed is included)."""
    cand: np.ndarray
    qps: np.ndarray
    mode: str            # "qps-stripe" or "cand-block"


def _group_keys(role: np.ndarray, cap: np.ndarray, static: np.ndarray) -> list:
    """Prefill group of each static candidate (its prefill caps in GPU-id order:
    the factorized path replays a group's prefill stage once); a dynamic
    candidate is a group of its own (it is replayed whole, in the joint kernel)."""
    return [tuple(int(w) for w, r in zip(cap[c], role[c]) if r == 0) if static[c] else ("dyn", c)
            for c in range(role.shape[0])]


def shard_grid(rank: int, world: int, role: np.ndarray, cap: np.ndarray, n_qps: int,
               static: np.ndarray | None = None, weight: np.ndarray | None = None) -> Shard:
    """Partition of the fixed (candidate × QPS) grid for ``rank`` of ``world``.
    ``static[c]``: candidate c is static (default all); ``weight[c]``: relative
    replay cost for balancing candidate blocks (default 1 static, 20 dynamic —
    a dynamic replay costs ~20x a static one per request)."""
    C = role.shape[0]
    if world <= 1:
        return Shard(np.arange(C), np.arange(n_qps), "qps-stripe")
    if n_qps >= world:
        return Shard(np.arange(C), np.arange(rank, n_qps, world), "qps-stripe")
    # candidate blocks: contiguous runs of whole prefill groups, balanced by weight
    st = np.ones(C, bool) if static is None else np.asarray(static, bool)
    w = np.where(st, 1.0, 20.0) if weight is None else np.asarray(weight, float)
    keys = _group_keys(role, cap, st)
    cuts = [0]
    for c in range(1, C):
        if keys[c] != keys[c - 1]:
            cuts.append(c)
    cuts.append(C)
    runs = [(cuts[k], cuts[k + 1]) for k in range(len(cuts) - 1)]
    total = w.sum()
    bounds = [0]
    acc = 0.0
    for a, b in runs:
        acc += w[a:b].sum()
        # close a block once this rank's share of the weight is reached
        if len(bounds) < world and acc >= total * len(bounds) / world:
            bounds.append(b)
    while len(bounds) < world:
        bounds.append(C)
    bounds.append(C)
    lo, hi = bounds[rank], bounds[rank + 1]
    return Shard(np.arange(lo, hi), np.arange(n_qps), "cand-block")


def gather_results(met: torch.Tensor, good: torch.Tensor, shards: list[Shard], n_cand: int, n_qps: int,
                   group=None) -> tuple[torch.Tensor, torch.Tensor]:
    """Gather met (int64) and goodput (FP64) blocks of every rank into global
    [n_cand, n_qps] arrays; ``shards`` = the Shard of every rank (same rule on
    every rank, so no index exchange is needed)."""
    world = len(shards)
    outs = []
    for local in (met, good):
        full = torch.zeros((n_cand, n_qps), dtype=local.dtype, device=local.device)
        if world <= 1:
            allb = local.reshape(1, -1)
        else:
            # gloo (CPU tests, the one-GPU multi-rank check) exchanges host tensors
            cdev = torch.device("cpu") if dist.get_backend(group) == "gloo" else local.device
            cap_n = max(len(s.cand) * len(s.qps) for s in shards)
            buf = torch.zeros(cap_n, dtype=local.dtype, device=cdev)
            buf[: local.numel()] = local.reshape(-1).to(cdev)
            allb = torch.zeros(world * cap_n, dtype=local.dtype, device=cdev)
            dist.all_gather_into_tensor(allb, buf, group=group)
            allb = allb.view(world, cap_n).to(local.device)
        for r, s in enumerate(shards):
            n = len(s.cand) * len(s.qps)
            if n:
                ci = torch.as_tensor(s.cand, device=local.device)
                qi = torch.as_tensor(s.qps, device=local.device)
                full[ci[:, None], qi[None, :]] = allb[r, :n].view(len(s.cand), len(s.qps))
        outs.append(full)
    return outs[0], outs[1]


def all_shards(world: int, role: np.ndarray, cap: np.ndarray, n_qps: int, static=None,
               weight=None) -> list[Shard]:
    return [shard_grid(r, world, role, cap, n_qps, static, weight) for r in range(world)]


def max_over_ranks(x: float, device=None, group=None) -> float:
    """Max of a host scalar over ranks (timing: the slowest rank defines the step)."""
    if not (dist.is_initialized() and dist.get_world_size(group) > 1):
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())


def evaluate_sharded(traces, qps, model, role, cap, policies, slo, budget_w, ctx=None, device=0,
                     cand_budget_w=None, group=None):
    """North-star multi-GPU evaluation through the public API: this rank
    evaluates its shard of the grid with padsim_evaluate_allocations (host
    buffers in and out), the met / goodput blocks are all-gathered (NCCL on
    CUDA tensors) and the argmax kernel runs on the gathered met.  Every rank
    returns the same global {met, goodput, argmax}; with one process it is
    exactly padsim_evaluate_allocations."""
    from .binding import Context, evaluate_allocations
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    role = np.asarray(role)
    cap = np.asarray(cap)
    C, Q = role.shape[0], len(qps)
    static = np.array([p["kind"] == 0 for p in policies])
    shards = all_shards(world, role, cap, Q, static)
    sh = shards[rank]
    own = ctx is None
    ctx = ctx or Context(device)
    try:
        dev = torch.device("cuda", device)
        if len(sh.cand) and len(sh.qps):
            cb = None if cand_budget_w is None else np.asarray(cand_budget_w)[sh.cand]
            out = evaluate_allocations(traces, [qps[q] for q in sh.qps], model, role[sh.cand], cap[sh.cand],
                                       [policies[c] for c in sh.cand], slo, budget_w, ctx=ctx, cand_budget_w=cb)
            if world == 1:          # one process: the call's own results (no exchange to do)
                return {"met": out["met"], "goodput": out["goodput"], "argmax": out["argmax"]}
            met_l = torch.as_tensor(out["met"]).to(dev)
            good_l = torch.as_tensor(out["goodput"]).to(dev)
        else:
            met_l = torch.zeros(0, dtype=torch.int64, device=dev)
            good_l = torch.zeros(0, dtype=torch.float64, device=dev)
        met, good = gather_results(met_l, good_l, shards, C, Q, group)
        capsum = torch.as_tensor(cap.sum(axis=1).astype(np.int32)).to(dev)
        am = torch.empty(Q, dtype=torch.int32, device=dev)
        met = met.contiguous()
        ctx.argmax_device(met.data_ptr(), C, Q, am.data_ptr(), torch.cuda.current_stream(dev).cuda_stream,
                          d_capsum_ptr=capsum.data_ptr())
        return {"met": met.cpu().numpy(), "goodput": good.cpu().numpy(), "argmax": am.cpu().numpy()}
    finally:
        if own:
            ctx.close()
