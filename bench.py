#!/usr/bin/env python
"""Benchmark: batched what-if evaluation (BASELINE.json metric) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg2] [--impl padsim|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...        (one rank per GPU, NCCL)

One *step* is one pass of the whole hot path (rows a1–a8 of SURVEY.md §8): every
candidate allocation × every QPS point × every trace is replayed (static and
dynamic kernels), reduced over traces and argmax-ed per QPS.  With N > 1 ranks
the fixed grid is sharded (strong scaling): QPS points striped
q mod N when n_qps ≥ N, else blocks of candidates; seeds are never split.  The
ranks' met / goodput blocks are all-gathered over NCCL and the global argmax
taken on the gathered array; ``value`` is the whole grid ÷ the max over ranks
of the device time.

``value`` times padsim_run with inputs resident in HBM (CUDA events on the
launch stream, L2 flushed between steps by a 512 MiB write).  ``e2e`` times the
public one-shot C-ABI call padsim_evaluate_allocations with host buffers (H2D
of traces + candidates, D2H of the results inside the timed region).
``cpu_baseline`` is the CPU oracle (oracle/, plain C DES) on a bounded,
deterministic sample of the same workload on this host's cores.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from workloads import (DEFAULT_MODEL, get_config, make_trace, policy,  # noqa: E402
                       static_candidates)
from workloads.configs import dynamic_candidates  # noqa: E402

PEAKS_PATH = os.path.join(ROOT, "MEASURED_PEAKS.json")
MICRO_PEAKS_PATH = os.path.join(ROOT, "profiles", "peaks_r02.json")   # tools/peaks_microbench.cu
TRAFFIC_PATH = os.path.join(ROOT, "profiles", "ncu_traffic.json")   # dram bytes/launch per kernel
# Algorithmic FP64 operations per simulated request: stage A —
# arrival scale (1 mul), its share of the prefill batch latency (1 div), TTFT
# (1 sub), transfer end (1 add) = 4; stage C — two segment boundaries (2 x (mul +
# add)), TPOT (sub + div), two SLO compares = 8; the joint replay does both = 12.
FP64_OPS_PER_REQ = {"stageA_kernel": 4, "stageC_kernel": 8, "joint_kernel": 12,
                    "stageA_wide_kernel": 4, "stageC_wide_kernel": 8}
WARP_INSTR_BUDGET = 15      # warp-instructions per simulated request (8-lane groups)


def build_workload(cfg: dict, rank: int = 0, enumerate_fn=None):
    """Candidates (role, cap, policies, per-candidate budgets), traces, qps.
    Every rank builds the same fixed grid (the shard is cut from it)."""
    N, B = cfg["n_gpus"], cfg["budget_w"]
    rows, pols, buds = [], [], []
    if cfg.get("space"):
        sp = cfg["space"]
        xpd = enumerate_fn(N, B, DEFAULT_MODEL["min_w"], DEFAULT_MODEL["max_w"], sp["step_w"])
        if sp.get("x_only"):
            xpd = xpd[xpd[:, 0] == sp["x_only"]]
        rows += [tuple(r) for r in xpd]
        pols += [policy("static")] * len(xpd)
        buds += [B] * len(xpd)
    for st in cfg.get("statics", []):
        rows.append(tuple(st[:3]))
        pols.append(policy("static"))
        buds.append(st[3] if len(st) > 3 else B)     # e.g. 4P4D-750 W at 6000 W
    for x, p, d, pol in dynamic_candidates(cfg):
        rows.append((x, p, d))
        pols.append(pol)
        buds.append(B)
    role, cap = static_candidates(N, rows)
    fams = cfg["family"] if isinstance(cfg["family"], tuple) else (cfg["family"],)
    S = cfg["seeds"]
    traces = [make_trace(f, s, cfg["n_req"]) for f in fams for s in range(S)]
    cb = np.asarray(buds, np.int32)
    return role, cap, pols, traces, list(cfg["qps"]), (None if (cb == B).all() else cb)


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self._stop = threading.Event()
        self._t = None

    def __enter__(self):
        def loop():
            while not self._stop.is_set():
                try:
                    out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits"], capture_output=True,
                                         text=True, timeout=5).stdout.strip()
                    if out:
                        self.rows.append([x.strip() for x in out.split(",")])
                except Exception:
                    pass
                self._stop.wait(0.2)
        self._t = threading.Thread(target=loop, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join(timeout=6)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in self.rows for k in range(4)
                          if len(r) > 3 + k and r[3 + k].lower().startswith("active")})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons, "samples": len(self.rows)}


def ncu_traffic(workload: str, kernel: str):
    """dram__bytes_read.sum + dram__bytes_write.sum of one launch of `kernel` on
    `workload`, from the committed ncu --set full capture (profiles/), or None."""
    try:
        return json.load(open(TRAFFIC_PATH)).get(workload, {}).get(kernel, {}).get("bytes")
    except Exception:
        return None


def ncu_field(workload: str, kernel: str, key: str):
    try:
        return json.load(open(TRAFFIC_PATH)).get(workload, {}).get(kernel, {}).get(key)
    except Exception:
        return None


def peaks():
    try:
        return json.load(open(PEAKS_PATH))
    except Exception:
        return {}


def cpu_baseline(cfg, role, cap, pols, traces, qps, cand_budget=None, seconds=15.0, gpu_rep=None):
    """The oracle as it stands on a bounded deterministic sample of the workload
    (host cores, then one thread).  With ``gpu_rep`` (the GPU's per-replay
    met / goodput / duration of the same grid) the sampled replays double as a
    parity check of the timed launch configuration: mismatches are counted."""
    import oracle
    cores = os.cpu_count() or 1
    C, Q, S = role.shape[0], len(qps), len(traces)
    total = C * Q * S
    B = cfg["budget_w"]

    def run(cs, q, nt):
        return oracle.evaluate(DEFAULT_MODEL, role[cs], cap[cs], [pols[i] for i in cs], B, cfg["slo"],
                               traces[:1], [qps[q]], n_threads=nt, per_replay=True,
                               cand_budget_w=None if cand_budget is None else cand_budget[cs])
    t0 = time.perf_counter()
    run(np.arange(min(2, C)), Q // 2, 1)
    per = max((time.perf_counter() - t0) / min(2, C), 1e-4)
    n_pairs = int(max(cores, min(C * Q, seconds * cores / per)))
    stride = max(1, (C * Q) // n_pairs)
    sel = set(range(0, C * Q, stride)[:n_pairs])
    # every dynamic candidate appears at least once (at QPS index c mod Q)
    sel |= {c * Q + c % Q for c in range(C) if pols[c]["kind"] != 0}
    sel = np.array(sorted(sel))
    cs_all, qs_all = sel // Q, sel % Q
    reps, mism = 0, 0
    t0 = time.perf_counter()
    for q in np.unique(qs_all):          # one evaluate() per QPS point uses all host threads
        cs = cs_all[qs_all == q]
        ev = run(cs, int(q), cores)
        reps += len(cs)
        if gpu_rep is not None:
            g_met = gpu_rep["met"][cs, q, 0]
            g_good = gpu_rep["goodput"][cs, q, 0]
            g_dur = gpu_rep["duration"][cs, q, 0]
            mism += int(((ev["rep_met"][:, 0, 0] != g_met) | (ev["rep_goodput"][:, 0, 0] != g_good) |
                         (ev["rep_duration"][:, 0, 0] != g_dur)).sum())
    dt = time.perf_counter() - t0
    # one host thread on a small slice of the same sample
    n1 = max(1, min(len(sel), int(max(1.0, seconds / 4) / per)))
    t1 = time.perf_counter()
    for k in sel[:: max(1, len(sel) // n1)][:n1]:
        run(np.array([k // Q]), int(k % Q), 1)
    dt1 = time.perf_counter() - t1
    R = traces[0]["s_unit"].size
    out = {"value": reps / dt, "unit": "evals/s", "cores": cores, "kind": "oracle",
           "sample": f"{reps} of {total} replays (every {stride}th (candidate,QPS) pair + every dynamic "
                     f"candidate once, trace seed 0), {dt:.1f} s on {cores} threads",
           "req_per_s": reps * R / dt,
           "one_thread": {"value": n1 / dt1, "unit": "evals/s", "cores": 1,
                          "sample": f"{n1} replays of the same sample, {dt1:.1f} s"}}
    if gpu_rep is not None:
        out["parity"] = {"replays": reps, "mismatches": mism,
                         "compared": "per-replay met, goodput, duration (exact) vs the timed GPU run"}
    return out


def run_reference(args, cfg, rank, world):
    """--impl reference: the CPU oracle as it stands, bounded sample per step."""
    if rank != 0:
        return
    import oracle                       # the reference arm is the oracle alone
    role, cap, pols, traces, qps, cb = build_workload(cfg, 0, oracle.enumerate_pool_uniform)
    vals = []
    last = None
    for k in range(args.warmup + args.steps):
        cb_ = cpu_baseline(cfg, role, cap, pols, traces, qps, cb, seconds=max(2.0, 20.0 / max(1, args.steps)))
        if k >= args.warmup:
            vals.append(cb_["value"])
            last = cb_
    v = float(np.mean(vals))
    R = traces[0]["s_unit"].size
    line = {"impl": "reference", "metric": "candidate-trace evaluations/sec", "value": v,
            "unit": "evals/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": None, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic",
            "config": {"workload": cfg["name"], "sample": last["sample"]},
            "cpu_baseline": dict(last, value=v),
            "e2e": {"value": v, "unit": "evals/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "sim_req_per_s": v * R}
    print(json.dumps(line), flush=True)


def micro_peaks():
    try:
        return json.load(open(MICRO_PEAKS_PATH))
    except Exception:
        return {}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="cfg4")
    ap.add_argument("--impl", default="padsim", choices=["padsim", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--backend", default="nccl", choices=["nccl", "gloo"],
                    help="process-group backend (gloo only to exercise the multi-rank path on one GPU)")
    ap.add_argument("--same-device", action="store_true",
                    help="all ranks on cuda:0 (multi-rank logic check on a 1-GPU box; not a scaling run)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    cfg = get_config(args.config)

    if args.impl == "reference":
        run_reference(args, cfg, rank, world)
        return

    import torch
    import torch.distributed as dist
    import paper_2601_12241_b200 as pkg
    from paper_2601_12241_b200.build import build
    from paper_2601_12241_b200.distributed import (all_shards, evaluate_sharded, gather_results,
                                                   max_over_ranks)
    if rank == 0:
        build()
    local_dev = 0 if args.same_device else local
    if world > 1:
        torch.cuda.set_device(local_dev)
        if args.backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_dev))
        else:
            dist.init_process_group("gloo")
        dist.barrier()
        build()     # no-op if rank 0 built it
    local = local_dev
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    stream = torch.cuda.current_stream(dev)

    # the fixed grid (BASELINE config) and this rank's shard of it
    role, cap, pols, traces, qps, cand_budget = build_workload(cfg, rank, pkg.enumerate_pool_uniform)
    C, Q, S = role.shape[0], len(qps), len(traces)
    R = traces[0]["s_unit"].size
    static = np.array([p["kind"] == 0 for p in pols])
    shards = all_shards(world, role, cap, Q, static)
    sh = shards[rank]
    Cl, Ql = len(sh.cand), len(sh.qps)
    ctx = pkg.Context(local, stream.cuda_stream)
    ctx.plan(traces, [qps[q] for q in sh.qps], DEFAULT_MODEL, role[sh.cand], cap[sh.cand],
             [pols[c] for c in sh.cand], cfg["slo"], cfg["budget_w"],
             cand_budget_w=None if cand_budget is None else cand_budget[sh.cand])
    d = ctx.device_results()

    def as_tensor(ptr, n, dtype, typestr):
        class _A:
            __cuda_array_interface__ = {"shape": (n,), "typestr": typestr, "data": (ptr, False),
                                        "version": 3, "strides": None}
        return torch.as_tensor(_A(), device=dev).view(dtype)

    met_dev = as_tensor(d.d_met, Cl * Ql, torch.int64, "<i8")
    good_dev = as_tensor(d.d_goodput, Cl * Ql, torch.float64, "<f8")
    capsum = torch.as_tensor(cap.sum(axis=1).astype(np.int32)).to(dev)
    am_glob = torch.empty(Q, dtype=torch.int32, device=dev)
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)

    def step():
        ctx.run(stream.cuda_stream)
        n = ctx.launch_count()
        if world > 1:      # the one exchange: allgather of the scores, then the global argmax
            met_g, _good_g = gather_results(met_dev, good_dev, shards, C, Q)
            ctx.argmax_device(met_g.data_ptr(), C, Q, am_glob.data_ptr(), stream.cuda_stream,
                              d_capsum_ptr=capsum.data_ptr())
            n += 1
        return n

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    launches = 0
    times = []
    kern_ms = []
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            flush.fill_(1.0)                       # L2 flush between timed steps (not timed)
            if world > 1:
                dist.barrier()
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            launches = step()
            e1.record(stream)
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1))
            kern_ms.append(ctx.kernel_times_ms())
    t_local = sum(times) / 1e3
    t_max = max_over_ranks(t_local, device=dev)
    units = C * Q * S                       # the whole fixed grid, over all ranks (strong scaling)
    value = units * args.steps / t_max
    ev_rep = as_tensor(d.d_rep_events, Cl * Ql * S, torch.int64, "<i8").view(Cl, Ql, S)
    is_dyn = torch.tensor([pols[c]["kind"] != 0 for c in sh.cand], device=dev)
    ev_static = int(ev_rep[~is_dyn].sum().item()) if Cl else 0
    ev_dyn = int(ev_rep[is_dyn].sum().item()) if Cl else 0
    ev_a = int(as_tensor(d.d_aux_events, d.n_aux_events, torch.int64, "<i8").sum().item()) \
        if d.n_aux_events > 0 else 0     # stage A instants (factorized static paths)
    if ev_a == 0:            # static replays ran in the joint kernel
        ev_dyn += ev_static
        ev_static = 0
    wide = ctx.static_path() == "warp"        # the warp-per-replay factorized stages
    # per-rank replay results of the timed configuration (for the parity sample)
    rep = ctx.fetch_replays()

    # per-kernel device times in isolation (kernels serialised on one stream; not the
    # timed region): the roofline's kernel time
    ctx.set_tuning({"serialize": 1})
    iso = []
    for k in range(4):
        flush.fill_(1.0)
        torch.cuda.synchronize()
        ctx.run(stream.cuda_stream)
        torch.cuda.synchronize()
        if k:
            iso.append(ctx.kernel_times_ms())
    ctx.set_tuning(None)
    iso = np.mean(np.array(iso), axis=0)

    r_sum = sum(int(t["s_unit"].size) for t in traces)
    static_idx = [c for c in sh.cand if pols[c]["kind"] == 0]
    groups = {tuple(int(v) for v in cap[c][role[c] == 0]) for c in static_idx}
    fact = ev_a > 0                       # a factorized static path ran (N <= 8, or wide N <= 64)
    req_k = {"stageA_kernel": len(groups) * Ql * r_sum if fact else 0,
             "stageC_kernel": len(static_idx) * Ql * r_sum if fact else 0,
             "joint_kernel": (Cl - len(static_idx) + (0 if fact else len(static_idx))) * Ql * r_sum}
    req_k["stageA_wide_kernel"] = req_k["stageA_kernel"]
    req_k["stageC_wide_kernel"] = req_k["stageC_kernel"]

    # e2e: the public API with host buffers (evaluate_sharded = padsim_evaluate_allocations on
    # this rank's shard + allgather + argmax; one process: exactly padsim_evaluate_allocations)
    e2e_times = []
    h2d = sum(t["s_unit"].nbytes + 4 * t["in_tok"].size * 2 + t["s_unit"].size for t in traces)
    h2d += Cl * (role.shape[1] * 5 + 48) + 8 * Ql
    d2h = Cl * Ql * 24 + Ql * 4 + (C * Q * 16 + Q * 4 if world > 1 else 0)
    for k in range(args.e2e_steps + 1 if args.e2e_steps > 0 else 0):
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        out = evaluate_sharded(traces, qps, DEFAULT_MODEL, role, cap, pols, cfg["slo"], cfg["budget_w"],
                               ctx=ctx, device=local, cand_budget_w=cand_budget)
        if k > 0:
            e2e_times.append(time.perf_counter() - t0)
    # median over the e2e steps (host wall clock includes OS / driver jitter), max over ranks
    e2e_t = max_over_ranks(float(np.median(e2e_times)) if e2e_times else float("nan"), device=dev)
    del out

    if rank == 0:
        pk = peaks()
        mp_ = micro_peaks()
        clocks = clk.summary()
        km = np.mean(np.array(kern_ms), axis=0) if kern_ms else np.zeros(3)
        names = (["stageA_wide_kernel", "stageC_wide_kernel", "joint_kernel"] if wide
                 else ["stageA_kernel", "stageC_kernel", "joint_kernel"])
        evs = [ev_a, ev_static, ev_dyn]
        # dominant kernel = the one with the most isolated device time
        dom = int(np.argmax(iso))
        fp64_ops = req_k[names[dom]] * FP64_OPS_PER_REQ[names[dom]]
        achieved = fp64_ops / (iso[dom] / 1e3) / 1e12 if iso[dom] > 0 else float("nan")
        peak_fp64 = (mp_.get("_derived", {}).get("fp64_pipe_ops_per_s") or 148 * 64 * 1965e6) / 1e12
        wipr = ncu_field(cfg["name"], names[dom], "warp_instr_per_request")
        cfg4 = get_config("cfg4")
        cfg4_replays = (955 + 21) * len(cfg4["qps"]) * cfg4["seeds"]
        line = {
            "metric": "candidate-trace evaluations/sec", "value": value, "unit": "evals/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": t_max / args.steps * 1e3, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": cfg["name"], "n_cand": C, "n_qps": Q, "n_traces": S, "n_req": R,
                       "replays": units, "family": cfg["family"], "shard": sh.mode,
                       "replays_rank0": Cl * Ql * S, "l2": "flushed between steps (512 MiB write)"},
            "sim_req_per_s": value * r_sum / S,
            "e2e": {"value": units / e2e_t, "unit": "evals/s", "h2d_bytes_per_step": int(h2d),
                    "d2h_bytes_per_step": int(d2h), "api": "evaluate_sharded -> padsim_evaluate_allocations",
                    "steps": len(e2e_times), "stat": "median"},
            "gpu_launches": launches,
            "roofline": {"bound": "alu", "achieved": achieved, "peak": peak_fp64, "unit": "TFLOP/s",
                         "frac": achieved / peak_fp64,
                         "traffic": ncu_traffic(cfg["name"], names[dom]),
                         "kernel": names[dom], "kernel_ms_isolated": float(iso[dom]),
                         "unit_basis": f"simulated requests x {FP64_OPS_PER_REQ[names[dom]]} algorithmic FP64 "
                                       "ops/request (SURVEY 8(d)) / isolated kernel time",
                         "requests_per_launch": req_k[names[dom]],
                         "peak_basis": "measured DFMA rate (profiles/peaks_r02.json, tools/peaks_microbench.cu)",
                         "issue": {"warp_instr_per_request": wipr, "budget": WARP_INSTR_BUDGET,
                                   "event_frac": (WARP_INSTR_BUDGET / wipr) if wipr else None,
                                   "issue_active": ncu_field(cfg["name"], names[dom], "issue_active"),
                                   "source": "ncu --set full of the dominant kernel (profiles/ncu_traffic.json)"},
                         "kernels_ms_isolated": {n: float(v) for n, v in zip(names, iso)},
                         "kernels_ms_concurrent_span": {n: float(v) for n, v in zip(names, km)},
                         "kernels_des_instants": {n: int(v) for n, v in zip(names, evs)}},
            "north_star_cfg4_seconds_at_this_rate": cfg4_replays / value,
            "clocks": clocks,
        }
        if not args.no_cpu_baseline and world == 1:
            line["cpu_baseline"] = cpu_baseline(cfg, role, cap, pols, traces, qps, cand_budget,
                                                args.cpu_seconds, gpu_rep=rep)
            line["parity"] = line["cpu_baseline"].pop("parity")
        print(json.dumps(line), flush=True)
    ctx.close()
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
