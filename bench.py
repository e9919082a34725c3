#!/usr/bin/env python
"""Benchmark: batched what-if evaluation (BASELINE.json metric) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg2] [--impl padsim|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...        (one rank per GPU, NCCL)

One *step* is one pass of the whole hot path (rows a1–a8 of SURVEY.md §8): every
candidate allocation × every QPS point × every trace is replayed (static and
dynamic kernels), reduced over traces and argmax-ed per QPS; with N > 1 ranks
the per-rank Σmet are all-reduced over NCCL and the global argmax recomputed.
Scaling is weak: rank r replays its own block of trace seeds (r·S … r·S+S−1),
so per-GPU work is fixed as N grows; the units all ranks processed ÷ the max
over ranks of the device time is ``value``.

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
TRAFFIC_PATH = os.path.join(ROOT, "profiles", "ncu_traffic.json")   # dram bytes/launch per kernel
OPS_PER_EVENT = 32          # algorithmic ALU ops of one DES event handler
# algorithmic DES events per simulated request: stage A
# arrival+routing, batch share, KV transfer end; stage C transfer-end routing, join,
# leave+scoring; the joint replay all six (controller ticks not counted)
EV_PER_REQ = {"stageA_kernel": 3, "stageC_kernel": 3, "joint_kernel": 6}
LANES_PER_SM = 128          # INT32/FP32 lanes per SM (4 SMSP x 32)


def build_workload(cfg: dict, rank: int = 0, enumerate_fn=None):
    """Candidates (role, cap, policies), traces (this rank's seed block), qps."""
    N, B = cfg["n_gpus"], cfg["budget_w"]
    rows, pols = [], []
    if cfg.get("space"):
        sp = cfg["space"]
        xpd = enumerate_fn(N, B, DEFAULT_MODEL["min_w"], DEFAULT_MODEL["max_w"], sp["step_w"])
        if sp.get("x_only"):
            xpd = xpd[xpd[:, 0] == sp["x_only"]]
        rows += [tuple(r) for r in xpd]
        pols += [policy("static")] * len(xpd)
    for xpd in cfg.get("statics", []):
        rows.append(tuple(xpd))
        pols.append(policy("static"))
    for x, p, d, pol in dynamic_candidates(cfg):
        rows.append((x, p, d))
        pols.append(pol)
    role, cap = static_candidates(N, rows)
    fams = cfg["family"] if isinstance(cfg["family"], tuple) else (cfg["family"],)
    S = cfg["seeds"]
    traces = [make_trace(f, rank * S + s, cfg["n_req"]) for f in fams for s in range(S)]
    return role, cap, pols, traces, list(cfg["qps"])


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


def cpu_baseline(cfg, role, cap, pols, traces, qps, seconds=15.0):
    """The oracle as it stands on a bounded deterministic sample of the workload."""
    import oracle
    cores = os.cpu_count() or 1
    C, Q, S = role.shape[0], len(qps), len(traces)
    total = C * Q * S
    # deterministic sample: every k-th (c, q) pair, all traces of seed 0 only
    t0 = time.perf_counter()
    probe = oracle.evaluate(DEFAULT_MODEL, role[:2], cap[:2], pols[:2], cfg["budget_w"], cfg["slo"],
                            traces[:1], qps[len(qps) // 2: len(qps) // 2 + 1], n_threads=1)
    del probe
    per = max((time.perf_counter() - t0) / 2, 1e-4)
    n_pairs = int(max(cores, min(C * Q, seconds * cores / per)))
    stride = max(1, (C * Q) // n_pairs)
    sel = np.arange(0, C * Q, stride)[:n_pairs]
    cs = sel // Q
    qs = sel % Q
    reps = 0
    t0 = time.perf_counter()
    # group by q so one evaluate() call per QPS point uses all host threads
    for q in np.unique(qs):
        cc = cs[qs == q]
        oracle.evaluate(DEFAULT_MODEL, role[cc], cap[cc], [pols[i] for i in cc], cfg["budget_w"],
                        cfg["slo"], traces[:1], [qps[q]], n_threads=cores)
        reps += len(cc)
    dt = time.perf_counter() - t0
    R = traces[0]["s_unit"].size
    return {"value": reps / dt, "unit": "evals/s", "cores": cores, "kind": "oracle",
            "sample": f"{reps} of {total} replays (every {stride}th (candidate,QPS) pair, trace seed 0), "
                      f"{dt:.1f} s", "req_per_s": reps * R / dt}


def run_reference(args, cfg, rank, world):
    """--impl reference: the CPU oracle as it stands, bounded sample per step."""
    if rank != 0:
        return
    import oracle                       # the reference arm is the oracle alone
    role, cap, pols, traces, qps = build_workload(cfg, 0, oracle.enumerate_pool_uniform)
    vals = []
    last = None
    for k in range(args.warmup + args.steps):
        cb = cpu_baseline(cfg, role, cap, pols, traces, qps, seconds=max(2.0, 20.0 / max(1, args.steps)))
        if k >= args.warmup:
            vals.append(cb["value"])
            last = cb
    v = float(np.mean(vals))
    R = traces[0]["s_unit"].size
    line = {"impl": "reference", "metric": "candidate-trace evaluations/sec", "value": v,
            "unit": "evals/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": None, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic",
            "config": {"workload": cfg["name"], "sample": last["sample"]},
            "cpu_baseline": dict(last, value=v),
            "e2e": {"value": v, "unit": "evals/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "sim_req_per_s": v * R}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="cfg4")
    ap.add_argument("--impl", default="padsim", choices=["padsim", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=3)
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
    from paper_2601_12241_b200.distributed import allreduce_met, max_over_ranks
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

    role, cap, pols, traces, qps = build_workload(cfg, rank, pkg.enumerate_pool_uniform)
    C, Q, S = role.shape[0], len(qps), len(traces)
    R = traces[0]["s_unit"].size
    n_req_total = sum(t["s_unit"].size for t in traces)
    ctx = pkg.Context(local)
    ctx.plan(traces, qps, DEFAULT_MODEL, role, cap, pols, cfg["slo"], cfg["budget_w"])
    d = ctx.device_results()

    def as_tensor(ptr, n, dtype, typestr):
        class _A:
            __cuda_array_interface__ = {"shape": (n,), "typestr": typestr, "data": (ptr, False),
                                        "version": 3, "strides": None}
        return torch.as_tensor(_A(), device=dev).view(dtype)

    met_dev = as_tensor(d.d_met, C * Q, torch.int64, "<i8")
    ev_dev = as_tensor(d.d_rep_events, C * Q * S, torch.int64, "<i8")
    met_glob = torch.empty(C * Q, dtype=torch.int64, device=dev)
    am_glob = torch.empty(Q, dtype=torch.int32, device=dev)
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)

    def step():
        ctx.run(stream.cuda_stream)
        if world > 1:
            met_glob.copy_(met_dev)
            allreduce_met(met_glob)
            ctx.argmax_device(met_glob.data_ptr(), C, Q, am_glob.data_ptr(), stream.cuda_stream)
        return 3 + (1 if world > 1 else 0) + (1 if any(p["kind"] for p in pols) else 0)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    launches = 0
    times = []
    replay_ms = []
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
            launches += step()
            e1.record(stream)
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1))
            replay_ms.append(ctx.replay_kernel_ms())
            kern_ms.append(ctx.kernel_times_ms())
    t_local = sum(times) / 1e3
    t_max = max_over_ranks(t_local, device=dev)
    units = C * Q * S * world
    value = units * args.steps / t_max
    ev_rep = ev_dev.view(C, Q, S)
    is_dyn = torch.tensor([p["kind"] != 0 for p in pols], device=dev)
    ev_static = int(ev_rep[~is_dyn].sum().item())
    ev_dyn = int(ev_rep[is_dyn].sum().item())
    ev_a = int(as_tensor(d.d_aux_events, d.n_aux_events, torch.int64, "<i8").sum().item()) \
        if d.n_aux_events > 0 else 0
    if ev_a == 0:            # N > 8: static replays run in the joint kernel
        ev_dyn += ev_static
        ev_static = 0
    events_per_launch = ev_a + ev_static + ev_dyn
    # simulated requests each kernel processes per launch (the roofline unit)
    r_sum = sum(int(t["s_unit"].size) for t in traces)
    static_idx = [c for c in range(C) if pols[c]["kind"] == 0]
    groups = {tuple(int(v) for v in cap[c][role[c] == 0]) for c in static_idx}
    fact = ev_a > 0                       # the factorized static path ran (N <= 8)
    req_k = {"stageA_kernel": len(groups) * Q * r_sum if fact else 0,
             "stageC_kernel": len(static_idx) * Q * r_sum if fact else 0,
             "joint_kernel": (C - len(static_idx) + (0 if fact else len(static_idx))) * Q * r_sum}

    # e2e: the public one-shot C-ABI call with host buffers
    e2e_times = []
    h2d = sum(t["s_unit"].nbytes + 4 * t["in_tok"].size * 2 + t["s_unit"].size for t in traces)
    h2d += role.nbytes + cap.nbytes + 48 * C + 8 * Q
    d2h = C * Q * 24 + Q * 4
    for k in range(args.e2e_steps + 1 if args.e2e_steps > 0 else 0):
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        out = pkg.evaluate_allocations(traces, qps, DEFAULT_MODEL, role, cap, pols, cfg["slo"],
                                       cfg["budget_w"], ctx=ctx)
        if world > 1:
            mg = torch.as_tensor(out["met"].ravel()).to(dev)
            allreduce_met(mg)
            mg.cpu()
        if k > 0:
            e2e_times.append(time.perf_counter() - t0)
    e2e_t = max_over_ranks(float(np.mean(e2e_times)) if e2e_times else float("nan"), device=dev)
    # restore the plan timed above (evaluate_allocations re-planned the ctx)

    if rank == 0:
        pk = peaks()
        clocks = clk.summary()
        f_mhz = clocks.get("sm_mhz") or pk.get("sm_max_mhz") or 1965.0
        r_ms = float(np.mean(replay_ms)) if replay_ms else float("nan")
        km = np.mean(np.array(kern_ms), axis=0) if kern_ms else np.zeros(3)
        names = ["stageA_kernel", "stageC_kernel", "joint_kernel"]
        evs = [ev_a, ev_static, ev_dyn]
        # dominant kernel = the one doing most of the algorithmic work (simulated
        # requests × events per request); kernels overlap on several streams, so
        # the longest event span is not necessarily the one the step is made of
        ops = [req_k[n] * EV_PER_REQ[n] * OPS_PER_EVENT for n in names]
        dom = int(np.argmax(ops))
        achieved = ops[dom] / (km[dom] / 1e3) / 1e12 if km[dom] > 0 else float("nan")
        peak = 148 * LANES_PER_SM * f_mhz * 1e6 / 1e12
        cfg4 = get_config("cfg4")
        cfg4_replays = (955 + 21) * len(cfg4["qps"]) * cfg4["seeds"]
        line = {
            "metric": "candidate-trace evaluations/sec", "value": value, "unit": "evals/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": t_max / args.steps * 1e3, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": cfg["name"], "n_cand": C, "n_qps": Q, "n_traces_per_rank": S,
                       "n_req": R, "replays_per_rank": C * Q * S, "family": cfg["family"],
                       "l2": "flushed between steps (512 MiB write)"},
            "sim_req_per_s": value * n_req_total / S,
            "e2e": {"value": units / e2e_t, "unit": "evals/s", "h2d_bytes_per_step": int(h2d),
                    "d2h_bytes_per_step": int(d2h), "api": "padsim_evaluate_allocations"},
            "gpu_launches": launches,
            "roofline": {"bound": "alu", "achieved": achieved, "peak": peak, "unit": "Tops/s",
                         "frac": achieved / peak, "traffic": ncu_traffic(cfg["name"], names[dom]),
                         "kernel": names[dom], "kernel_ms": float(km[dom]),
                         "unit_basis": "simulated requests x events/request x ops/event",
                         "requests_per_launch": req_k[names[dom]],
                         "events_per_request": EV_PER_REQ[names[dom]], "ops_per_event": OPS_PER_EVENT,
                         "des_instants_per_launch": evs[dom],
                         "ncu_issue_active": ncu_field(cfg["name"], names[dom], "issue_active"),
                         "peak_basis": f"148 SM x 128 lanes x {f_mhz:.0f} MHz (sampled clock)",
                         "kernels_ms": {n: float(v) for n, v in zip(names, km)},
                         "kernels_events": {n: int(v) for n, v in zip(names, evs)},
                         "replay_kernels_ms": r_ms},
            "north_star_cfg4_seconds_at_this_rate": cfg4_replays / value,
            "clocks": clocks,
        }
        if not args.no_cpu_baseline and world == 1:
            line["cpu_baseline"] = cpu_baseline(cfg, role, cap, pols, traces, qps, args.cpu_seconds)
        print(json.dumps(line), flush=True)
    ctx.close()
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
