"""Load balance of the joint (dynamic) replays: events per replay and the
per-warp-item divergence bound (max over lanes vs mean), for a config.

    python tools/joint_balance.py --config cfg3 [--lpw 16]
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from bench import build_workload  # noqa: E402
from workloads import DEFAULT_MODEL, get_config  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg3")
ap.add_argument("--lpw", type=int, default=16)
a = ap.parse_args()

import paper_2601_12241_b200 as pkg  # noqa: E402

cfg = get_config(a.config)
role, cap, pols, traces, qps, _cb = build_workload(cfg, 0, pkg.enumerate_pool_uniform)
ctx = pkg.Context(0)
ctx.plan(traces, qps, DEFAULT_MODEL, role, cap, pols, cfg["slo"], cfg["budget_w"], cand_budget_w=_cb)
ctx.run()
ms = ctx.kernel_times_ms()
ev = ctx.fetch_replays()["events"]          # [C, Q, S]
ctx.close()
dyn = np.array([p["kind"] != "static" for p in pols])
e = ev[dyn]                                  # [Cd, Q, S]
Cd, Q, S = e.shape
out = {"config": a.config, "kernel_ms": ms, "dyn_replays": int(e.size),
       "events_total": int(e.sum()), "events_per_replay_mean": float(e.mean()),
       "events_per_replay_max": int(e.max()), "per_q_mean": e.mean(axis=(0, 2)).tolist(),
       "per_trace_mean": e.mean(axis=(0, 1)).tolist()}
for lpw in (4, 8, 16, 32):
    items = []
    for s in range(S):
        flat = e[:, :, s].T.reshape(-1)      # u = q * Cd + c order
        for i0 in range(0, flat.size, lpw):
            blk = flat[i0:i0 + lpw]
            items.append((blk.max(), blk.mean()))
    items = np.array(items, dtype=np.float64)
    out[f"lpw{lpw}"] = {"items": len(items), "sum_max_over_sum_mean": float(items[:, 0].sum() / items[:, 1].sum()),
                        "max_item_over_mean_item": float(items[:, 0].max() / items[:, 0].mean())}
print(json.dumps(out))
