"""Load balance of the stage C (static decode) replays: instants per replay and
the per-warp-item bound (sum over items of the max over lanes vs the mean), in
the planner's lane order (decode-pool class, then prefill group, stable over
the candidate index; u = q * n_cc + cc).

    python tools/stagec_balance.py --config cfg4
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
ap.add_argument("--config", default="cfg4")
a = ap.parse_args()

import paper_2601_12241_b200 as pkg  # noqa: E402

cfg = get_config(a.config)
role, cap, pols, traces, qps, cb = build_workload(cfg, 0, pkg.enumerate_pool_uniform)
ctx = pkg.Context(0)
ctx.plan(traces, qps, DEFAULT_MODEL, role, cap, pols, cfg["slo"], cfg["budget_w"], cand_budget_w=cb)
ctx.run()
ms = ctx.kernel_times_ms()
ev = ctx.fetch_replays()["events"]          # [C, Q, S]
ctx.close()
st = [c for c, p in enumerate(pols) if p["kind"] == 0]
y = (role[st] == 1).sum(axis=1)
kcls = np.select([y <= 1, y <= 2, y <= 4, y <= 5], [0, 1, 2, 3], 4)
pre = [tuple(cap[c][role[c] == 0]) for c in st]
gid = {}
grp = np.array([gid.setdefault(p, len(gid)) for p in pre])
order = sorted(range(len(st)), key=lambda i: (kcls[i], grp[i], i))
out = {"config": a.config, "kernel_ms": ms}
for k in range(5):
    idx = [st[i] for i in order if kcls[i] == k]
    if not idx:
        continue
    e = ev[idx]                              # [n_cc, Q, S]
    n_cc, Q, S = e.shape
    items = []
    for s in range(S):
        flat = e[:, :, s].T.reshape(-1)      # u = q * n_cc + cc
        for i0 in range(0, flat.size, 32):
            blk = flat[i0:i0 + 32]
            items.append((blk.max(), blk.mean()))
    items = np.array(items, dtype=np.float64)
    out[f"class{k}"] = {"n_cc": n_cc, "inst_mean": float(e.mean()), "inst_max": int(e.max()),
                        "sum_max_over_sum_mean": float(items[:, 0].sum() / items[:, 1].sum())}
print(json.dumps(out))
