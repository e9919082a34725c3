"""Time one padsim_run on a deterministic subset of a BASELINE config.

    python tools/time_subset.py --config cfg5 --cands 64 --qps 2 --traces 1 [--runs 2]

Prints replays, simulated requests, replay-kernel ms and simulated req/s.
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from bench import build_workload  # noqa: E402
from workloads import DEFAULT_MODEL, get_config  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg5")
ap.add_argument("--cands", type=int, default=64)
ap.add_argument("--qps", type=int, default=2)
ap.add_argument("--traces", type=int, default=1)
ap.add_argument("--runs", type=int, default=2)
a = ap.parse_args()

import paper_2601_12241_b200 as pkg  # noqa: E402
from paper_2601_12241_b200.build import build  # noqa: E402

build()
cfg = get_config(a.config)
role, cap, pols, traces, qps = build_workload(cfg, 0, pkg.enumerate_pool_uniform)
C = role.shape[0]
stride = max(1, C // a.cands)
sel = list(range(0, C, stride))[: a.cands]
role, cap, pols = role[sel], cap[sel], [pols[i] for i in sel]
qps = qps[:: max(1, len(qps) // a.qps)][: a.qps]
traces = traces[: a.traces]
ctx = pkg.Context(0)
t0 = time.time()
ctx.plan(traces, qps, DEFAULT_MODEL, role, cap, pols, cfg["slo"], cfg["budget_w"])
plan_s = time.time() - t0
ms = []
for _ in range(a.runs):
    ctx.run()
    ms.append(ctx.replay_kernel_ms())
res = ctx.fetch()
ctx.close()
reps = len(sel) * len(qps) * len(traces)
nreq = sum(t["s_unit"].size for t in traces) * len(sel) * len(qps)
best = min(ms)
print(json.dumps({"config": a.config, "n_gpus_sim": cfg["n_gpus"], "replays": reps, "sim_requests": nreq,
                  "replay_ms": ms, "plan_s": plan_s, "sim_req_per_s": nreq / (best / 1e3),
                  "met_total": int(res["met"].sum())}))
