"""Host-side cost of the one-shot API pieces for a BASELINE config: padsim_plan
(validation, upload, launch planning), padsim_run (device), fetch — wall clock,
repeated (the e2e bench number is their sum plus the H2D/D2H copies).

    python tools/time_plan.py --config cfg4 [--reps 5]
"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from bench import build_workload  # noqa: E402
from workloads import DEFAULT_MODEL, get_config  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg4")
ap.add_argument("--reps", type=int, default=5)
a = ap.parse_args()

import paper_2601_12241_b200 as pkg  # noqa: E402

cfg = get_config(a.config)
role, cap, pols, traces, qps, cb = build_workload(cfg, 0, pkg.enumerate_pool_uniform)
ctx = pkg.Context(0)
for k in range(a.reps + 1):
    t0 = time.perf_counter()
    ctx.plan(traces, qps, DEFAULT_MODEL, role, cap, pols, cfg["slo"], cfg["budget_w"], cand_budget_w=cb)
    t1 = time.perf_counter()
    ctx.run()
    res = ctx.fetch()
    t2 = time.perf_counter()
    out = pkg.evaluate_allocations(traces, qps, DEFAULT_MODEL, role, cap, pols, cfg["slo"], cfg["budget_w"],
                                   cand_budget_w=cb, ctx=ctx)
    t3 = time.perf_counter()
    if k:
        print(f"plan {1e3 * (t1 - t0):.1f} ms  run+fetch {1e3 * (t2 - t1):.1f} ms  "
              f"evaluate_allocations {1e3 * (t3 - t2):.1f} ms  device {ctx.replay_kernel_ms():.1f} ms")
ctx.close()
