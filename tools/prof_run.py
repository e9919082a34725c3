"""One padsim_run of a (reduced) BASELINE config for ncu captures.

    python tools/prof_run.py [--config cfg2] [--traces 2] [--runs 2]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from bench import build_workload  # noqa: E402
from workloads import DEFAULT_MODEL, get_config  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg2")
ap.add_argument("--traces", type=int, default=0, help="limit traces (0 = all)")
ap.add_argument("--runs", type=int, default=2)
ap.add_argument("--cand-stride", type=int, default=1, help="every k-th candidate only")
ap.add_argument("--tuning", default="{}", help="padsim_set_tuning overrides (JSON)")
a = ap.parse_args()

import paper_2601_12241_b200 as pkg  # noqa: E402
from paper_2601_12241_b200.build import build  # noqa: E402

build()
cfg = get_config(a.config)
role, cap, pols, traces, qps, cb = build_workload(cfg, 0, pkg.enumerate_pool_uniform)
if a.traces:
    traces = traces[: a.traces]
if a.cand_stride > 1:
    role, cap = role[:: a.cand_stride], cap[:: a.cand_stride]
    pols = pols[:: a.cand_stride]
    cb = None if cb is None else cb[:: a.cand_stride]
import json  # noqa: E402
ctx = pkg.Context(0, tuning=json.loads(a.tuning))
ctx.plan(traces, qps, DEFAULT_MODEL, role, cap, pols, cfg["slo"], cfg["budget_w"], cand_budget_w=cb)
for _ in range(a.runs):
    ctx.run()
    print("replay ms", ctx.replay_kernel_ms())
ctx.close()
