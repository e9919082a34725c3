"""A/B of launch tunings on one box: padsim_run time (CUDA events around the
whole run) of a BASELINE config under several padsim_set_tuning overrides,
interleaved runs, median per tuning.  Results are identical by construction
(every variant is parity-tested); this only measures speed.

    python tools/tune_sweep.py --config cfg3 --runs 3 '{}' '{"joint_lanes_per_warp": 8}'
"""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from bench import build_workload  # noqa: E402
from workloads import DEFAULT_MODEL, get_config  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg3")
ap.add_argument("--runs", type=int, default=3)
ap.add_argument("--traces", type=int, default=0, help="limit traces (0 = all)")
ap.add_argument("--cand-stride", type=int, default=1, help="every k-th candidate only")
ap.add_argument("--qps-stride", type=int, default=1,
                help="QPS points q with q mod k == offset (one rank's shard of the strong split)")
ap.add_argument("--qps-offset", type=int, default=0)
ap.add_argument("--flush", action="store_true",
                help="as bench.py: a 512 MiB device write and a synchronize before the measured run")
ap.add_argument("tunings", nargs="+")
a = ap.parse_args()

import paper_2601_12241_b200 as pkg  # noqa: E402
from paper_2601_12241_b200.build import build  # noqa: E402

build()
cfg = get_config(a.config)
role, cap, pols, traces, qps, cb = build_workload(cfg, 0, pkg.enumerate_pool_uniform)
if a.traces:
    traces = traces[: a.traces]
if a.qps_stride > 1:
    qps = qps[a.qps_offset:: a.qps_stride]
if a.cand_stride > 1:
    role, cap, pols = role[:: a.cand_stride], cap[:: a.cand_stride], pols[:: a.cand_stride]
    cb = None if cb is None else cb[:: a.cand_stride]
# one context at a time (each plans its scratch against the free device memory),
# tunings interleaved round by round
ms = [[] for _ in a.tunings]
kms = [None for _ in a.tunings]
met = [None for _ in a.tunings]
for _ in range(a.runs):
    for j, t in enumerate(a.tunings):
        ctx = pkg.Context(0, tuning=json.loads(t))
        ctx.plan(traces, qps, DEFAULT_MODEL, role, cap, pols, cfg["slo"], cfg["budget_w"], cand_budget_w=cb)
        ctx.run()                                  # warm-up
        if a.flush:
            import torch
            fl = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
            fl.fill_(1.0)
            torch.cuda.synchronize()
            del fl
        ctx.run()
        ms[j].append(ctx.replay_kernel_ms())
        kms[j] = [round(x, 2) for x in ctx.kernel_times_ms()]
        met[j] = ctx.fetch()["met"]
        ctx.close()
for t, m, km, mt in zip(a.tunings, ms, kms, met):
    print(json.dumps({"config": a.config, "tuning": json.loads(t), "ms": statistics.median(m),
                      "kernels_ms": km, "all_ms": m, "met_equal": bool((mt == met[0]).all())}))
