"""Small runs of every replay-kernel variant for compute-sanitizer
(racecheck / synccheck / memcheck of the mbarrier + TMA bulk-copy kernels):

    compute-sanitizer --tool racecheck python tools/sanitize_small.py <variant>

variants: stageA32 stageA128 stageA256 stageC5 joint32 joint128 joint168 jointg coal n64 wide64 wide16
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import paper_2601_12241_b200 as pkg  # noqa: E402
from workloads import (DEFAULT_MODEL, DEFAULT_SLO, PHASE_SLO, make_trace, policy,  # noqa: E402
                       static_candidates)

which = sys.argv[1] if len(sys.argv) > 1 else "stageA32"
B, slo, tuning = 4800, DEFAULT_SLO, {}
traces = [make_trace("lb", 1, 200)]
xpd = [(1, 750, 575), (2, 700, 550), (3, 675, 525), (4, 600, 600), (5, 600, 600), (6, 550, 650), (7, 500, 700)]
if which.startswith("stage"):
    role, cap = static_candidates(8, xpd)
    pols = [policy("static")] * len(xpd)
    tuning = {"stageA32": dict(stage_a_threads=32), "stageA128": dict(stage_a_threads=128),
              "stageA256": dict(stage_a_threads=256),
              "stageC5": dict(stage_c_classes=5, stage_c_batch_lists=31)}[which]
elif which.startswith("joint"):
    role, cap = static_candidates(8, [(4, 600, 600), (3, 600, 600)])
    pols = [policy("dyn-both", cooldown_s=2.0), policy("dyn-gpu", cooldown_s=2.0)]
    traces, slo = [make_trace("phase", 2, 300)], PHASE_SLO
    tuning = {"joint32": dict(joint_threads=32, joint_reg_cap=0), "joint128": dict(joint_threads=128),
              "joint168": dict(joint_threads=32, joint_reg_cap=1),
              "jointg": dict(joint_groups=1)}[which]
elif which == "coal":
    cap = np.full((1, 16), 600, np.int32)
    role = np.zeros((1, 16), np.uint8)
    pols = [policy("coalesced")]
    B = 9600
elif which.startswith("wide"):            # N > 8 wide-node factorized path (one warp per replay)
    N = 64 if which == "wide64" else 16
    role, cap = static_candidates(N, [(N // 2, 600, 600), (N - 1, 600, 400), (1, 700, 560)])
    pols = [policy("static")] * 3
    B = 600 * N
    traces = [make_trace("long_output", 1, 200), make_trace("lb", 2, 150)]
    tuning = dict(wide_chunk=1)
else:                                     # n64: N > 8 joint kernel (keys in global scratch)
    role, cap = static_candidates(64, [(32, 600, 600), (20, 700, 540)])
    pols = [policy("static")] * 2
    B = 38400
    traces = [make_trace("long_prompt", 1, 200)]
    tuning = dict(wide_path=0)
ctx = pkg.Context(0, tuning=tuning)
ctx.plan(traces, [0.5, 2.0], DEFAULT_MODEL, role, cap, pols, slo, B)
ctx.run()
print(which, ctx.fetch()["met"].ravel()[:6], "launches", ctx.launch_count())
ctx.close()
