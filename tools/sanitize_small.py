"""Small static / coalesced / dynamic runs for compute-sanitizer (debug aid)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import paper_2601_12241_b200 as pkg  # noqa: E402
from workloads import DEFAULT_MODEL, DEFAULT_SLO, make_trace, policy, static_candidates  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "static"
if which == "static":
    role, cap = static_candidates(8, [(1, 750, 575), (3, 675, 525), (4, 600, 600)])
    pols = [policy("static")] * 3
    B = 4800
elif which == "coal16":
    cap = np.full((1, 16), 600, np.int32)
    role = np.zeros((1, 16), np.uint8)
    pols = [policy("coalesced")]
    B = 9600
else:
    role, cap = static_candidates(8, [(4, 600, 600)])
    pols = [policy("dyn-both", cooldown_s=2.0)]
    B = 4800
ctx = pkg.Context(0)
ctx.plan([make_trace("lb", 1, 300)], [0.5, 2.0], DEFAULT_MODEL, role, cap, pols, DEFAULT_SLO, B)
ctx.run()
print(which, ctx.fetch()["met"].ravel()[:6])
ctx.close()
