"""Surrogate calibration and the BASELINE.json configuration grids (inputs).

DEFAULT_MODEL is SPEC's surrogate calibration (D1 anchors S:92, D2 params
S:93, limits S:223; 32-slot KV buffer P:285) — an *input*, like the
calibration file of S:75–98.  The configs restate BASELINE.json ``configs``
as concrete grids.  Candidate *enumeration* is method
arithmetic (row a1) and is done by each side from ``space``.
"""
from __future__ import annotations

import itertools

import numpy as np

DEFAULT_MODEL = {
    "min_w": 400, "max_w": 750,                               # P:156 cap range
    "prefill": [(400, 1.0), (700, 1.72), (750, 1.8)],         # S:92 D1, P:289 1.8x
    "decode": [(400, 1.0), (600, 1.4), (750, 1.45)],          # S:92 D1, P:289 1.3-1.5x
    "rate": 13000.0, "eff": 0.15,                             # S:93 D2
    "dec_fixed": 0.008, "dec_per_seq": 0.00025, "dec_per_ctx": 0.0,
    "kvb": 131072.0, "bw": 48e9, "ovh": 0.0005,
    "max_pb": 16, "pb_tokens": 16384, "max_db": 64, "slots": 32,
    "chunk": 512,                                             # S:264 coalesced-mode chunk
}

# Alg. 1 constants (S:372 defaults; P:294 sub-second tick, P:300 cooldown 2–6 s,
# P:161 settle "hundreds of ms", P:294 reassignment 2–5 s, P:449 decode peak 600 W)
DEFAULT_POLICY = {
    "kind": 0, "threshold": 8, "step_w": 50, "dec_ceiling_w": 600, "window_stamp": 0,
    "cooldown_s": 4.0, "tick_s": 0.25, "window_s": 5.0, "settle_s": 0.3, "reassign_s": 3.0,
}
KIND = {"static": 0, "dyn-power": 1, "dyn-gpu": 2, "dyn-both": 3,
        "coalesced": 4}   # non-disaggregated baseline with chunked prefill

DEFAULT_SLO = {"ttft": 1.0, "tpot": (0.040, 0.040)}    # Fig. 5a
PHASE_SLO = {"ttft": 1.0, "tpot": (0.040, 0.020)}      # §5.2


def policy(kind: str = "static", **kw) -> dict:
    p = dict(DEFAULT_POLICY)
    p["kind"] = KIND[kind]
    p.update(kw)
    return p


def static_candidates(n_gpus: int, xpd) -> tuple[np.ndarray, np.ndarray]:
    """(x, p, d) rows → role[C][N] (GPUs 0..x-1 prefill) and cap[C][N]."""
    xpd = np.asarray(xpd, dtype=np.int64).reshape(-1, 3)
    C = xpd.shape[0]
    role = np.ones((C, n_gpus), dtype=np.uint8)
    cap = np.zeros((C, n_gpus), dtype=np.int32)
    for c, (x, p, d) in enumerate(xpd):
        role[c, :x] = 0
        cap[c, :x] = p
        cap[c, x:] = d
    return role, cap


CONFIGS = {
    # 1: 4P4D, 100 W grid, 13 static candidates, one 200-req LB trace at QPS/GPU 1.5
    "cfg1": dict(n_gpus=8, budget_w=4800, space=dict(step_w=100, x_only=4), dynamic=None,
                 qps=[1.5], family="lb", seeds=1, n_req=200, slo=DEFAULT_SLO),
    # 2: all xPyD x 25 W pool-uniform caps (955), 16 QPS points, 8 seeds x 2000 (Fig. 1 sweep)
    "cfg2": dict(n_gpus=8, budget_w=4800, space=dict(step_w=25), dynamic=None,
                 qps=[0.25 * k for k in range(1, 17)], family="lb", seeds=8, n_req=2000,
                 slo=DEFAULT_SLO),
    # 3: dynamic policies swept on the two-phase trace (Fig. 9 / Fig. 10)
    "cfg3": dict(n_gpus=8, budget_w=4800, space=None, dynamic="sweep",
                 # static references of Fig. 5a / §5.1: 4P4D-600, 5P3D-600,
                 # 4P-750/4D-450, 4P-675/4D-525 at the node's 4800 W, and 4P4D-750 at 6000 W
                 # (x, p, d[, budget_w])
                 statics=[(4, 600, 600), (5, 600, 600), (4, 750, 450), (4, 675, 525), (4, 750, 750, 6000)],
                 qps=[1.5, 2.0, 2.5, 3.0], family="phase", seeds=8, n_req=10000, slo=PHASE_SLO),
    # 4: exhaustive static + dynamic, 64 QPS x 32 seeds (north-star target)
    "cfg4": dict(n_gpus=8, budget_w=4800, space=dict(step_w=25), dynamic="splits",
                 qps=[0.0625 * k for k in range(1, 65)], family="lb", seeds=32, n_req=2000,
                 slo=DEFAULT_SLO),
    # 5: 64 simulated GPUs, 38.4 kW, long-prompt / long-output mixes, 100k requests
    "cfg5": dict(n_gpus=64, budget_w=38400, space=dict(step_w=25), dynamic=None,
                 qps=[0.5 * k for k in range(1, 9)], family=("long_prompt", "long_output"),
                 seeds=2, n_req=100000, slo=DEFAULT_SLO),
}


def dynamic_candidates(cfg: dict):
    """Dynamic candidates: (x, p, d, policy-dict) rows (start allocation + policy)."""
    rows = []
    if cfg.get("dynamic") == "sweep":
        for kind in ("dyn-power", "dyn-both"):
            for th, cd, st, win in itertools.product((2, 4, 8, 16), (2.0, 3.0, 4.0, 5.0, 6.0),
                                                     (25, 50, 100), (2.5, 5.0, 10.0)):
                rows.append((4, 600, 600, policy(kind, threshold=th, cooldown_s=cd, step_w=st,
                                                  window_s=win)))
        for th, cd, win in itertools.product((2, 4, 8, 16), (2.0, 3.0, 4.0, 5.0, 6.0),
                                             (2.5, 5.0, 10.0)):
            rows.append((4, 600, 600, policy("dyn-gpu", threshold=th, cooldown_s=cd, window_s=win)))
    elif cfg.get("dynamic") == "splits":
        for kind in ("dyn-power", "dyn-gpu", "dyn-both"):
            for x in range(1, cfg["n_gpus"]):
                rows.append((x, 600, 600, policy(kind)))
    return rows


def get_config(name: str) -> dict:
    cfg = dict(CONFIGS[name])
    cfg["name"] = name
    return cfg
