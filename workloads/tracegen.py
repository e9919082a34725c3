"""Seeded synthetic request traces (a2 inputs; SURVEY.md §8(d) trace table).

A trace is four arrays of length R:
  s_unit  float64  cumulative *unit-rate* arrival times (first gap > 0);
                   arrival at QPS q on N GPUs is s_unit * (1/(q*N)) — that
                   scaling is method arithmetic and lives on each side.
  in_tok  int32    prompt tokens (≥ 1)
  out_tok int32    output tokens (≥ 1; the first one is produced by prefill)
  phase   uint8    0/1, selects the per-phase TPOT SLO

Randomness: numpy PCG64 streams keyed by (seed, family, purpose) so the
gap stream and the length stream are independent and traces are
reproducible byte for byte.  Common random numbers across QPS points: the
same unit-rate trace is scaled to every QPS (A16).

Families:
  lb           Poisson; in ~ U{512..8192}, out ~ U{128..256}    (LongBench-like, ≤8K in)
  lb_bursty    Gamma renewal, shape 0.25 (CV 2), mean 1; same lengths
  phase        Poisson; first half 8192/128 (phase 0), second half 500/500 (phase 1)
  long_prompt  Poisson; in ~ U{4096..8192}, out ~ U{64..256}
  long_output  Poisson; in ~ U{256..1024}, out ~ U{512..2048}
"""
from __future__ import annotations

import numpy as np

FAMILIES = {"lb": 1, "lb_bursty": 2, "phase": 3, "long_prompt": 4, "long_output": 5}
_GAPS, _LENGTHS = 1, 2


def _rng(seed: int, family: str, purpose: int) -> np.random.Generator:
    ss = np.random.SeedSequence([int(seed), FAMILIES[family], purpose])
    return np.random.Generator(np.random.PCG64(ss))


def make_trace(family: str, seed: int, n_req: int) -> dict:
    if family not in FAMILIES:
        raise ValueError(f"unknown trace family {family!r}")
    R = int(n_req)
    g = _rng(seed, family, _GAPS)
    if family == "lb_bursty":
        gaps = g.gamma(shape=0.25, scale=4.0, size=R)
        gaps = np.where(gaps > 0.0, gaps, np.finfo(np.float64).tiny)
    else:
        gaps = g.standard_exponential(size=R)
    s_unit = np.cumsum(gaps.astype(np.float64))
    lg = _rng(seed, family, _LENGTHS)
    phase = np.zeros(R, dtype=np.uint8)
    if family in ("lb", "lb_bursty"):
        in_tok = lg.integers(512, 8192, size=R, endpoint=True)
        out_tok = lg.integers(128, 256, size=R, endpoint=True)
    elif family == "phase":
        h = R // 2
        in_tok = np.where(np.arange(R) < h, 8192, 500)
        out_tok = np.where(np.arange(R) < h, 128, 500)
        phase[h:] = 1
    elif family == "long_prompt":
        in_tok = lg.integers(4096, 8192, size=R, endpoint=True)
        out_tok = lg.integers(64, 256, size=R, endpoint=True)
    else:  # long_output
        in_tok = lg.integers(256, 1024, size=R, endpoint=True)
        out_tok = lg.integers(512, 2048, size=R, endpoint=True)
    return {"s_unit": np.ascontiguousarray(s_unit, dtype=np.float64),
            "in_tok": np.ascontiguousarray(in_tok, dtype=np.int32),
            "out_tok": np.ascontiguousarray(out_tok, dtype=np.int32),
            "phase": phase, "family": family, "seed": int(seed)}
