"""Seeded synthetic inputs shared by the oracle side and the product side.

This package holds *inputs only*: trace generators (arrival process + length
mixes), the surrogate calibration constants (SPEC D1/D2, an input to the
method exactly like a calibration file) and the configuration grids
of BASELINE.json.  It contains none of the method's arithmetic (no latency
model, no replay, no enumeration, no scoring) and imports neither
``oracle`` nor ``paper_2601_12241_b200``.
"""
from .tracegen import make_trace, FAMILIES  # noqa: F401
from .configs import (DEFAULT_MODEL, DEFAULT_POLICY, DEFAULT_SLO, PHASE_SLO, CONFIGS,  # noqa: F401
                      policy, static_candidates, get_config)
