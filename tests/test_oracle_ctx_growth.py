"""Oracle pins for the context-growing decode cost — SURVEY §8(f) row 4,
reading A40.  CPU only.

The decode context of the step ending at boundary s is
C(s) = Σ_active (in_i + s − join_i) (prompt + tokens generated before the step,
S:70 "per_ctx·C"), so inside a constant-composition segment the step latency
is an arithmetic progression and boundary k is its partial sum.  The pins sum
the per-step latencies one step at a time from that definition (independent of
the oracle's closed-form evaluation order) and check the special cases that
reduce to A14/A15 exactly."""
import numpy as np
import pytest

import oracle
from workloads import DEFAULT_MODEL, DEFAULT_SLO, make_trace, policy, static_candidates

PC = 2e-7                     # per-context-token decode cost (s)
S_DEC_600 = 1.4               # Appendix A: s_dec(600)
ROLE, CAP = static_candidates(2, [(1, 600, 600)])


def _tr(s_unit, ins, outs):
    n = len(s_unit)
    return {"s_unit": np.asarray(s_unit, float), "in_tok": np.asarray(ins, np.int32),
            "out_tok": np.asarray(outs, np.int32), "phase": np.zeros(n, np.uint8)}


def _step(n, ctx):
    return (0.008 + 0.00025 * n + PC * ctx) / S_DEC_600


def _rep(tr, model, pol=None, qps=0.5):
    return oracle.replay(model, ROLE[0], CAP[0], pol or policy("static"), 1200, DEFAULT_SLO, tr, qps)


def test_single_request_sums_growing_steps():
    m = dict(DEFAULT_MODEL, dec_per_ctx=PC, ctx_growth=1)
    o = _rep(_tr([0.0], [1000], [5]), m)
    te = o["transfer_end"][0]
    # joins at step 0; steps 1..4 see contexts 1000+1 .. 1000+4
    want = sum(_step(1, 1000 + s) for s in range(1, 5))
    assert o["completion"][0] - te == pytest.approx(want, rel=1e-12)
    # without growth every step sees the prompt only (A15)
    m0 = dict(DEFAULT_MODEL, dec_per_ctx=PC, ctx_growth=0)
    o0 = _rep(_tr([0.0], [1000], [5]), m0)
    assert o0["completion"][0] - o0["transfer_end"][0] == pytest.approx(4 * _step(1, 1000), rel=1e-12)
    assert o["completion"][0] > o0["completion"][0]


def test_two_members_leave_and_new_segment():
    # two identical prompts at t = 0 share a prefill batch and transfer ends, so
    # both join the idle decode GPU at the same boundary (join step 0)
    m = dict(DEFAULT_MODEL, dec_per_ctx=PC, ctx_growth=1)
    o = _rep(_tr([0.0, 0.0], [800, 800], [3, 6]), m)
    te = o["transfer_end"]
    assert te[0] == te[1]
    # steps 1-2 with both (context 2·800 + 2s), then steps 3-5 with the second (800 + s)
    c0 = te[0] + sum(_step(2, 1600 + 2 * s) for s in (1, 2))
    c1 = c0 + sum(_step(1, 800 + s) for s in (3, 4, 5))
    assert o["completion"][0] == pytest.approx(c0, rel=1e-12)
    assert o["completion"][1] == pytest.approx(c1, rel=1e-12)


def test_reduces_exactly_without_ctx_cost():
    # per_ctx = 0: growth changes nothing, bit for bit (A14)
    tr = make_trace("lb", 3, 300)
    role, cap = static_candidates(8, [(4, 600, 600), (3, 700, 500)])
    for c in range(2):
        for kind in ("static", "coalesced"):
            a = oracle.replay(DEFAULT_MODEL, role[c], cap[c], policy(kind), 4800, DEFAULT_SLO, tr, 1.5)
            b = oracle.replay(dict(DEFAULT_MODEL, ctx_growth=1), role[c], cap[c], policy(kind), 4800,
                              DEFAULT_SLO, tr, 1.5)
            for k in ("ttft", "tpot", "completion"):
                assert np.array_equal(a[k], b[k]), (kind, k)


def test_growth_monotone_and_coalesced_single():
    tr = make_trace("lb", 4, 400)
    role, cap = static_candidates(8, [(4, 600, 600)])
    base = dict(DEFAULT_MODEL, dec_per_ctx=PC)
    a = oracle.replay(dict(base, ctx_growth=0), role[0], cap[0], policy("static"), 4800, DEFAULT_SLO, tr, 1.0)
    b = oracle.replay(dict(base, ctx_growth=1), role[0], cap[0], policy("static"), 4800, DEFAULT_SLO, tr, 1.0)
    # prefill and transfers are unaffected; decode only gets slower with growth
    assert np.array_equal(a["prefill_end"], b["prefill_end"])
    assert np.mean(b["tpot"]) > np.mean(a["tpot"])
    assert b["met"] <= a["met"]
    # coalesced, isolated request, chunk ≥ prompt: decode steps see in + s
    m = dict(base, ctx_growth=1, chunk=8192)
    o = oracle.replay(m, np.zeros(2, np.uint8), np.array([600, 600], np.int32), policy("coalesced"), 1200,
                      DEFAULT_SLO, _tr([0.0], [2000], [4]), 0.5)
    want = sum(_step(1, 2000 + s) for s in (1, 2, 3))
    assert o["completion"][0] - o["prefill_end"][0] == pytest.approx(want, rel=1e-12)


def test_validation():
    with pytest.raises(Exception):
        _rep(_tr([0.0], [10], [2]), dict(DEFAULT_MODEL, ctx_growth=2))
