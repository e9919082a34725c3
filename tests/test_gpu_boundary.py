"""SLO-boundary decisions on the non-records path (GPU ↔ oracle, bit-exact).

Every path scores a completion as the oracle does: tpot = (t − pe) / (out − 1)
in FP64, then the inclusive test `tpot <= TPOT_SLO` (A6) and the 1e-9-relative
near-boundary test.  (A division-free variant that decided the tests from the
margin was measured slower and not adopted.)  These SLOs are
placed exactly on, and within 1e-12 … 3e-9 relative of, tpot values the oracle
produced, so both outcomes of every decision are exercised on the non-records
path; met / near counts and the SLO-sweep counts must equal the oracle's
(north_star: bit-exact)."""
import numpy as np
import pytest

import oracle
from workloads import DEFAULT_MODEL, DEFAULT_SLO, make_trace, policy, static_candidates

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pkg():
    from paper_2601_12241_b200.build import build
    build()
    import paper_2601_12241_b200 as p
    return p


@pytest.mark.parametrize("wide", [0, 1], ids=["thread-stages", "warp-stages"])
def test_tpot_boundary_decisions_exact(pkg, wide):
    xpd = [(4, 600, 600), (4, 750, 450), (5, 650, 510), (6, 550, 700), (2, 700, 560), (7, 450, 750)]
    role, cap = static_candidates(8, xpd + [(4, 600, 600), (3, 600, 600)])
    pols = [policy("static")] * len(xpd) + [policy("dyn-both", cooldown_s=2.0), policy("dyn-power")]
    xpd = xpd + [None, None]          # the joint kernel (dynamic) takes the same decisions
    traces = [make_trace("lb", s, 400) for s in range(2)]
    qps = [0.75, 2.0, 3.5]
    o = oracle.replay(DEFAULT_MODEL, role[0], cap[0], pols[0], 4800, DEFAULT_SLO, traces[0], qps[1])
    tp = np.sort(o["tpot"][traces[0]["out_tok"] > 1])
    T = float(tp[tp.size // 2])                     # an exact tpot of some request
    slo = {"ttft": 2.0, "tpot": (T, T)}
    f = [1 + 2e-10, 1 - 2e-10, 1 + 1e-9, 1 + 2.9e-9, 1 + 3.1e-9, 1 + 1e-12, 1 - 1e-12]
    sweep = [{"ttft": 2.0, "tpot": (T * x, T * x)} for x in f] + \
            [{"ttft": 2.0, "tpot": (np.nextafter(T, 1.0), np.nextafter(T, 0.0))}]
    ctx = pkg.Context(0, tuning=dict(wide_path=wide))
    try:
        ctx.plan(traces, qps, DEFAULT_MODEL, role, cap, pols, slo, 4800)
        ctx.set_slo_sweep(sweep)
        ctx.run()
        res = ctx.fetch()
        ex = ctx.fetch_extras()
    finally:
        ctx.close()
    ref = oracle.evaluate(DEFAULT_MODEL, role, cap, pols, 4800, slo, traces, qps, n_threads=8)
    assert np.array_equal(res["met"], ref["met"])
    assert np.array_equal(res["near_boundary"], ref["near_boundary"])
    assert res["near_boundary"].sum() > 0          # the boundary was hit
    metk = np.zeros((len(xpd), len(qps), len(sweep)), np.int64)
    for c in range(len(xpd)):
        for q in range(len(qps)):
            for s in range(2):
                r = oracle.replay(DEFAULT_MODEL, role[c], cap[c], pols[c], 4800, slo, traces[s], qps[q])
                metk[c, q] += oracle.met_for_slos(r["ttft"], r["tpot"], traces[s]["phase"], sweep)
    assert np.array_equal(ex["met_sweep"], metk)
