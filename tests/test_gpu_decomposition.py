"""GPU ↔ oracle parity for SURVEY §8(f) row 2: the Fig. 6 split of TTFT into
queueing delay and prefill execution (TTFT = queue + exec + KV transfer,
S:96–97) and nearest-rank TTFT/TPOT percentiles.

Sums: the kernels add in batch-completion order, the oracle in request-id
order — FP64 agreement within the north_star 1e-9 relative bar.
Percentiles: exact (a sort moves values, no arithmetic)."""
import numpy as np
import pytest

import oracle
from workloads import DEFAULT_MODEL, DEFAULT_SLO, PHASE_SLO, make_trace, policy, static_candidates

pytestmark = pytest.mark.gpu

RTOL = 1e-9


@pytest.fixture(scope="module")
def pkg():
    from paper_2601_12241_b200.build import build
    build()
    import paper_2601_12241_b200 as p
    return p


def _run(pkg, traces, qps, role, cap, pols, slo, budget, records=False, joint=False, pcts=None,
         wide=-1):
    # wide: padsim_tuning.wide_path (-1 the planner's choice, 0 / 1 force the
    # thread-per-replay / warp-per-replay static stages of N <= 8 nodes)
    ctx = pkg.Context(0, tuning=dict(wide_path=wide))
    try:
        ctx.plan(traces, qps, DEFAULT_MODEL, role, cap, pols, slo, budget, records=records, joint=joint)
        ctx.run()
        dec = ctx.fetch_decomposition()
        pc = ctx.fetch_percentiles(pcts) if pcts is not None else None
        rec = ctx.fetch_records() if records else None
    finally:
        ctx.close()
    return dec, pc, rec


def _check_decomposition(dec, traces, qps, role, cap, pols, slo, budget):
    for c in range(role.shape[0]):
        for q, qv in enumerate(qps):
            sq = se = 0.0
            for s, tr in enumerate(traces):
                o = oracle.replay(DEFAULT_MODEL, role[c], cap[c], pols[c], budget, slo, tr, qv)
                gq, ge = dec["rep_queue"][c, q, s], dec["rep_exec"][c, q, s]
                assert np.isclose(gq, o["sum_queue"], rtol=RTOL, atol=1e-12), (c, q, s, gq, o["sum_queue"])
                assert np.isclose(ge, o["sum_exec"], rtol=RTOL, atol=1e-12), (c, q, s, ge, o["sum_exec"])
                sq += o["sum_queue"]
                se += o["sum_exec"]
            assert np.isclose(dec["sum_queue"][c, q], sq, rtol=RTOL, atol=1e-12)
            assert np.isclose(dec["sum_exec"][c, q], se, rtol=RTOL, atol=1e-12)


XPD = [(1, 750, 575), (3, 675, 525), (4, 600, 600), (6, 550, 700), (2, 450, 650)]


@pytest.mark.parametrize("joint,wide", [(False, 0), (False, 1), (True, -1)])
def test_decomposition_static(pkg, joint, wide):
    role, cap = static_candidates(8, XPD)
    pols = [policy("static")] * len(XPD)
    traces = [make_trace("lb", 70 + s, 400) for s in range(2)] + [make_trace("lb_bursty", 5, 300)]
    qps = [0.25, 1.5, 3.0, 5.0]
    dec, _, _ = _run(pkg, traces, qps, role, cap, pols, DEFAULT_SLO, 4800, joint=joint, wide=wide)
    _check_decomposition(dec, traces, qps, role, cap, pols, DEFAULT_SLO, 4800)
    # Fig. 6 backpressure shape: queueing grows with load for the 1P7D split
    assert dec["sum_queue"][0, -1] > dec["sum_queue"][0, 0]


def test_decomposition_dynamic_and_wide(pkg):
    role, cap = static_candidates(8, [(4, 600, 600), (3, 600, 600)])
    pols = [policy("dyn-both", cooldown_s=2.0), policy("dyn-power", step_w=25)]
    traces = [make_trace("phase", s, 800) for s in range(2)]
    qps = [1.5, 3.0]
    dec, _, _ = _run(pkg, traces, qps, role, cap, pols, PHASE_SLO, 4800)
    _check_decomposition(dec, traces, qps, role, cap, pols, PHASE_SLO, 4800)
    # N = 16 goes through the shared-memory-table joint kernel
    r16, c16 = static_candidates(16, [(8, 600, 600), (5, 700, 550)])
    p16 = [policy("static"), policy("dyn-both", cooldown_s=2.0)]
    t16 = [make_trace("lb", 9, 600)]
    d16, _, _ = _run(pkg, t16, [1.0, 2.5], r16, c16, p16, DEFAULT_SLO, 9600)
    _check_decomposition(d16, t16, [1.0, 2.5], r16, c16, p16, DEFAULT_SLO, 9600)


PCTS = [1, 50, 90, 99, 100]


def _check_percentiles(pc, rec, traces, qps, role, cap, pols, slo, budget):
    for c in range(role.shape[0]):
        for q, qv in enumerate(qps):
            for s, tr in enumerate(traces):
                R = tr["s_unit"].size
                o = oracle.replay(DEFAULT_MODEL, role[c], cap[c], pols[c], budget, slo, tr, qv)
                for k, p in enumerate(PCTS):
                    for m in ("ttft", "tpot"):
                        want = oracle.percentile(o[m], p) if R else np.nan
                        got = pc[m][c, q, s, k]
                        if R == 0:
                            assert np.isnan(got)
                        else:
                            assert got == want, (m, c, q, s, p, got, want)
                            # and it is the nearest rank of the GPU's own records
                            assert got == np.sort(rec[m][c, q, s, :R])[(p * R + 99) // 100 - 1]


@pytest.mark.parametrize("wide", [0, 1])
def test_percentiles_exact(pkg, wide):
    role, cap = static_candidates(8, XPD[:3])
    pols = [policy("static")] * 2 + [policy("dyn-both", cooldown_s=2.0)]
    traces = [make_trace("lb", 3, 500), make_trace("lb_bursty", 4, 37),
              {"s_unit": np.zeros(0), "in_tok": np.zeros(0, np.int32), "out_tok": np.zeros(0, np.int32),
               "phase": np.zeros(0, np.uint8)}]
    qps = [0.5, 2.5]
    _, pc, rec = _run(pkg, traces, qps, role, cap, pols, DEFAULT_SLO, 4800, records=True, pcts=PCTS,
                      wide=wide)
    _check_percentiles(pc, rec, traces, qps, role, cap, pols, DEFAULT_SLO, 4800)


def test_percentiles_global_sort_path(pkg):
    # more than 16384 requests: the bitonic buffer does not fit in shared memory
    role, cap = static_candidates(8, [(4, 600, 600)])
    pols = [policy("static")]
    traces = [make_trace("lb", 11, 17000)]
    qps = [1.0]
    _, pc, rec = _run(pkg, traces, qps, role, cap, pols, DEFAULT_SLO, 4800, records=True, pcts=PCTS)
    _check_percentiles(pc, rec, traces, qps, role, cap, pols, DEFAULT_SLO, 4800)


def test_percentile_validation(pkg):
    role, cap = static_candidates(8, [(4, 600, 600)])
    tr = [make_trace("lb", 0, 20)]
    ctx = pkg.Context(0)
    try:
        ctx.plan(tr, [1.0], DEFAULT_MODEL, role, cap, [policy("static")], DEFAULT_SLO, 4800)
        ctx.run()
        with pytest.raises(pkg.PadsimError):
            ctx.fetch_percentiles([90])          # plan without records
        ctx.plan(tr, [1.0], DEFAULT_MODEL, role, cap, [policy("static")], DEFAULT_SLO, 4800, records=True)
        ctx.run()
        for bad in ([0], [101], list(range(1, 18))):
            with pytest.raises(pkg.PadsimError):
                ctx.fetch_percentiles(bad)
        assert ctx.fetch_percentiles([100])["ttft"].shape == (1, 1, 1, 1)
    finally:
        ctx.close()
