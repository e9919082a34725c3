"""GPU ↔ oracle parity for the coalesced (non-disaggregated, chunked-prefill)
baseline replay — SURVEY §8(f) row 3 (readings A33–A37).
Per-request records bit-exact, met / argmax exact, decomposition sums within
1e-9 relative."""
import numpy as np
import pytest

import oracle
from gpu_helpers import compare_records
from workloads import DEFAULT_MODEL, DEFAULT_SLO, make_trace, policy, static_candidates

pytestmark = pytest.mark.gpu

CO = policy("coalesced")


@pytest.fixture(scope="module")
def pkg():
    from paper_2601_12241_b200.build import build
    build()
    import paper_2601_12241_b200 as p
    return p


def _caps(n, rows):
    cap = np.asarray(rows, np.int32).reshape(-1, n)
    role = np.zeros_like(cap, dtype=np.uint8)
    role[:, n // 2:] = 1          # ignored by the coalesced replay (A33)
    return role, cap


def _tr(s_unit, ins, outs):
    n = len(s_unit)
    return {"s_unit": np.asarray(s_unit, float), "in_tok": np.asarray(ins, np.int32),
            "out_tok": np.asarray(outs, np.int32), "phase": np.zeros(n, np.uint8)}


@pytest.mark.parametrize("family", ["lb", "lb_bursty", "long_output"])
def test_coalesced_records_exact(pkg, family):
    role, cap = _caps(8, [[600] * 8, [550, 650] * 4, [400] * 8, [750] * 4 + [450] * 4])
    traces = [make_trace(family, 20 + s, 400) for s in range(2)]
    qps = [0.25, 1.0, 2.5, 4.0]
    compare_records(traces, qps, DEFAULT_MODEL, role, cap, [CO] * 4, DEFAULT_SLO, 4800)


def test_coalesced_edge_cases_and_model_variants(pkg):
    role, cap = _caps(2, [[600, 600], [750, 450]])
    ties = _tr(np.zeros(30), np.full(30, 700), np.full(30, 4))            # all at t = 0
    ones = _tr(np.arange(20) * 0.01, np.arange(1, 21) * 97, np.ones(20))  # out = 1
    ragged = _tr(np.linspace(0, 2, 25), np.arange(25) * 333 + 1, np.arange(25) % 7 + 1)
    traces = [ties, ones, ragged]
    for m in (DEFAULT_MODEL, dict(DEFAULT_MODEL, chunk=64), dict(DEFAULT_MODEL, chunk=8192),
              dict(DEFAULT_MODEL, max_db=2), dict(DEFAULT_MODEL, dec_per_ctx=3e-7)):
        compare_records(traces, [0.5, 3.0], m, role, cap, [CO] * 2, DEFAULT_SLO, 1200)


def test_coalesced_n16_and_mixed_plan(pkg):
    # N = 16 coalesced next to static and dynamic disaggregated candidates in one plan
    r16, c16 = _caps(16, [[600] * 16])
    compare_records([make_trace("lb", 4, 500)], [0.5, 2.0], DEFAULT_MODEL, r16, c16, [CO],
                    DEFAULT_SLO, 9600)
    rs, cs = static_candidates(8, [(4, 750, 450), (4, 600, 600)])
    rc, cc = _caps(8, [[600] * 8])
    role = np.concatenate([rs, rc, rs[1:]])
    cap = np.concatenate([cs, cc, cs[1:]])
    pols = [policy("static"), policy("static"), CO, policy("dyn-both", cooldown_s=2.0)]
    traces = [make_trace("lb", 8 + s, 300) for s in range(2)]
    compare_records(traces, [0.5, 1.5, 3.0], DEFAULT_MODEL, role, cap, pols, DEFAULT_SLO, 4800)


def test_coalesced_decomposition_and_sweep(pkg):
    role, cap = _caps(8, [[600] * 8, [500] * 8])
    traces = [make_trace("lb", 31, 500), make_trace("lb_bursty", 32, 400)]
    qps = [0.5, 2.0]
    sweep = [{"ttft": 0.5, "tpot": (0.025, 0.025)}, {"ttft": 2.0, "tpot": (0.08, 0.08)}]
    ctx = pkg.Context(0)
    try:
        ctx.plan(traces, qps, DEFAULT_MODEL, role, cap, [CO] * 2, DEFAULT_SLO, 4800, records=True)
        ctx.set_slo_sweep(sweep)
        ctx.run()
        dec = ctx.fetch_decomposition()
        ext = ctx.fetch_extras()
        pc = ctx.fetch_percentiles([50, 90, 99])
    finally:
        ctx.close()
    for c in range(2):
        for q, qv in enumerate(qps):
            msum = np.zeros(2, np.int64)
            for s, tr in enumerate(traces):
                o = oracle.replay(DEFAULT_MODEL, role[c], cap[c], CO, 4800, DEFAULT_SLO, tr, qv)
                assert np.isclose(dec["rep_queue"][c, q, s], o["sum_queue"], rtol=1e-9, atol=1e-12)
                assert np.isclose(dec["rep_exec"][c, q, s], o["sum_exec"], rtol=1e-9, atol=1e-12)
                msum += oracle.met_for_slos(o["ttft"], o["tpot"], tr["phase"], sweep)
                for k, p in enumerate((50, 90, 99)):
                    assert pc["ttft"][c, q, s, k] == oracle.percentile(o["ttft"], p)
                    assert pc["tpot"][c, q, s, k] == oracle.percentile(o["tpot"], p)
            assert np.array_equal(ext["met_sweep"][c, q, :2], msum)
            assert ext["watts_sum"][c, q] == 2 * float(cap[c].sum())     # static: Σ caps per trace


def test_coalesced_validation(pkg):
    role, cap = _caps(8, [[750] * 8])
    with pytest.raises(pkg.PadsimError):      # 6000 W > 4800 W budget
        pkg.evaluate_allocations([make_trace("lb", 0, 10)], [1.0], DEFAULT_MODEL, role, cap, [CO],
                                 DEFAULT_SLO, 4800)
    with pytest.raises(pkg.PadsimError):
        pkg.evaluate_allocations([make_trace("lb", 0, 10)], [1.0], dict(DEFAULT_MODEL, chunk=0), role,
                                 cap, [CO], DEFAULT_SLO, 6000)
