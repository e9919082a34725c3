"""Helpers shared by the GPU parity tests: run the same seeded inputs through
the CUDA path (via the C ABI) and through the oracle, compare."""
import numpy as np

import oracle
import paper_2601_12241_b200 as pkg

REC = ("ttft", "tpot", "prefill_end", "completion", "transfer_end")
RTOL = 1e-9   # north_star: FP64 per-request latencies within 1e-9 relative


def gpu_records(traces, qps, model, role, cap, pols, slo, budget, tuning=None, cand_budget=None):
    ctx = pkg.Context(0, tuning=tuning)
    try:
        ctx.plan(traces, qps, model, role, cap, pols, slo, budget, records=True, cand_budget_w=cand_budget)
        ctx.run()
        res = ctx.fetch()
        rep = ctx.fetch_replays()
        rec = ctx.fetch_records()
    finally:
        ctx.close()
    return res, rep, rec


def compare_records(traces, qps, model, role, cap, pols, slo, budget, exact=True, tuning=None,
                    cand_budget=None):
    """Per-request, per-replay comparison; returns number of requests compared.
    ``tuning``: launch-configuration overrides (padsim_set_tuning) to exercise.

    Static candidates of N ≤ 8 nodes have two planner paths — the thread-per-replay
    stages (wide_path = 0) and, for small workloads like these, the warp-per-replay
    wide path (the planner's auto choice, forced by wide_path = 1): unless the
    tuning names one, both are run and compared."""
    tuning = dict(tuning or {})
    runs = [tuning]
    if role.shape[1] <= 8 and "wide_path" not in tuning and any(p["kind"] == 0 for p in pols):
        runs = [dict(tuning, wide_path=0), dict(tuning, wide_path=1)]
    outs = [gpu_records(traces, qps, model, role, cap, pols, slo, budget, t, cand_budget) for t in runs]
    n = 0
    for c in range(role.shape[0]):
        for q, qv in enumerate(qps):
            for s, tr in enumerate(traces):
                bc = budget if cand_budget is None else int(cand_budget[c])
                o = oracle.replay(model, role[c], cap[c], pols[c], bc, slo, tr, qv)
                R = tr["s_unit"].size
                for t, (_res, rep, rec) in zip(runs, outs):
                    for k in REC:
                        g = rec[k][c, q, s, :R]
                        if exact:
                            bad = np.nonzero(g != o[k])[0]
                        else:
                            bad = np.nonzero(~np.isclose(g, o[k], rtol=RTOL, atol=0))[0]
                        assert bad.size == 0, (t, k, c, q, s, bad[:5], g[bad[:5]], o[k][bad[:5]])
                    assert rep["met"][c, q, s] == o["met"], (t, c, q, s)
                    assert rep["near_boundary"][c, q, s] == o["near_boundary"], t
                    assert rep["duration"][c, q, s] == o["duration"], t
                    assert rep["goodput"][c, q, s] == o["goodput"], t
                n += R
    ev = oracle.evaluate(model, role, cap, pols, budget, slo, traces, qps, n_threads=8,
                         cand_budget_w=cand_budget)
    for t, (res, _rep, _rec) in zip(runs, outs):
        assert np.array_equal(res["met"], ev["met"]), t
        assert np.array_equal(res["argmax"], ev["argmax"]), t
        assert np.array_equal(res["near_boundary"], ev["near_boundary"]), t
        assert np.array_equal(res["goodput"], ev["goodput"]), t
    return n
