"""GPU ↔ oracle parity through the C ABI (north_star bar: chosen allocation and
SLO-met counts bit-exact; FP64 per-request latencies and goodput within 1e-9
relative — the implementation in fact reproduces them bit for bit, which is
what these tests demand).  Inputs are the seeded synthetic traces of
workloads/ at the shapes of BASELINE.json's configs."""
import numpy as np
import pytest

import oracle
from gpu_helpers import compare_records, gpu_records
from workloads import (DEFAULT_MODEL, DEFAULT_SLO, PHASE_SLO, make_trace, policy,
                       static_candidates)

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pkg():
    from paper_2601_12241_b200.build import build
    build()
    import paper_2601_12241_b200 as p
    return p


XPD = [(1, 750, 575), (2, 700, 550), (3, 675, 525), (4, 600, 600), (4, 750, 450), (5, 600, 600),
       (6, 550, 700), (7, 500, 750), (4, 400, 400), (2, 450, 650)]


@pytest.mark.parametrize("family", ["lb", "lb_bursty"])
def test_static_records_exact(pkg, family):
    role, cap = static_candidates(8, XPD)
    pols = [policy("static")] * len(XPD)
    traces = [make_trace(family, s, 300) for s in range(2)]
    qps = [0.25, 1.0, 1.5, 2.5, 4.0]
    n = compare_records(traces, qps, DEFAULT_MODEL, role, cap, pols, DEFAULT_SLO, 4800)
    assert n == len(XPD) * len(qps) * 600


@pytest.mark.parametrize("bl_mask", ["16", "31", "0"])
def test_fine_decode_pool_classes(pkg, bl_mask):
    # large workloads split stage C into five decode-pool classes (KW = 1, 2, 4, 5, 7)
    # and use sorted batch lists for the KW = 7 class; force both on a small case
    # (every y = 1..7 appears; batch lists on no / the largest / every class):
    # records bit-exact
    # (with five classes the dynamic replays next to them use the 168-register
    # joint variant: two dynamic candidates exercise it)
    xpd = [(7, 500, 700), (6, 550, 650), (5, 600, 600), (4, 600, 600), (3, 650, 560),
           (2, 700, 540), (1, 750, 575), (4, 600, 600), (5, 600, 600)]
    role, cap = static_candidates(8, xpd)
    pols = [policy("static")] * 7 + [policy("dyn-both", cooldown_s=2.0), policy("dyn-power")]
    traces = [make_trace("lb", s, 250) for s in range(2)]
    compare_records(traces, [0.5, 1.5, 3.0], DEFAULT_MODEL, role, cap, pols, DEFAULT_SLO, 4800,
                    tuning=dict(stage_c_classes=5, stage_c_batch_lists=int(bl_mask)))


# Every launch variant the planner can pick for a large workload, forced on small
# cases: stage A CTAs of 256 (the cfg 4 headline path: KV slots in global scratch),
# 128 and 32 threads; joint replays in 128-thread CTAs, in 168-register one-warp
# CTAs, after stage A; few lanes per warp item.  Records bit-exact against the oracle.
TUNINGS = [dict(stage_a_threads=256), dict(stage_a_threads=128), dict(stage_a_threads=32),
           dict(joint_threads=128), dict(joint_threads=32, joint_reg_cap=1),
           dict(joint_after_stage_a=1, joint_lanes_per_warp=4),
           dict(stage_a_threads=256, stage_c_classes=5, joint_reg_cap=1),
           dict(joint_groups=1), dict(joint_groups=1, joint_threads=128),
           dict(joint_groups=1, stage_c_classes=5)]


@pytest.mark.parametrize("tuning", TUNINGS, ids=lambda t: ",".join(f"{k}={v}" for k, v in t.items()))
def test_launch_variants_records_exact(pkg, tuning):
    xpd = XPD[:6]
    role, cap = static_candidates(8, xpd + [(4, 600, 600), (3, 600, 600)])
    pols = [policy("static")] * len(xpd) + [policy("dyn-both", cooldown_s=2.0), policy("dyn-power")]
    traces = [make_trace("lb", 7 + s, 260) for s in range(2)] + [make_trace("phase", 3, 300)]
    compare_records(traces, [0.5, 1.5, 3.0], DEFAULT_MODEL, role, cap, pols, PHASE_SLO, 4800, tuning=tuning)


def test_window_stamp_completion_and_candidate_budgets(pkg):
    # policy window_stamp = 1 (SPEC S:309/S:357 completion-stamped TTFT samples) and
    # per-candidate budgets (Fig. 5a's 4P4D-750 W reference at 6000 W; a
    # 4000 W dyn-gpu candidate whose DistributeUniformPower target is 500 W)
    xpd = [(4, 600, 600), (5, 600, 600), (4, 750, 750), (3, 500, 500), (4, 600, 600)]
    role, cap = static_candidates(8, xpd)
    pols = [policy("dyn-both", window_stamp=1, cooldown_s=2.0), policy("dyn-power", window_stamp=1),
            policy("static"), policy("dyn-gpu", window_stamp=1, cooldown_s=2.0), policy("dyn-both")]
    cb = np.array([4800, 4800, 6000, 4000, 4800], np.int32)
    traces = [make_trace("phase", s, 600) for s in range(2)]
    compare_records(traces, [1.5, 2.5], DEFAULT_MODEL, role, cap, pols, PHASE_SLO, 4800, cand_budget=cb)
    with pytest.raises(pkg.PadsimError) as e:          # 6000 W candidate under the 4800 W node budget
        pkg.evaluate_allocations(traces, [1.5], DEFAULT_MODEL, role[2:3], cap[2:3], pols[2:3], PHASE_SLO, 4800)
    assert e.value.rc == -3


@pytest.mark.parametrize("groups", [0, 1], ids=["thread", "lane-groups"])
@pytest.mark.parametrize("kind", ["dyn-power", "dyn-gpu", "dyn-both"])
def test_dynamic_records_exact(pkg, kind, groups):
    # groups = 1: the lane-group joint kernel (group_path.cuh), one lane per GPU
    xpd = [(4, 600, 600), (5, 600, 600), (3, 600, 600), (4, 750, 450)]
    role, cap = static_candidates(8, xpd)
    pols = [policy(kind, cooldown_s=2.0), policy(kind, threshold=2, window_s=2.5, cooldown_s=3.0),
            policy(kind, step_w=25), policy(kind, step_w=100, window_s=10.0)]
    traces = [make_trace("phase", s, 800) for s in range(2)]
    qps = [1.5, 2.0, 3.0]
    compare_records(traces, qps, DEFAULT_MODEL, role, cap, pols, PHASE_SLO, 4800,
                    tuning=dict(joint_groups=groups))


def test_mixed_static_dynamic_and_argmax(pkg):
    cands = pkg.enumerate_pool_uniform(8, 4800, 400, 750, 50)
    role, cap = static_candidates(8, cands)
    pols = [policy("static")] * len(cands)
    drole, dcap = static_candidates(8, [(x, 600, 600) for x in range(1, 8)])
    role = np.concatenate([role, drole])
    cap = np.concatenate([cap, dcap])
    pols = pols + [policy("dyn-both")] * 7
    traces = [make_trace("lb", s, 250) for s in range(2)]
    qps = [0.5, 1.5, 2.5]
    got = pkg.evaluate_allocations(traces, qps, DEFAULT_MODEL, role, cap, pols, DEFAULT_SLO, 4800)
    ref = oracle.evaluate(DEFAULT_MODEL, role, cap, pols, 4800, DEFAULT_SLO, traces, qps, n_threads=8)
    assert np.array_equal(got["met"], ref["met"])
    assert np.array_equal(got["argmax"], ref["argmax"])
    assert np.array_equal(got["near_boundary"], ref["near_boundary"])
    assert np.array_equal(got["goodput"], ref["goodput"])


def _tr(s_unit, ins, outs, phase=None):
    n = len(s_unit)
    return {"s_unit": np.asarray(s_unit, float), "in_tok": np.asarray(ins, np.int32),
            "out_tok": np.asarray(outs, np.int32),
            "phase": np.zeros(n, np.uint8) if phase is None else np.asarray(phase, np.uint8)}


def test_edge_cases(pkg):
    role, cap = static_candidates(8, [(4, 600, 600), (1, 750, 575), (7, 600, 450)])
    pols = [policy("static")] * 3
    ties = _tr(np.zeros(40), np.full(40, 512), np.full(40, 3))              # all at t=0
    ones = _tr(np.arange(30) * 0.01, np.arange(1, 31) * 300, np.ones(30))   # out = 1
    single = _tr([0.5], [8192], [128])
    big = _tr(np.linspace(0, 1, 50), np.full(50, 20000), np.full(50, 2))    # head > token budget
    traces = [ties, ones, single, big]
    for m in (DEFAULT_MODEL, dict(DEFAULT_MODEL, slots=1), dict(DEFAULT_MODEL, max_pb=1),
              dict(DEFAULT_MODEL, max_db=2), dict(DEFAULT_MODEL, dec_per_ctx=2e-7),
              dict(DEFAULT_MODEL, pb_tokens=600)):
        compare_records(traces, [0.5, 3.0], m, role, cap, pols, DEFAULT_SLO, 4800)


@pytest.mark.parametrize("classes", [3, 5])
def test_short_outputs_small_wheel(pkg, classes):
    # every output ≤ 32 tokens: the decode timing wheel is its minimum (32 finish steps),
    # so the half-size heads of the KW = 4 / 5 classes have 16 buckets and a bucket's two
    # finish steps are 16 apart; heavy load keeps both in use
    rng = np.random.default_rng(11)
    R = 600
    tr = _tr(np.cumsum(rng.exponential(1.0, R)), rng.integers(256, 4096, R), rng.integers(1, 33, R))
    role, cap = static_candidates(8, XPD)
    compare_records([tr], [1.0, 4.0, 8.0], DEFAULT_MODEL,
                    role, cap, [policy("static")] * len(XPD), DEFAULT_SLO, 4800,
                    tuning=dict(stage_c_classes=classes, wide_path=0))


def test_empty_trace(pkg):
    role, cap = static_candidates(8, [(4, 600, 600)])
    empty = _tr([], [], [])
    res, rep, _ = gpu_records([empty, make_trace("lb", 0, 20)], [1.0], DEFAULT_MODEL, role, cap,
                              [policy("static")], DEFAULT_SLO, 4800)
    assert rep["met"][0, 0, 0] == 0 and rep["goodput"][0, 0, 0] == 0.0


def test_small_and_large_nodes(pkg):
    # N = 2 (tiny node) and N = 64 (cfg 5 shape, small trace)
    r2, c2 = static_candidates(2, [(1, 600, 600), (1, 750, 450)])
    compare_records([make_trace("lb", 3, 200)], [0.5, 1.5], DEFAULT_MODEL, r2, c2,
                    [policy("static")] * 2, DEFAULT_SLO, 1200)
    r64, c64 = static_candidates(64, [(32, 600, 600), (40, 675, 475), (10, 750, 550)])
    compare_records([make_trace("long_prompt", 1, 1500), make_trace("long_output", 1, 600)],
                    [0.5, 2.0], DEFAULT_MODEL, r64, c64, [policy("static")] * 3, DEFAULT_SLO, 38400)
    pd = [policy("dyn-both", cooldown_s=2.0)] * 2
    compare_records([make_trace("phase", 2, 3000)], [1.5], DEFAULT_MODEL, r64[:2], c64[:2], pd,
                    PHASE_SLO, 38400)


def test_cfg2_full_size_sampled(pkg):
    # BASELINE cfg 2 at full size on the GPU (955 x 16 QPS x 8 seeds x 2000 req) in the
    # launch configuration bench.py times; the oracle recomputes a sample of replays.
    cands = pkg.enumerate_pool_uniform(8, 4800, 400, 750, 25)
    assert len(cands) == 955
    role, cap = static_candidates(8, cands)
    pols = [policy("static")] * len(cands)
    traces = [make_trace("lb", s, 2000) for s in range(8)]
    qps = [0.25 * k for k in range(1, 17)]
    ctx = pkg.Context(0)
    ctx.plan(traces, qps, DEFAULT_MODEL, role, cap, pols, DEFAULT_SLO, 4800)
    ctx.run()
    res = ctx.fetch()
    rep = ctx.fetch_replays()
    ctx.close()
    assert np.array_equal(res["met"], rep["met"].sum(axis=2))
    rng = np.random.default_rng(2026)
    for _ in range(40):
        c, q, s = int(rng.integers(955)), int(rng.integers(16)), int(rng.integers(8))
        o = oracle.replay(DEFAULT_MODEL, role[c], cap[c], pols[c], 4800, DEFAULT_SLO, traces[s], qps[q])
        assert rep["met"][c, q, s] == o["met"], (c, q, s)
        assert rep["duration"][c, q, s] == o["duration"]
        assert rep["goodput"][c, q, s] == o["goodput"]
    # properties at any size: attainment in [0, 1]; every replay ran to completion
    assert (rep["met"] >= 0).all() and (rep["met"] <= 2000).all()
    assert (rep["duration"] > 0).all() and (rep["events"] > 0).all()
    # argmax is the per-QPS maximum of Σmet with the (Σcaps, index) tie-break
    capsum = cap.sum(axis=1)
    for q in range(16):
        key = np.lexsort((np.arange(955), capsum, -res["met"][:, q]))
        assert res["argmax"][q] == key[0]


def test_cfg3_dynamic_sampled(pkg):
    # cfg 3 shape (10k-request two-phase trace, dynamic policies) — sampled replays
    xpd = [(4, 600, 600)] * 4
    role, cap = static_candidates(8, xpd)
    pols = [policy("dyn-power", threshold=4), policy("dyn-gpu", cooldown_s=5.0),
            policy("dyn-both", step_w=25, window_s=2.5), policy("dyn-both", threshold=16, window_s=10.0)]
    traces = [make_trace("phase", 0, 10000)]
    qps = [2.0, 3.0]
    res, rep, rec = gpu_records(traces, qps, DEFAULT_MODEL, role, cap, pols, PHASE_SLO, 4800)
    for c in range(4):
        for q in range(2):
            o = oracle.replay(DEFAULT_MODEL, role[c], cap[c], pols[c], 4800, PHASE_SLO, traces[0], qps[q])
            assert rep["met"][c, q, 0] == o["met"]
            assert np.array_equal(rec["completion"][c, q, 0], o["completion"])
            assert np.array_equal(rec["ttft"][c, q, 0], o["ttft"])


def test_determinism(pkg):
    role, cap = static_candidates(8, XPD)
    pols = [policy("static")] * 8 + [policy("dyn-both")] * 2
    traces = [make_trace("lb", s, 500) for s in range(3)]
    a = pkg.evaluate_allocations(traces, [1.0, 2.0], DEFAULT_MODEL, role, cap, pols, DEFAULT_SLO, 4800)
    b = pkg.evaluate_allocations(traces, [1.0, 2.0], DEFAULT_MODEL, role, cap, pols, DEFAULT_SLO, 4800)
    for k in a:
        assert a[k].tobytes() == b[k].tobytes()


def test_validation_errors(pkg):
    role, cap = static_candidates(8, [(4, 600, 600), (4, 700, 600)])
    pols = [policy("static")] * 2
    with pytest.raises(pkg.PadsimError) as e:
        pkg.evaluate_allocations([make_trace("lb", 0, 10)], [1.0], DEFAULT_MODEL, role, cap, pols,
                                 DEFAULT_SLO, 4800)
    assert e.value.rc == -3 and e.value.bad_index == 1
    bad = dict(DEFAULT_MODEL, prefill=[(400, 1.0), (700, 0.9), (750, 1.8)])
    with pytest.raises(pkg.PadsimError) as e:
        pkg.evaluate_allocations([make_trace("lb", 0, 10)], [1.0], bad, role[:1], cap[:1], pols[:1],
                                 DEFAULT_SLO, 4800)
    assert e.value.rc == -5
    tr = make_trace("lb", 0, 10)
    tr["in_tok"][3] = 0
    with pytest.raises(pkg.PadsimError) as e:
        pkg.evaluate_allocations([tr], [1.0], DEFAULT_MODEL, role[:1], cap[:1], pols[:1], DEFAULT_SLO, 4800)
    assert e.value.rc == -6


def test_controller_device_matches_host_and_oracle(pkg):
    # the kernel's __device__ ctl_step (padsim_controller_decide_device) against the
    # host padsim_step_controller and the oracle's Alg. 1 step on random states
    from paper_2601_12241_b200.binding import step_controller as host_step
    rng = np.random.default_rng(5)
    ctx = pkg.Context(0)
    try:
        for trial in range(300):
            n = int(rng.integers(2, 9))
            x = int(rng.integers(1, n))
            role = [0] * x + [1] * (n - x)
            cmd = [int(v) for v in rng.choice(np.arange(400, 751, 25), n)]
            drain = [0] * n
            if rng.random() < 0.2:
                drain[int(rng.integers(n))] = 1
            st = dict(role=role, cmd=cmd, draining=drain, last_move=float(rng.choice([0.0, 3.0, 9.5])))
            stats = dict(ttft_stat=float(rng.choice([0.0, 0.5, 1.0, 1.4])),
                         tpot_stat=float(rng.choice([0.0, 0.02, 0.04, 0.05])),
                         ttft_slo=1.0, tpot_slo=0.04, q_prefill=int(rng.integers(0, 20)),
                         load=[int(v) for v in rng.integers(0, 5, n)])
            kind = ["static", "dyn-power", "dyn-gpu", "dyn-both"][trial % 4]
            pol = policy(kind, step_w=int(rng.choice([25, 50, 100])),
                         dec_ceiling_w=int(rng.choice([600, 750])))
            budget = max(4800, 400 * n)
            now = float(rng.choice([5.0, 10.0, 13.5]))
            a_dev = ctx.decide_device(pol, DEFAULT_MODEL, budget, st, stats, now)
            a_host, _ = host_step(pol, DEFAULT_MODEL, budget, st, stats, now)
            a_or, _ = oracle.step_controller(pol, DEFAULT_MODEL, budget, dict(st, drain_pending=int(sum(drain) > 0)),
                                             dict(stats), now)
            assert a_dev == a_host == a_or, (trial, a_dev, a_host, a_or)
    finally:
        ctx.close()


def test_enumeration_on_gpu_build(pkg):
    for N, B in ((8, 4800), (64, 38400)):
        assert np.array_equal(pkg.enumerate_pool_uniform(N, B, 400, 750, 25),
                              oracle.enumerate_pool_uniform(N, B, 400, 750, 25))


def test_joint_kernel_matches_factorized_path(pkg):
    # the same static candidates through the factorized stages (default) and through
    # the joint kernel (PADSIM_JOINT): identical per-request records, both = oracle
    role, cap = static_candidates(8, XPD)
    pols = [policy("static")] * len(XPD)
    traces = [make_trace("lb", 40 + s, 400) for s in range(2)] + [make_trace("lb_bursty", 3, 300)]
    qps = [0.5, 1.75, 3.5]
    outs = []
    for joint, groups in ((False, 0), (True, 0), (True, 1)):
        ctx = pkg.Context(0, tuning=dict(joint_groups=groups))
        try:
            ctx.plan(traces, qps, DEFAULT_MODEL, role, cap, pols, DEFAULT_SLO, 4800, records=True,
                     joint=joint)
            ctx.run()
            outs.append((ctx.fetch(), ctx.fetch_replays(), ctx.fetch_records()))
        finally:
            ctx.close()
    (ra, pa, ca) = outs[0]
    for rb, pb, cb in outs[1:]:        # joint kernel, one thread / one lane group per replay
        for k in ra:
            assert np.array_equal(ra[k], rb[k]), k
        for k in ("met", "near_boundary", "duration", "goodput"):
            assert np.array_equal(pa[k], pb[k]), k
        for k in ca:
            assert np.array_equal(ca[k], cb[k]), k
    ref = oracle.evaluate(DEFAULT_MODEL, role, cap, pols, 4800, DEFAULT_SLO, traces, qps, n_threads=8)
    assert np.array_equal(ra["met"], ref["met"]) and np.array_equal(ra["argmax"], ref["argmax"])


def test_cfg1_full_exact(pkg):
    # BASELINE cfg 1 in full: 4P4D on a 100 W grid (13 candidates), one 200-request trace
    xpd = pkg.enumerate_pool_uniform(8, 4800, 400, 750, 100)
    xpd = xpd[xpd[:, 0] == 4]
    assert len(xpd) == 13
    role, cap = static_candidates(8, xpd)
    pols = [policy("static")] * 13
    compare_records([make_trace("lb", 0, 200)], [1.5], DEFAULT_MODEL, role, cap, pols, DEFAULT_SLO, 4800)


def test_cfg4_shape_sampled(pkg):
    # cfg 4 shape: static + dynamic (3 policies x 7 splits at 600 W), R = 2000; sampled oracle
    cands = pkg.enumerate_pool_uniform(8, 4800, 400, 750, 50)
    role, cap = static_candidates(8, cands)
    drole, dcap = static_candidates(8, [(x, 600, 600) for x in range(1, 8)] * 3)
    role = np.concatenate([role, drole])
    cap = np.concatenate([cap, dcap])
    pols = [policy("static")] * len(cands) + [policy(k) for k in ("dyn-power", "dyn-gpu", "dyn-both")
                                               for _ in range(7)]
    traces = [make_trace("lb", s, 2000) for s in range(2)]
    qps = [0.0625 * k for k in (4, 16, 24, 32, 48, 64)]
    ctx = pkg.Context(0)
    ctx.plan(traces, qps, DEFAULT_MODEL, role, cap, pols, DEFAULT_SLO, 4800)
    ctx.run()
    rep = ctx.fetch_replays()
    ctx.close()
    rng = np.random.default_rng(4)
    picks = [(int(c), int(rng.integers(len(qps))), int(rng.integers(2)))
             for c in list(rng.integers(len(cands), size=12)) + list(range(len(cands), len(pols)))]
    for c, q, s in picks:
        o = oracle.replay(DEFAULT_MODEL, role[c], cap[c], pols[c], 4800, DEFAULT_SLO, traces[s], qps[q])
        assert rep["met"][c, q, s] == o["met"], (c, q, s)
        assert rep["duration"][c, q, s] == o["duration"]
        assert rep["goodput"][c, q, s] == o["goodput"]


@pytest.mark.parametrize("wide", [0, 1], ids=["thread-stages", "warp-stages"])
def test_slo_sweep_qps_per_watt_max80(pkg, wide):
    # Fig. 8 SLO scaling (0.5x-2x), Fig. 5b TPOT 25 ms, QPS/W,
    # max QPS at >= 80 % attainment — static and dynamic candidates
    xpd = [(4, 600, 600), (4, 750, 450), (4, 675, 525), (5, 600, 600), (3, 700, 540)]
    role, cap = static_candidates(8, xpd + [(4, 600, 600), (4, 600, 600)])
    pols = [policy("static")] * 5 + [policy("dyn-power", cooldown_s=2.0), policy("dyn-both")]
    traces = [make_trace("lb", s, 600) for s in range(2)]
    qps = [0.5, 1.0, 1.5, 2.0]
    slos = [{"ttft": f * 1.0, "tpot": (f * 0.04, f * 0.04)} for f in (0.5, 2.0)] + \
           [{"ttft": 1.0, "tpot": (0.025, 0.025)}]
    ctx = pkg.Context(0, tuning=dict(wide_path=wide))
    try:
        ctx.plan(traces, qps, DEFAULT_MODEL, role, cap, pols, DEFAULT_SLO, 4800)
        ctx.set_slo_sweep(slos)
        ctx.run()
        res = ctx.fetch()
        ex = ctx.fetch_extras()
    finally:
        ctx.close()
    C, Q = role.shape[0], len(qps)
    metk = np.zeros((C, Q, len(slos)), np.int64)
    qpw = np.zeros((C, Q))
    watts = np.zeros((C, Q))
    for c in range(C):
        for q in range(Q):
            for s in range(2):
                o = oracle.replay(DEFAULT_MODEL, role[c], cap[c], pols[c], 4800, DEFAULT_SLO, traces[s], qps[q])
                metk[c, q] += oracle.met_for_slos(o["ttft"], o["tpot"], traces[s]["phase"], slos)
                qpw[c, q] += o["qps_per_watt"]
                watts[c, q] += o["avg_watts"]
    assert np.array_equal(ex["met_sweep"], metk)
    assert np.array_equal(ex["qps_per_watt"], qpw)
    assert np.array_equal(ex["watts_sum"], watts)
    nreq = sum(t["s_unit"].size for t in traces)
    for c in range(C):
        for k in range(len(slos) + 1):
            m = res["met"][c] if k == 0 else metk[c, :, k - 1]
            ok = [q for q in range(Q) if 5 * m[q] >= 4 * nreq]
            want = max(ok, key=lambda q: qps[q]) if ok else -1
            assert ex["max_qps80"][c, k] == want, (c, k)


def test_long_trace_wide_index(pkg):
    # n_req > 32767 switches stage C to 32-bit stream indices: same results as the oracle
    role, cap = static_candidates(8, [(4, 700, 500), (3, 750, 475)])
    pols = [policy("static")] * 2
    traces = [make_trace("lb", 77, 40000)]
    qps = [1.25, 2.5]
    res, rep, rec = gpu_records(traces, qps, DEFAULT_MODEL, role, cap, pols, DEFAULT_SLO, 4800)
    for c in range(2):
        for q in range(2):
            o = oracle.replay(DEFAULT_MODEL, role[c], cap[c], pols[c], 4800, DEFAULT_SLO, traces[0], qps[q])
            assert rep["met"][c, q, 0] == o["met"]
            assert np.array_equal(rec["completion"][c, q, 0], o["completion"])
            assert np.array_equal(rec["tpot"][c, q, 0], o["tpot"])


def test_non_uniform_caps_within_pools(pkg):
    # per-GPU cap vectors that are not pool-uniform ("as long as the
    # aggregate GPU power adheres to its power limit, the power allocated to each GPU can vary")
    # and interleaved role layouts: the ABI takes full vectors; both GPU paths = oracle
    role = np.array([[0, 1, 0, 1, 0, 1, 1, 1], [1, 1, 0, 0, 0, 1, 0, 1], [0, 0, 0, 1, 1, 1, 1, 1]],
                    np.uint8)
    cap = np.array([[750, 450, 700, 500, 650, 400, 600, 550], [600, 400, 725, 700, 675, 500, 650, 450],
                    [750, 725, 700, 400, 425, 450, 500, 550]], np.int32)
    pols = [policy("static")] * 3
    traces = [make_trace("lb", 90 + s, 300) for s in range(2)]
    compare_records(traces, [0.75, 2.0], DEFAULT_MODEL, role, cap, pols, DEFAULT_SLO, 4800)
    compare_records(traces[:1], [1.5], DEFAULT_MODEL, role, cap,
                    [policy("dyn-both", cooldown_s=2.0)] * 3, DEFAULT_SLO, 4800)


@pytest.mark.parametrize("N,xpd,kind", [(8, (4, 600, 600), "static"), (8, (3, 700, 500), "dyn-both"),
                                         (16, (9, 650, 500), "static")])
def test_replay_records_abi(pkg, N, xpd, kind):
    # padsim_replay_records (SURVEY §8(b) parity helper): one candidate, one trace, one
    # QPS point through the C ABI — the per-request records are the oracle's, bit for bit
    role, cap = static_candidates(N, [xpd])
    pol = policy(kind, cooldown_s=2.0)
    tr = make_trace("phase" if kind != "static" else "lb", 17, 700)
    slo = PHASE_SLO if kind != "static" else DEFAULT_SLO
    got = pkg.replay_records(tr, 2.0, DEFAULT_MODEL, role[0], cap[0], pol, slo, 600 * N)
    ref = oracle.replay(DEFAULT_MODEL, role[0], cap[0], pol, 600 * N, slo, tr, 2.0)
    for k in ("ttft", "tpot", "prefill_end", "completion"):
        assert np.array_equal(got[k], ref[k]), k
    with pytest.raises(pkg.PadsimError) as e:          # Σ caps over the budget
        pkg.replay_records(tr, 2.0, DEFAULT_MODEL, role[0], cap[0], pol, slo, 100)
    assert e.value.rc == -3
