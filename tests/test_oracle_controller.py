"""Oracle pins for Algorithm 1 and the dynamic replay (c.3) — CPU only.

Pins: SPEC's controller examples, the DynPower convergence the
paper reports ("converged on the same power distribution as the static
4P-750W/4D-450W"), cooldown / role-bound / masking invariants
 and budget safety.
"""
import json
import os

import numpy as np
import pytest

import oracle
from workloads import DEFAULT_SLO, PHASE_SLO, make_trace, policy, static_candidates

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "appendix_a.json")))
SLO = {"ttft_slo": 1.0, "tpot_slo": 0.040}


def st(x, p, d, n=8, last_move=0.0, **kw):
    s = dict(role=[0] * x + [1] * (n - x), cmd=[p] * x + [d] * (n - x), last_move=last_move)
    s.update(kw)
    return s


def obs(ttft, tpot, q=0, load=None, **kw):
    o = dict(ttft_stat=ttft, tpot_stat=tpot, q_prefill=q, load=load or [0] * 8, **SLO)
    o.update(kw)
    return o


def test_tick_dp_move_power(model):
    # TTFT 1.4 > 1, queue 12 > 8, TPOT 18 ms < 40 ms, cooldown elapsed -> MovePower D->P
    a, s = oracle.step_controller(policy("dyn-power"), model, 4800, st(4, 600, 600),
                                  obs(1.4, 0.018, q=12), now=10.0)
    assert a["kind"] == 1 and a["direction"] == 0
    assert a["new_cap"] == [650] * 4 + [550] * 4
    assert s["last_move"] == 10.0


def test_tick_both_violated_none(model):
    # both SLOs violated -> neither guard holds
    a, s = oracle.step_controller(policy("dyn-both"), model, 4800, st(4, 600, 600),
                                  obs(1.4, 0.050, q=12), now=10.0)
    assert a["kind"] == 0 and s["last_move"] == 0.0


def test_tick_cooldown(model):
    # now - last_move = 1 s < cooldown 4 s -> none; strict '>' at equality (A20)
    for now in (6.0, 9.0):
        a, _ = oracle.step_controller(policy("dyn-both"), model, 4800, st(4, 600, 600, last_move=5.0),
                                      obs(1.4, 0.018, q=12), now=now)
        assert a["kind"] == 0
    a, _ = oracle.step_controller(policy("dyn-both"), model, 4800, st(4, 600, 600, last_move=5.0),
                                  obs(1.4, 0.018, q=12), now=9.0000001)
    assert a["kind"] == 1


def test_threshold_guard(model):
    # Alg. 1 |Q_P| > THRESHOLD strict
    a, _ = oracle.step_controller(policy("dyn-power"), model, 4800, st(4, 600, 600),
                                  obs(1.4, 0.018, q=8), now=10.0)
    assert a["kind"] == 0


@pytest.mark.parametrize("row", GOLD["move_power"]["rows"])
def test_move_power_examples(model, row):
    # S:335-336
    x, p, d, d_new, p_new = row
    a, _ = oracle.step_controller(policy("dyn-power"), model, 4800, st(x, p, d),
                                  obs(1.4, 0.018, q=12), now=10.0)
    assert a["new_cap"] == [p_new] * x + [d_new] * (8 - x)


def test_limits_reached(model):
    # S:337 4P@750/4D@450 D->P -> limits reached; dyn-power saturates (no move)
    a, s = oracle.step_controller(policy("dyn-power"), model, 4800, st(4, 750, 450),
                                  obs(1.4, 0.018, q=12), now=10.0)
    assert a["kind"] == 3 and s["last_move"] == 0.0
    # S:338 P->D with decode at the 600 W dynamic ceiling -> limits reached
    a, _ = oracle.step_controller(policy("dyn-power"), model, 4800, st(4, 600, 600),
                                  obs(0.5, 0.050), now=10.0)
    assert a["kind"] == 3
    # S:344 decode all at 400 (floor) -> limits for D->P
    a, _ = oracle.step_controller(policy("dyn-power"), model, 4800, st(4, 600, 400),
                                  obs(1.4, 0.018, q=12), now=10.0)
    assert a["kind"] == 3
    # S:345 4P4D@600 -> not reached D->P
    a, _ = oracle.step_controller(policy("dyn-power"), model, 4800, st(4, 600, 600),
                                  obs(1.4, 0.018, q=12), now=10.0)
    assert a["kind"] == 1


def test_move_gpu_examples(model):
    # after a move all caps uniform 4800/8 = 600; decode batches {0,3,5} -> the 0
    a, s = oracle.step_controller(policy("dyn-both"), model, 4800, st(5, 600, 400),
                                  obs(1.4, 0.018, q=12, load=[0, 0, 0, 0, 0, 3, 0, 5]), now=10.0)
    # decode donors at floor -> limits reached -> MoveGPU of the least loaded decode GPU (6)
    assert a["kind"] == 2 and a["gpu"] == 6 and a["new_cap"] == [600] * 8
    assert s["draining"][6] == 1 and s["drain_pending"] == 1
    # a second MoveGPU while a role change is pending -> saturated
    a2, _ = oracle.step_controller(policy("dyn-gpu"), model, 4800,
                                   dict(s, last_move=0.0), obs(1.4, 0.018, q=12), now=20.0)
    assert a2["kind"] == 3


def test_move_gpu_role_bounds(model):
    # 7 decode + 1 prefill, P->D -> rejected (would zero prefill)
    a, _ = oracle.step_controller(policy("dyn-gpu"), model, 4800, st(1, 600, 600),
                                  obs(0.5, 0.050), now=10.0)
    assert a["kind"] == 3
    a, _ = oracle.step_controller(policy("dyn-gpu"), model, 4800, st(2, 600, 600),
                                  obs(0.5, 0.050, load=[100, 50, 0, 0, 0, 0, 0, 0]), now=10.0)
    assert a["kind"] == 2 and a["gpu"] == 1


def test_policy_masking(model):
    # static never acts; dyn-gpu goes straight to MoveGPU; dyn-power never moves GPUs
    a, _ = oracle.step_controller(policy("static"), model, 4800, st(4, 600, 600),
                                  obs(1.4, 0.018, q=12), now=10.0)
    assert a["kind"] == 0
    a, _ = oracle.step_controller(policy("dyn-gpu"), model, 4800, st(4, 600, 600),
                                  obs(1.4, 0.018, q=12), now=10.0)
    assert a["kind"] == 2


def _dyn_run(model, pol, tr, qps, slo, x=4, p=600, d=600, budget=4800):
    role, cap = static_candidates(8, [(x, p, d)])
    return oracle.replay(model, role[0], cap[0], pol, budget, slo, tr, qps, log_cap=200000)


def test_dynpower_convergence(model):
    # S:517 / P:409: stationary prefill-heavy 8K/128, QPS/GPU 1.5, 4800 W, 4P4D@600
    # -> prefill 750, decode 450 within 120 s, then stays (3 moves, then saturated)
    R = 2500
    g = np.random.default_rng(11)
    tr = dict(s_unit=np.cumsum(g.standard_exponential(R)), in_tok=np.full(R, 8192, np.int32),
              out_tok=np.full(R, 128, np.int32), phase=np.zeros(R, np.uint8))
    r = _dyn_run(model, policy("dyn-power"), tr, 1.5, DEFAULT_SLO)
    moves = [rec for rec in r["log"] if rec[1] == oracle.LOG_MOVE_POWER]
    assert len(moves) == 3 and all(m[3] == 0 for m in moves)
    caps = {}
    for t, typ, gpu, a, b in r["log"]:
        if typ == oracle.LOG_CAPS:
            caps[gpu] = (t, a)
    assert [caps[g][1] for g in range(8)] == [750] * 4 + [450] * 4
    assert max(c[0] for c in caps.values()) <= 120.0
    assert r["n_moves_gpu"] == 0 and r["n_flips"] == 0


def _audit(r, pol, budget, n=8):
    log = r["log"]
    assert not r["log_overflow"]
    # budget safety
    for t, typ, gpu, a, b in log:
        if typ == oracle.LOG_BUDGET:
            assert a <= budget
    # cooldown spacing
    acts = [rec[0] for rec in log if rec[1] in (oracle.LOG_MOVE_POWER, oracle.LOG_MOVE_GPU)]
    for t0, t1 in zip(acts, acts[1:]):
        assert t1 - t0 > pol["cooldown_s"]
    # role bounds
    for t, typ, gpu, a, b in log:
        if typ == oracle.LOG_ROLES:
            assert 1 <= a and 1 <= b and a + b <= n
    # masking
    kinds = {rec[1] for rec in log}
    if pol["kind"] == 1:
        assert oracle.LOG_MOVE_GPU not in kinds and oracle.LOG_FLIP not in kinds
    if pol["kind"] == 2:
        assert oracle.LOG_MOVE_POWER not in kinds
    # post-MoveGPU caps uniform budget/N after the settle (S:516 iii)
    for k, rec in enumerate(log):
        if rec[1] == oracle.LOG_MOVE_GPU:
            nxt = [x for x in log[k + 1:] if x[1] == oracle.LOG_CAPS][:n]
            assert all(x[3] == budget // n for x in nxt)


@pytest.mark.parametrize("kind", ["dyn-power", "dyn-gpu", "dyn-both"])
@pytest.mark.parametrize("qps", [1.5, 2.5])
def test_dynamic_invariants_phase_trace(model, kind, qps):
    tr = make_trace("phase", 5, 2000)
    pol = policy(kind, cooldown_s=2.0)
    r = _dyn_run(model, pol, tr, qps, PHASE_SLO)
    _audit(r, pol, 4800)
    R = 2000
    assert np.all(r["completion"] >= r["transfer_end"])
    assert np.all(r["transfer_end"] > r["prefill_end"])
    assert np.all(r["ttft"] > 0)
    if kind != "dyn-power":
        assert r["n_moves_gpu"] > 0           # the phase shift forces role moves
    assert r["met"] <= R


def test_dynamic_beats_static_on_phase_trace(model):
    # SPEC acceptance #7 ordering (smoke, calibration-dependent; not a parity pin)
    tr = make_trace("phase", 1, 2000)
    base = _dyn_run(model, policy("static"), tr, 2.0, PHASE_SLO)["met"]
    both = _dyn_run(model, policy("dyn-both"), tr, 2.0, PHASE_SLO)["met"]
    assert both >= base


def test_provisioned_power_integral(model):
    # time-weighted mean of Σ effective caps; recompute from the budget log
    tr = make_trace("phase", 7, 1500)
    pol = policy("dyn-both", cooldown_s=2.0)
    r = _dyn_run(model, pol, tr, 2.0, PHASE_SLO)
    a0 = tr["s_unit"][0] * (1.0 / (2.0 * 8.0))
    last = r["completion"].max()
    pts = [(t, a) for t, typ, g, a, b in r["log"] if typ == oracle.LOG_BUDGET]
    # budget records: (time, Σ eff) at t = 0 and after every settle
    acc, prev, cur = 0.0, a0, pts[0][1]
    for t, v in pts[1:]:
        if t in [x[0] for x in r["log"] if x[1] == oracle.LOG_SETTLE]:
            if t > a0:
                acc += cur * (t - prev)
                prev = t
            cur = v
    acc += cur * (last - prev)
    assert r["avg_watts"] == pytest.approx(acc / (last - a0), rel=1e-12)
    assert 8 * 400 <= r["avg_watts"] <= 4800
    assert r["qps_per_watt"] == pytest.approx(r["goodput"] / r["avg_watts"], rel=1e-15)


def test_static_provisioned_power_is_capsum(model):
    role, cap = static_candidates(8, [(3, 700, 500)])
    r = oracle.replay(model, role[0], cap[0], policy("static"), 4800, DEFAULT_SLO,
                      make_trace("lb", 3, 300), 1.0)
    assert r["avg_watts"] == pytest.approx(3 * 700 + 5 * 500, rel=1e-15)


def test_met_for_slos_recount(model):
    role, cap = static_candidates(8, [(4, 700, 500)])
    tr = make_trace("lb", 8, 600)
    r = oracle.replay(model, role[0], cap[0], policy("static"), 4800, DEFAULT_SLO, tr, 1.5)
    slos = [{"ttft": f * 1.0, "tpot": (f * 0.04, f * 0.04)} for f in (0.5, 1.0, 2.0)] + \
           [{"ttft": 1.0, "tpot": (0.025, 0.025)}]
    got = oracle.met_for_slos(r["ttft"], r["tpot"], tr["phase"], slos)
    for k, s in enumerate(slos):
        assert got[k] == int(((r["ttft"] <= s["ttft"]) & (r["tpot"] <= s["tpot"][0])).sum())
    assert got[1] == r["met"]
    assert got[0] <= got[1] <= got[2]                       # monotone in SLO slack
