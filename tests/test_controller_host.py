"""padsim_step_controller (the C-ABI's pure host Alg. 1 step, include/padsim.h)
against the oracle — CPU only (the host step needs no device).

1. Recorded sequences: dynamic oracle replays (Alg. 1 P:207-251 on the
   §5.2 two-phase trace) log, at every controller tick, the window
   statistics, |Q_P|, per-GPU load, drain-completion times, the decision and the
   node state after the tick.  Feeding the recorded observations through the
   host step from the candidate's initial state must reproduce every decision and
   every post-tick state (roles, draining, commanded / effective caps, pending
   raises, last_move): settle and flip timing included.
2. Random states: the decision alone equals the oracle's Alg. 1 step.
"""
import numpy as np
import pytest

import oracle
from workloads import DEFAULT_MODEL, PHASE_SLO, make_trace, policy, static_candidates


@pytest.fixture(scope="module")
def host_step():
    from paper_2601_12241_b200.build import build
    build()
    from paper_2601_12241_b200.binding import step_controller
    return step_controller


CASES = [("dyn-power", dict(cooldown_s=2.0), 2.0), ("dyn-gpu", dict(cooldown_s=2.0), 2.5),
         ("dyn-both", dict(cooldown_s=2.0), 2.0), ("dyn-both", dict(step_w=100, window_s=2.5), 3.0),
         ("dyn-gpu", dict(threshold=2, reassign_s=1.5, window_stamp=1), 1.5),
         ("dyn-both", dict(window_stamp=1, cooldown_s=3.0), 2.5)]


@pytest.mark.parametrize("kind,kw,qps", CASES)
def test_recorded_tick_sequences(host_step, kind, kw, qps):
    xpd = (4, 600, 600)
    role, cap = static_candidates(8, [xpd])
    pol = policy(kind, **kw)
    tr = make_trace("phase", 11, 2500)
    r = oracle.replay(DEFAULT_MODEL, role[0], cap[0], pol, 4800, PHASE_SLO, tr, qps, log_cap=1,
                      tick_cap=20000)
    assert not r["ticks_overflow"] and len(r["ticks"]) > 100
    n = 8
    st = dict(role=[int(v) for v in role[0]], cmd=[int(v) for v in cap[0]], eff=[int(v) for v in cap[0]],
              raise_=[0] * n, draining=[0] * n, last_move=0.0)
    st["raise"] = st.pop("raise_")
    acted = 0
    for k, tk in enumerate(r["ticks"]):
        stats = dict(ttft_stat=tk["ttft_stat"], tpot_stat=tk["tpot_stat"], ttft_slo=tk["ttft_slo"],
                     tpot_slo=tk["tpot_slo"], q_prefill=tk["q_prefill"], load=tk["load"],
                     drained_empty=tk["drained_empty"])
        a, st = host_step(pol, DEFAULT_MODEL, 4800, st, stats, tk["t"])
        assert (a["kind"], a["direction"], a["gpu"]) == (tk["kind"], tk["direction"], tk["gpu"]), (k, tk["t"])
        assert st["role"] == tk["role"] and st["draining"] == tk["draining"], (k, tk["t"])
        assert st["cmd"] == tk["cmd"] and st["eff"] == tk["eff"] and st["raise"] == tk["raise_to"], (k, tk["t"])
        assert st["last_move"] == tk["last_move"]
        acted += a["kind"] in (1, 2)
    assert acted >= 1
    # the recorded replays are not degenerate: moves and (dyn-gpu) role flips happen
    if kind != "dyn-power":
        assert r["n_flips"] >= 1


def test_random_states_match_oracle_decision(host_step):
    rng = np.random.default_rng(7)
    for trial in range(400):
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
        pol = policy(kind, step_w=int(rng.choice([25, 50, 100])), dec_ceiling_w=int(rng.choice([600, 750])))
        budget = max(4800, 400 * n)
        now = float(rng.choice([5.0, 10.0, 13.5]))
        a1, s1 = host_step(pol, DEFAULT_MODEL, budget, st, stats, now)
        a2, s2 = oracle.step_controller(pol, DEFAULT_MODEL, budget, dict(st, drain_pending=int(sum(drain) > 0)),
                                        dict(stats), now)
        assert a1 == a2, (trial, a1, a2)
        # targets after the move = commanded caps + pending raises
        tgt = [r if r > 0 else c for r, c in zip(s1["raise"], s1["cmd"])]
        assert tgt == s2["cmd"] and s1["draining"] == s2["draining"] and s1["last_move"] == s2["last_move"]


def test_settle_and_flip_transitions(host_step):
    # hand-worked: a move at t = 10 with settle 0.3 s; decreases are effective (and
    # raises applied) only from t = 10.3; a drained GPU that emptied at
    # t = 11 flips at 11 + reassign 3 s
    pol = policy("dyn-both", step_w=50)
    st = dict(role=[0, 0, 0, 0, 1, 1, 1, 1], cmd=[600] * 8, eff=[600] * 8, draining=[0] * 8, last_move=0.0)
    hot = dict(ttft_stat=1.4, tpot_stat=0.01, ttft_slo=1.0, tpot_slo=0.04, q_prefill=12, load=[0] * 8)
    a, s = host_step(pol, DEFAULT_MODEL, 4800, st, hot, 10.0)
    assert a["kind"] == 1 and a["new_cap"] == [650] * 4 + [550] * 4
    assert s["cmd"] == [600] * 4 + [550] * 4 and s["eff"] == [600] * 8 and s["raise"] == [650] * 4 + [0] * 4
    quiet = dict(hot, ttft_stat=0.5, q_prefill=0)
    a, s2 = host_step(pol, DEFAULT_MODEL, 4800, s, quiet, 10.25)
    assert a["kind"] == 0 and s2["eff"] == [600] * 8
    a, s3 = host_step(pol, DEFAULT_MODEL, 4800, s2, quiet, 10.3)
    assert s3["eff"] == [650] * 4 + [550] * 4 and s3["cmd"] == s3["eff"] and s3["raise"] == [0] * 8
    # drain + flip
    s4 = dict(s3, draining=[0, 0, 0, 0, 1, 0, 0, 0])
    e = [-1.0] * 8
    e[4] = 11.0
    a, s5 = host_step(pol, DEFAULT_MODEL, 4800, s4, dict(quiet, drained_empty=e), 13.9)
    assert s5["role"][4] == 1 and s5["draining"][4] == 1 and s5["flip_deadline"][4] == 14.0
    a, s6 = host_step(pol, DEFAULT_MODEL, 4800, s5, dict(quiet, drained_empty=e), 14.0)
    assert s6["role"][4] == 0 and s6["draining"][4] == 0 and s6["flip_deadline"][4] < 0


def test_rejects_bad_state(host_step):
    from paper_2601_12241_b200.binding import PadsimError
    pol = policy("dyn-both")
    st = dict(role=[0, 1], cmd=[300, 600], last_move=0.0)
    obs = dict(ttft_stat=0.0, tpot_stat=0.0, ttft_slo=1.0, tpot_slo=0.04)
    with pytest.raises(PadsimError) as e:
        host_step(pol, DEFAULT_MODEL, 1200, st, obs, 1.0)
    assert e.value.rc == -2
    with pytest.raises(PadsimError) as e:
        host_step(pol, DEFAULT_MODEL, 1200, dict(role=[0, 2], cmd=[600, 600]), obs, 1.0)
    assert e.value.rc == -1
