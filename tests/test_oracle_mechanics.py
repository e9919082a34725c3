"""Oracle pins for the dynamic-replay mechanics and the SLO scoring boundary — CPU only.

Expected values come from tests/golden/mechanics.json, written by the hand
derivation tests/golden/derive_mechanics.py (c.1 formulas + the c.2/c.3 rules
applied by hand to scenarios small enough to follow step by step; it never
calls the oracle).  Each scenario is built so that a plausible mistake in the
oracle fails it (noted per test):
  (a) settle        PAPER.md:159-161 (§2.2): decreases at t+settle, raises
                    at the same settle instant, caps read at batch / segment start,
                    a decode GPU restarts its segment at its next boundary;
  (b) window        Alg. 1, A22: TTFT stamped at first token, window
                    [t-W, t] inclusive;
  (c) MoveGPU       P:294: queued prompts re-routed in queue order, the
                    role flips reassign_s after the GPU empties;
  (d) phase switch  S:375: the controller's TPOT SLO switches at the first
                    phase-1 arrival;
  (e) SLO boundary  A6: inclusive <=, near band 1e-9 relative.
"""
import json
import os

import numpy as np
import pytest

import oracle

G = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "mechanics.json")))


def _trace(t):
    n = len(t["s_unit"])
    return dict(s_unit=np.asarray(t["s_unit"], float), in_tok=np.asarray(t["in_tok"], np.int32),
                out_tok=np.asarray(t["out_tok"], np.int32),
                phase=np.asarray(t.get("phase", [0] * n), np.uint8))


def _run(model, sc, policy=None):
    pol = policy or sc["policy"]
    slo = dict(ttft=sc["slo"]["ttft"], tpot=tuple(sc["slo"]["tpot"]))
    return oracle.replay(model, sc["role"], sc["cap"], pol, sc["budget"], slo, _trace(sc["trace"]),
                         sc["qps"], log_cap=100000)


def _moves(r):
    return [(t, gpu, a) for t, typ, gpu, a, b in r["log"]
            if typ in (oracle.LOG_MOVE_POWER, oracle.LOG_MOVE_GPU)]


def test_a_settle_prefill_caps(model):
    # a raise applied at command time (2.0) would run batch 3 (start 2.2215) at
    # 700 W; a cap read at batch END would run it at 700 W too
    sc = G["settle"]
    r = _run(model, sc)
    e = sc["expect"]
    assert list(r["prefill_end"]) == e["prefill_end"]
    assert r["prefill_end"][6] != sc["wrong_variants"]["raise_at_command_pe6"]
    mv = [(t, a) for t, typ, g, a, b in r["log"] if typ == oracle.LOG_MOVE_POWER]
    assert [list(m) for m in mv] == e["moves"]
    st = [t for t, typ, g, a, b in r["log"] if typ == oracle.LOG_SETTLE]
    assert st == e["settles"]
    assert r["n_moves_power"] == e["n_moves_power"] and r["n_moves_gpu"] == 0
    caps = {}
    for t, typ, g, a, b in r["log"]:
        if typ == oracle.LOG_CAPS:
            caps[g] = a
    assert [caps[0], caps[1]] == e["final_caps"]


def test_a_settle_decode_segment_restart(model):
    # the decode cut takes effect at 2.3 (not at the 2.0 command) and the worker
    # restarts its segment at the first boundary >= 2.3 with the new step time
    sc = G["settle"]
    r = _run(model, sc)
    e = sc["expect"]
    assert r["completion"][0] == e["r0_completion"]
    assert r["tpot"][0] == e["r0_tpot"]
    assert e["r0_segments"][1][1] != sc["wrong_variants"]["cut_at_command_k1"]
    # every other request has out = 1 and completes at its transfer end
    assert np.all(r["completion"][1:] == r["transfer_end"][1:])
    assert np.all(r["tpot"][1:] == 0.0)


def test_b_window_inclusive_at_first_token(model):
    # stamping TTFT at completion (SPEC's variant) or an exclusive lower window
    # edge would leave the window empty at t = 1.0 -> no move
    sc = G["window"]["inclusive"]
    r = _run(model, sc)
    mv = _moves(r)
    assert mv and mv[0][0] == sc["expect_first_move_t"]
    assert r["prefill_end"][0] == G["window"]["pe0"]


def test_b_window_excludes_older_sample(model):
    sc = G["window"]["exclusive"]
    assert sc["policy"]["window_s"] < G["window"]["inclusive"]["policy"]["window_s"]
    r = _run(model, sc)
    assert all(t >= sc["expect_no_move_before"] for t, _, _ in _moves(r))


@pytest.mark.parametrize("mode", ["first_token", "completion"])
def test_b_window_stamping_modes(model, mode):
    # policy window_stamp: 0 = TTFT sample at the first token (A22), 1 = at
    # completion: the first move lands at 1.0 / 2.0
    sc = G["window_completion"][mode]
    r = _run(model, sc)
    mv = _moves(r)
    assert mv and mv[0][0] == sc["expect_first_move_t"]
    if mode == "completion":          # no move before r0/r1 complete: their decode is undisturbed
        assert r["completion"][0] == r["completion"][1] == G["window_completion"]["c01"]


def test_c_move_gpu_reroute_and_flip(model):
    # reversed re-routing would give r8 the last batch; a flip without the
    # reassignment delay would split r9/r11 over two decode GPUs
    sc = G["move_gpu"]
    r = _run(model, sc)
    e = sc["expect"]
    assert list(r["prefill_end"]) == e["prefill_end"]
    assert list(r["completion"]) == e["completion"]
    assert r["prefill_end"][8] != sc["wrong_variants"]["reversed_reroute_pe8"]
    assert r["completion"][9] != sc["wrong_variants"]["flip_without_reassign_comp9"]
    gm = [(t, g, a) for t, typ, g, a, b in r["log"] if typ == oracle.LOG_MOVE_GPU]
    assert [list(x) for x in gm] == [e["move_gpu"]]
    fl = [(t, g) for t, typ, g, a, b in r["log"] if typ == oracle.LOG_FLIP]
    assert [list(x) for x in fl] == [e["flip"]]
    assert r["n_moves_gpu"] == e["n_moves_gpu"] and r["n_flips"] == e["n_flips"]


def test_d_phase2_tpot_switch(model):
    # switching at the first phase-1 completion, or judging each sample by its own
    # phase, would leave the 0.030 s TPOT sample under its 0.04 s SLO -> no move at 2.0
    sc = G["phase_switch"]
    r = _run(model, sc)
    e = sc["expect"]
    assert r["tpot"][0] == e["r0_tpot"]
    mv = [(t, a) for t, typ, g, a, b in r["log"] if typ == oracle.LOG_MOVE_POWER]
    assert mv and list(mv[0]) == e["first_move"]
    caps = {}
    for t, typ, g, a, b in r["log"]:
        if typ == oracle.LOG_CAPS and t <= 2.0 + sc["policy"]["settle_s"]:
            caps[g] = a
    assert [caps[0], caps[1]] == e["caps_after"]


@pytest.mark.parametrize("case", G["boundary"]["cases"])
def test_e_slo_boundary(model, case):
    sc = G["boundary"]
    ttft_slo, tpot_slo, met, near = case
    slo = dict(ttft=ttft_slo, tpot=(tpot_slo, tpot_slo))
    r = oracle.replay(model, sc["role"], sc["cap"], dict(G["settle"]["policy"], kind=0), sc["budget"],
                      slo, _trace(sc["trace"]), sc["qps"])
    assert r["ttft"][0] == sc["ttft"] and r["tpot"][0] == sc["tpot"]
    assert (r["met"], r["near_boundary"]) == (met, near)
    # the SLO-sweep recount uses the same inclusive test
    assert oracle.met_for_slos(r["ttft"], r["tpot"], np.zeros(1, np.uint8), [slo])[0] == met
