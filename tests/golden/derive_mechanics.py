#!/usr/bin/env python
"""Hand derivation of the dynamic-replay mechanics pins (tests/golden/mechanics.json).

NOT the oracle and not a simulator: each scenario below is small enough that
its timeline follows from the rules of SURVEY.md §8(c) c.2/c.3 by hand — the
derivation is written out step by step in the comments, and the only
arithmetic is the c.1 model formulas (pinned by Appendix A) and the FP64 sums
the rules name (A14 boundaries ``t_seg + (double)k*L``, prefill ends
``t + lat``).  Nothing here imports ``oracle/`` or the CUDA path.

    python tests/golden/derive_mechanics.py      # rewrites mechanics.json

Passages: settle / source-before-sink PAPER.md:159-161 (§2.2), P:291;
MoveGPU drain + reassignment P:294 (§3.3); window metrics Alg. 1
P:213 ("recent metrics"), readings A22 (TTFT stamped at first token, TPOT at
completion, window [t-W, t] inclusive); controller TPOT SLO switch at the
first phase-1 arrival S:375; inclusive SLO test A6 (SPEC D11 S:410).
"""
import json
import math
import os

HERE = os.path.dirname(os.path.abspath(__file__))
A = json.load(open(os.path.join(HERE, "appendix_a.json")))

# ---- c.1 model (SPEC D1/D2 S:92-93), op order of SURVEY §8(c) c.1 --------------
PRE = [(400, 1.0), (700, 1.72), (750, 1.8)]
DEC = [(400, 1.0), (600, 1.4), (750, 1.45)]
RATE, EFF, FIXED, PER_SEQ = 13000.0, 0.15, 0.008, 0.00025


def speedup(curve, w):
    if w == curve[-1][0]:
        return curve[-1][1]
    j = max(k for k in range(len(curve) - 1) if curve[k][0] <= w)
    diff = curve[j + 1][1] - curve[j][1]
    frac = float(w - curve[j][0]) / float(curve[j + 1][0] - curve[j][0])
    return curve[j][1] + diff * frac


def prefill_lat(T, b, w):
    be = 1.0 + EFF * float(b - 1)
    return (float(T) / (RATE * be)) / speedup(PRE, w)


def decode_lat(n, w):
    return (FIXED + PER_SEQ * float(n)) / speedup(DEC, w)


KV8192 = A["kv_lat"]["rows"][0][1]                # 0.022869621333333333 (Appendix A)
D600_2 = A["prefill_lat"]["rows"][3][3]           # prefill_lat(16384, 2, 600)
P600_1 = A["prefill_lat"]["rows"][2][3]           # prefill_lat(8192, 1, 600)
L1_600 = A["decode_lat"]["rows"][2][2]            # decode_lat(1, 600)
L1_400 = A["decode_lat"]["rows"][1][2]            # decode_lat(1, 400)
assert prefill_lat(16384, 2, 600) == D600_2 and prefill_lat(8192, 1, 600) == P600_1
assert decode_lat(1, 600) == L1_600 and decode_lat(1, 400) == L1_400


def first_k_ge(t0, L, k_lo, tau):
    """smallest k >= k_lo with t0 + (double)k*L >= tau (A14 boundary)"""
    k = k_lo
    while t0 + float(k) * L < tau:
        k += 1
    return k


def settle():
    """Scenario A — MovePower settle (c.3 'Per-GPU caps').

    Node: N=2, GPU0 prefill @600 W, GPU1 decode @600 W, B=1200.  dyn-power,
    THRESHOLD 0, step 100 W, decode ceiling 600, tick 1 s, cooldown 1.5 s,
    settle 0.3 s, window 100 s.  SLO TTFT 0.5 s, TPOT 10 s.  24 requests at
    t=0, 8192 prompt tokens; r0 has 600 output tokens, the rest 1.

    Prefill: one worker, FIFO batches of two (16384-token budget, A9), each
    batch starts when the previous ends.  Controller: tick 1.0 is inside the
    cooldown (1.0 > 1.5 false); at tick 2.0 the TTFT window holds first-token
    samples 0.74 and 1.48 (> 0.5), |Q_P| = 18 > 0, the TPOT window holds the
    out=1 completions (TPOT 0 < 10) -> D->P MovePower: decode 600->500
    (commanded at 2.0, effective at 2.3), prefill 600->700 applied at the settle
    instant 2.3.  Tick 3.0: cooldown.  Tick 4.0: again D->P: decode 500->400,
    prefill 700->750 (ceiling), both at 4.3.  Tick 6.0: prefill at its ceiling
    -> limits reached -> saturated (dyn-power).  A prefill batch reads the
    EFFECTIVE cap at its start (c.3 'Cap reads').
    """
    eff_p = [(0.0, 600), (2.3, 700), (4.3, 750)]      # (from time, effective prefill cap)

    def cap_at(t):
        return [c for (t0, c) in eff_p if t >= t0][-1]

    ends, t = [], 0.0
    for k in range(12):
        t = t + prefill_lat(16384, 2, cap_at(t))       # dispatch at t, end = t + lat
        ends.append(t)
    pe = [ends[i // 2] for i in range(24)]
    # decode: r0 alone on GPU1 (others have out = 1 and complete at transfer end).
    pe0 = pe[0]
    te0 = pe0 + KV8192
    # segment 1 at 600 W from te0; the decrease to 500 W is effective at 2.3 and
    # the worker starts a new segment at its first boundary >= 2.3 (dirty)
    L1 = decode_lat(1, 600)
    k1 = first_k_ge(te0, L1, 1, 2.3)
    t1 = te0 + float(k1) * L1
    L2 = decode_lat(1, 500)
    k2 = k1 + first_k_ge(t1, L2, 1, 4.3)               # segment 2 relative step
    t2 = t1 + float(k2 - k1) * L2
    L3 = decode_lat(1, 400)
    fin = 599                                           # finish step = 0 + out - 1
    assert fin > k2
    comp0 = t2 + float(fin - k2) * L3
    tpot0 = (comp0 - pe0) / 599.0
    return dict(
        _doc=settle.__doc__,
        model_overrides={}, n_gpus=2, role=[0, 1], cap=[600, 600], budget=1200,
        policy=dict(kind=1, threshold=0, step_w=100, dec_ceiling_w=600, cooldown_s=1.5, tick_s=1.0,
                    window_s=100.0, settle_s=0.3, reassign_s=3.0),
        slo=dict(ttft=0.5, tpot=[10.0, 10.0]), qps=1.0,
        trace=dict(s_unit=[0.0] * 24, in_tok=[8192] * 24, out_tok=[600] + [1] * 23),
        expect=dict(prefill_end=pe, r0_segments=[[te0, 0, 600], [t1, k1, 500], [t2, k2, 400]],
                    r0_completion=comp0, r0_tpot=tpot0,
                    moves=[[2.0, 0], [4.0, 0]], settles=[2.3, 4.3 + 0.0], n_moves_power=2,
                    final_caps=[750, 400]),
        wrong_variants=dict(
            # a raise applied at command time: batch 3 (start 2.2215 < 2.3) would run at 700 W
            raise_at_command_pe6=ends[2] + prefill_lat(16384, 2, 700),
            # a decrease applied at command time: the decode restart at the first boundary >= 2.0
            cut_at_command_k1=first_k_ge(te0, L1, 1, 2.0)))


def window():
    """Scenario B — window membership and TTFT stamping (Alg. 1; A22).

    N=2, GPU0 prefill @600, GPU1 decode @600, B=1200; dyn-power, THRESHOLD 0,
    step 50, tick 1 s, cooldown 0.5 s, settle 0.3 s.  SLO TTFT 0.5 s, TPOT
    10 s.  Six requests at t=0 (8192 prompt, 200 output tokens).  Batch [r0,r1]
    ends at pe0 = prefill_lat(16384,2,600) = 0.7405 (two TTFT samples of value
    0.7405 > 0.5, stamped at first token = pe0); [r2,r3] ends 1.4810 > 1.0, so
    at tick 1.0 |Q_P| = 2 > 0 and no completion has happened (r0/r1 decode 199
    steps past 0.76), i.e. the TPOT window is empty (stat 0 < SLO).  With
    window_s = W_in = 1.0 - pe0 the window [1.0 - W, 1.0] starts exactly at pe0:
    inclusive -> the samples count -> D->P MovePower at t = 1.0.  With W_out
    (the next double below W_in for which 1.0 - W_out > pe0) they are outside:
    window empty -> stat 0 -> no move at 1.0; at tick 2.0 the window
    [2.0 - W_out, 2.0] holds no first-token sample either (1.48 < 1.74, the
    next batch ends 2.22) -> no move at 2.0.  Under SPEC's completion stamping
    the window at 1.0 would be empty even with W_in.
    """
    pe0 = D600_2
    w_in = 1.0 - pe0
    assert 1.0 - w_in == pe0
    w_out = w_in
    while not (1.0 - w_out > pe0):
        w_out = math.nextafter(w_out, 0.0)
    assert w_out < w_in
    base = dict(n_gpus=2, role=[0, 1], cap=[600, 600], budget=1200,
                slo=dict(ttft=0.5, tpot=[10.0, 10.0]), qps=1.0,
                trace=dict(s_unit=[0.0] * 6, in_tok=[8192] * 6, out_tok=[200] * 6))
    pol = dict(kind=1, threshold=0, step_w=50, dec_ceiling_w=600, cooldown_s=0.5, tick_s=1.0,
               settle_s=0.3, reassign_s=3.0)
    return dict(_doc=window.__doc__, pe0=pe0,
                inclusive=dict(base, policy=dict(pol, window_s=w_in), expect_first_move_t=1.0),
                exclusive=dict(base, policy=dict(pol, window_s=w_out), expect_no_move_before=2.5))


def window_completion():
    """Scenario B' — the same window under SPEC's completion stamping (policy
    window_stamp = 1; "completion-time-stamped", "over completions in
    [now - W, now]").  Eight requests at t=0 (8192 prompt): r0, r1 have 200
    output tokens, r2..r7 one (they complete at their transfer end, TPOT 0).
    Window W = W_in = 1.0 - pe0 as in scenario B.  First-token stamping: the
    samples of r0/r1 (stamped pe0) are in the window at tick 1.0 and |Q_P| = 4
    -> move at 1.0.  Completion stamping: no request completes before 1.0
    (r2/r3 transfer-complete at e2 + kv = 1.504), so the window is empty at
    1.0; at tick 2.0 it is [2.0 - W, 2.0] = [1.7405, 2.0]: r2/r3's stamps
    (1.504) are outside, r0/r1 complete together at c = te0 + 199*L2 (alone on
    the decode GPU, n = 2: out = 1 requests never join a decode batch) = 1.97,
    inside, with TTFT 0.7405 > 0.5; [r6, r7] are still queued (|Q_P| = 2) ->
    first move at 2.0.
    """
    pe0 = D600_2
    w_in = 1.0 - pe0
    te0 = pe0 + KV8192
    c01 = te0 + 199.0 * decode_lat(2, 600)
    assert 2.0 - w_in <= c01 <= 2.0
    e2 = pe0 + D600_2
    assert e2 + KV8192 < 2.0 - w_in
    base = dict(n_gpus=2, role=[0, 1], cap=[600, 600], budget=1200,
                slo=dict(ttft=0.5, tpot=[10.0, 10.0]), qps=1.0,
                trace=dict(s_unit=[0.0] * 8, in_tok=[8192] * 8, out_tok=[200, 200] + [1] * 6))
    pol = dict(kind=1, threshold=0, step_w=50, dec_ceiling_w=600, cooldown_s=0.5, tick_s=1.0,
               settle_s=0.3, reassign_s=3.0, window_s=w_in)
    return dict(_doc=window_completion.__doc__, c01=c01,
                first_token=dict(base, policy=dict(pol, window_stamp=0), expect_first_move_t=1.0),
                completion=dict(base, policy=dict(pol, window_stamp=1), expect_first_move_t=2.0))


def move_gpu():
    """Scenario C — MoveGPU: re-routing in queue order, flip at empty + reassign
    ("drained of all in-flight requests ... reassignment latency"; S:256;
    c.3 MoveGPU).

    N=3: GPU0, GPU1 prefill, GPU2 decode, all 600 W, B=1800 (uniform B/N = 600,
    so DistributeUniformPower changes nothing).  dyn-gpu, THRESHOLD 0, tick 1 s,
    cooldown 0.5 s, settle 0.3 s, reassign 1.0 s, window 100 s.  SLO TTFT 100 s,
    TPOT 1e-6 s.  14 requests at t=0 (8192 prompt, 2 output tokens).

    t=0: arrivals in id order go to the least-outstanding prefill GPU, lowest id:
    even ids -> GPU0, odd -> GPU1.  Batches of two: GPU0 [r0,r2] [r4,r6] [r8,r10]
    [r12]; GPU1 [r1,r3] [r5,r7] ...; the first pair ends at e1 = 0.7405, the
    second at e2 = e1 + 0.7405 = 1.4810.  r0..r3 transfer (te = e1 + kv) and all
    join GPU2 (n = 4), completing one step later with TPOT ~ 0.029 > 1e-6.
    Tick 1.0: TTFT p90 0.74 < 100, TPOT p90 > 1e-6 -> P->D; dyn-gpu -> MoveGPU:
    donors GPU0/GPU1 both hold 40960 outstanding tokens -> lowest id GPU0
    drains.  Its queued r8, r10, r12 are re-routed in that order to GPU1, whose
    queue becomes r9, r11, r13, r8, r10, r12: batches [r9,r11] end e3 = e2+d,
    [r13,r8] e4 = e3+d, [r10,r12] e5 = e4+d.  GPU0's in-service batch [r4,r6]
    ends at e2 -> empty -> role flip at e2 + 1.0.  Before the flip every
    transfer goes to GPU2: r9/r11 (te = e3 + kv < flip) join GPU2 together
    (n = 2).  After the flip GPU0 is a decode GPU: r8 (lower id, same instant as
    r13) -> GPU0, r13 -> GPU2, each alone (n = 1); r10 -> GPU0, r12 -> GPU2.
    Later ticks: drain pending, then one prefill GPU left -> saturated.
    """
    d = D600_2
    e1 = d
    e2 = e1 + d
    e3 = e2 + d
    e4 = e3 + d
    e5 = e4 + d
    flip_t = e2 + 1.0
    L1, L2, L4 = decode_lat(1, 600), decode_lat(2, 600), decode_lat(4, 600)
    pe = {0: e1, 1: e1, 2: e1, 3: e1, 4: e2, 5: e2, 6: e2, 7: e2, 9: e3, 11: e3, 13: e4, 8: e4,
          10: e5, 12: e5}
    comp = {}
    for i in (0, 1, 2, 3):
        comp[i] = (e1 + KV8192) + 1.0 * L4
    for i in (4, 5, 6, 7):
        comp[i] = (e2 + KV8192) + 1.0 * L4
    for i in (9, 11):
        comp[i] = (e3 + KV8192) + 1.0 * L2
    for i in (8, 13):
        comp[i] = (e4 + KV8192) + 1.0 * L1
    for i in (10, 12):
        comp[i] = (e5 + KV8192) + 1.0 * L1
    assert e3 + KV8192 < flip_t < e4 + KV8192
    return dict(
        _doc=move_gpu.__doc__, n_gpus=3, role=[0, 0, 1], cap=[600, 600, 600], budget=1800,
        policy=dict(kind=2, threshold=0, step_w=50, dec_ceiling_w=600, cooldown_s=0.5, tick_s=1.0,
                    window_s=100.0, settle_s=0.3, reassign_s=1.0),
        slo=dict(ttft=100.0, tpot=[1e-6, 1e-6]), qps=1.0,
        trace=dict(s_unit=[0.0] * 14, in_tok=[8192] * 14, out_tok=[2] * 14),
        expect=dict(prefill_end=[pe[i] for i in range(14)], completion=[comp[i] for i in range(14)],
                    move_gpu=[1.0, 0, 1], flip=[flip_t, 0], n_moves_gpu=1, n_flips=1),
        wrong_variants=dict(reversed_reroute_pe8=e5, flip_without_reassign_comp9=(e3 + KV8192) + L1))


def phase_switch():
    """Scenario D — controller TPOT SLO switches at the first phase-1 ARRIVAL
    (P:407 two-phase SLO 40 -> 20 ms).

    N=2, GPU0 prefill @650, GPU1 decode @500, B=1200; dyn-power, THRESHOLD 0,
    step 50, ceiling 600, tick 1 s, cooldown 0.5 s, settle 0.3 s, window 100 s.
    SLO TTFT 100 s, TPOT (phase 0: 0.04 s, phase 1: 0.001 s).  r0 (phase 0,
    8192/2) at t=0 completes at ~0.42 with TPOT = kv + decode_lat(1,500) ~ 0.030
    (stamped at completion).  r1 (phase 1, 8192/500) arrives at 1.2 (s_unit 2.4
    at q=1, N=2) and completes after 4 s.  Tick 1.0: SLO 0.04 -> TPOT 0.030 <
    0.04 and TTFT 0.39 < 100: no guard holds -> nothing.  Tick 2.0: the phase-1
    arrival switched the controller SLO to 0.001 -> TPOT 0.030 > 0.001, TTFT <
    100 -> P->D MovePower at 2.0: prefill 650 -> 600, decode 500 -> 550.
    """
    pe0 = prefill_lat(8192, 1, 650)
    tp0 = ((pe0 + KV8192) + 1.0 * decode_lat(1, 500) - pe0) / 1.0
    return dict(
        _doc=phase_switch.__doc__, n_gpus=2, role=[0, 1], cap=[650, 500], budget=1200,
        policy=dict(kind=1, threshold=0, step_w=50, dec_ceiling_w=600, cooldown_s=0.5, tick_s=1.0,
                    window_s=100.0, settle_s=0.3, reassign_s=3.0),
        slo=dict(ttft=100.0, tpot=[0.04, 0.001]), qps=1.0,
        trace=dict(s_unit=[0.0, 2.4], in_tok=[8192, 8192], out_tok=[2, 500], phase=[0, 1]),
        expect=dict(r0_tpot=tp0, first_move=[2.0, 1], caps_after=[600, 550]))


def boundary():
    """Scenario E — inclusive SLO test and the near-boundary band (A6: S:448,
    S:410 "ttft = 1.0 exactly -> met"; c.2 step 5: near iff |v - SLO| <=
    1e-9*SLO).  One 8192/128 request at t=0 on 1P1D @600/600: TTFT =
    0.4257796257796258, TPOT = 0.006072932901387327 (Appendix A)."""
    row = A["single_request"]["rows"][0]
    tt, tp = row["prefill_end"], row["tpot"]
    cases = []
    # (ttft_slo, tpot_slo, met, near)
    cases.append([tt, 1.0, 1, 1])                                   # equal -> met, near
    cases.append([math.nextafter(tt, 0.0), 1.0, 0, 1])              # SLO one ulp below -> missed
    cases.append([math.nextafter(tt, 1.0), 1.0, 1, 1])
    cases.append([tt * (1.0 + 2e-9), 1.0, 1, 0])                    # outside the near band
    cases.append([tt / (1.0 + 5e-10), 1.0, 0, 1])                   # inside the band, missed
    cases.append([1.0, tp, 1, 1])
    cases.append([1.0, math.nextafter(tp, 0.0), 0, 1])
    cases.append([1.0, tp * (1.0 + 2e-9), 1, 0])
    cases.append([1.0, tp * (1.0 - 2e-9), 0, 0])
    for c in cases:
        slo, v = (c[0], tt) if c[1] == 1.0 else (c[1], tp)
        assert (abs(v - slo) <= 1e-9 * slo) == bool(c[3])
    return dict(_doc=boundary.__doc__, n_gpus=2, role=[0, 1], cap=[600, 600], budget=1200,
                trace=dict(s_unit=[0.0], in_tok=[8192], out_tok=[128]), qps=1.0,
                ttft=tt, tpot=tp, cases=cases)


def main():
    out = dict(_source=__doc__, settle=settle(), window=window(), window_completion=window_completion(),
               move_gpu=move_gpu(),
               phase_switch=phase_switch(), boundary=boundary())
    with open(os.path.join(HERE, "mechanics.json"), "w") as f:
        json.dump(out, f, indent=1)
        f.write("\n")


if __name__ == "__main__":
    main()
