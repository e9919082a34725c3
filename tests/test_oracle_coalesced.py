"""Oracle pins for the coalesced (non-disaggregated, chunked-prefill) baseline
replay — SURVEY §8(f) row 3 (SPEC coalesced_step S:262–269; readings
A33–A37 in DESIGN.md §3).  CPU only.

Pins come from outside the oracle: Appendix A constants (tests/golden), the
SPEC worked examples of S:266–268 (chunk count; fused step = sum of the two
component latencies; pure decode step), closed forms for an isolated request,
and invariants."""
import json
import os

import numpy as np
import pytest

import oracle
from workloads import DEFAULT_MODEL, DEFAULT_SLO, make_trace, policy

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "appendix_a.json")))
CO = policy("coalesced")
ROLE2 = np.array([0, 1], np.uint8)


def _tr(s_unit, ins, outs):
    n = len(s_unit)
    return {"s_unit": np.asarray(s_unit, float), "in_tok": np.asarray(ins, np.int32),
            "out_tok": np.asarray(outs, np.int32), "phase": np.zeros(n, np.uint8)}


def _rep(tr, cap=(600, 600), model=DEFAULT_MODEL, qps=0.5, role=ROLE2, budget=4800):
    # qps 0.5 on N = 2 GPUs: inv_lam = 1/(0.5*2) = 1.0, arrivals = s_unit exactly
    return oracle.replay(model, role, np.asarray(cap, np.int32), CO, budget, DEFAULT_SLO, tr, qps)


def _pl(T, w):
    # Appendix A: s_pre(600) = 1.48, s_pre(750) = 1.8 (D1 anchors); rate 13000 tok/s
    s = {600: 1.48, 750: 1.8}[w]
    return (T / 13000.0) / s


def _dl(n, w):
    s = {600: 1.4, 750: 1.45}[w]
    return (0.008 + 0.00025 * n) / s


def test_isolated_request_chunk_ge_prompt_matches_appendix_a():
    # one chunk covers the prompt: prefill_end = prefill_lat(8192,1,600) (Appendix A), no
    # KV transfer (A33), then 127 decode steps of L = decode_lat(1,600) (Appendix A)
    m = dict(DEFAULT_MODEL, chunk=8192)
    o = _rep(_tr([0.0], [8192], [128]), model=m)
    pe = [v for T, b, w, v in GOLD["prefill_lat"]["rows"] if (T, b, w) == (8192, 1, 600)][0]
    L = [v for n, w, v in GOLD["decode_lat"]["rows"] if (n, w) == (1, 600)][0]
    assert o["prefill_end"][0] == pe
    assert o["transfer_end"][0] == pe
    assert o["completion"][0] == pe + 127.0 * L
    assert o["tpot"][0] == pytest.approx(L, rel=1e-14)


def test_chunk_count_and_closed_form():
    # a 1024-token prompt with chunk 512 and no decodes takes 2 chunk steps
    o = _rep(_tr([0.0], [1024], [5]))
    assert o["events"] == 1 + 2 + 4          # arrival, 2 chunk steps, 4 decode steps
    # Σ chunk latencies = the whole prompt's latency up to rounding (linear in T)
    assert o["ttft"][0] == pytest.approx(_pl(1024, 600), rel=1e-14)
    assert o["ttft"][0] == _pl(512, 600) + _pl(512, 600)
    L = _dl(1, 600)
    assert o["completion"][0] - o["prefill_end"][0] == pytest.approx(4 * L, rel=1e-13)
    # ragged last chunk: 1300 = 512 + 512 + 276
    o2 = _rep(_tr([0.0], [1300], [1]))
    assert o2["events"] == 1 + 3
    assert o2["ttft"][0] == pytest.approx(_pl(1300, 600), rel=1e-14)
    assert o2["tpot"][0] == 0.0 and o2["completion"][0] == o2["prefill_end"][0]   # out = 1 (A7)


def test_fused_step_is_sum_of_component_latencies():
    # a chunk step with active decodes lasts prefill_lat(chunk) + decode_lat(n).
    # r0 (512 in, 10 out) arrives at 0 on GPU 0; r1 (512 in, 3 out) arrives mid-way through
    # r0's first decode step; both GPUs have 0 outstanding prompt tokens, so r1 also goes to
    # GPU 0 (lowest id, A34) and its chunk starts at r0's next boundary, fused with r0.
    pl, L1, L2 = _pl(512, 600), _dl(1, 600), _dl(2, 600)
    a1 = pl + 0.5 * L1
    o = _rep(_tr([0.0, a1], [512, 512], [10, 3]))
    pe0 = pl
    b1 = pe0 + L1                       # r0's first decode step (segment from pe0)
    pe1 = b1 + (pl + L1)                # fused step: chunk of r1 + decode of r0
    assert o["prefill_end"][0] == pe0
    assert o["prefill_end"][1] == pe1
    # then n = 2 until r1 leaves after 2 more steps; r0 has 10-1-2-2 = 5 steps left at n = 1
    c1 = pe1 + 2.0 * L2
    assert o["completion"][1] == c1
    assert o["completion"][0] == c1 + 5.0 * L1
    # queueing delay of r1 = wait for the boundary; exec = the fused step
    assert o["sum_queue"] == pytest.approx(b1 - a1, rel=1e-12)
    assert o["sum_exec"] == pytest.approx(pl + (pl + L1), rel=1e-12)


def test_pure_decode_and_routing_by_outstanding_tokens():
    # r1 arrives while r0's prompt is outstanding on GPU 0 → GPU 1 (A34); both isolated
    o = _rep(_tr([0.0, 0.001], [4096, 512], [2, 2]))
    assert o["ttft"][1] == pytest.approx(_pl(512, 600), rel=1e-14)
    assert o["ttft"][0] == pytest.approx(_pl(4096, 600), rel=1e-14)
    # no prefill pending → a pure decode step of decode_lat(1)
    assert o["completion"][1] == o["prefill_end"][1] + _dl(1, 600)


def test_roles_ignored_and_cap_speedup():
    tr = make_trace("lb", 5, 300)
    a = _rep(tr, cap=(600, 600), role=np.array([0, 1], np.uint8))
    b = _rep(tr, cap=(600, 600), role=np.array([1, 1], np.uint8))
    for k in ("ttft", "tpot", "completion"):
        assert np.array_equal(a[k], b[k])
    lo = _rep(make_trace("lb", 6, 1), cap=(600, 600))
    hi = _rep(make_trace("lb", 6, 1), cap=(750, 750), budget=6000)
    # isolated request: TTFT scales exactly with 1/s_pre (1.8/1.48)
    assert lo["ttft"][0] / hi["ttft"][0] == pytest.approx(1.8 / 1.48, rel=1e-12)


@pytest.mark.parametrize("family", ["lb", "lb_bursty", "long_output"])
def test_invariants_random(family):
    N = 8
    role = np.zeros(N, np.uint8)
    cap = np.full(N, 600, np.int32)
    tr = make_trace(family, 2, 600)
    for q in (0.5, 2.0, 4.0):
        o = oracle.replay(DEFAULT_MODEL, role, cap, CO, 4800, DEFAULT_SLO, tr, q)
        a = tr["s_unit"] * (1.0 / (q * N))
        R = tr["s_unit"].size
        assert np.all(np.isfinite(o["completion"]))                      # conservation
        # TTFT at least the whole prompt's chunked latency at this cap
        lower = (tr["in_tok"] / 13000.0) / 1.48
        assert np.all(o["ttft"] >= lower * (1 - 1e-12))
        assert np.all(o["completion"] >= o["prefill_end"])
        assert np.array_equal(o["transfer_end"], o["prefill_end"])      # A33
        # decomposition: TTFT = queueing + prefill execution span (no transfer term)
        assert o["sum_queue"] + o["sum_exec"] == pytest.approx(float(np.sum(o["ttft"])), rel=1e-9)
        assert np.all(o["prefill_start"] >= a)
        # every decode step is at least decode_lat(1) at 600 W
        multi = tr["out_tok"] > 1
        assert np.all(o["tpot"][multi] >= _dl(1, 600) * (1 - 1e-12))
        assert o["met"] <= R


def test_backpressure_with_load():
    N = 8
    role = np.zeros(N, np.uint8)
    cap = np.full(N, 600, np.int32)
    tr = make_trace("lb", 9, 1500)
    t = [float(np.mean(oracle.replay(DEFAULT_MODEL, role, cap, CO, 4800, DEFAULT_SLO, tr, q)["ttft"]))
         for q in (0.25, 1.0, 3.0)]
    assert t[0] < t[1] < t[2]


def test_validation():
    tr = _tr([0.0], [100], [2])
    with pytest.raises(Exception):
        _rep(tr, cap=(750, 750), budget=1200)                 # Σ caps > budget
    with pytest.raises(Exception):
        _rep(tr, model=dict(DEFAULT_MODEL, chunk=0))          # chunk ≥ 1
