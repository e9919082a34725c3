"""Oracle pins for c.1 (model), p90, enumeration (a1) — CPU only.

Every pin comes from outside the oracle: SURVEY Appendix A/B values and SPEC
worked examples (tests/golden/appendix_a.json, with citations), closed-form
identities and an independent brute-force count.
"""
import json
import os

import numpy as np
import pytest

import oracle

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "appendix_a.json")))


def test_speedup_pins(model):
    for w, s in GOLD["speedup_prefill"].items():
        if w.startswith("_"):
            continue
        assert oracle.speedup(model, "prefill", int(w)) == s, w
    for w, s in GOLD["speedup_decode"].items():
        if w.startswith("_"):
            continue
        assert oracle.speedup(model, "decode", int(w)) == s, w


def test_speedup_paper_ratios(model):
    # P:289 "up to a 1.8x speedup for a 1.87x increase in power" (S:88 exact)
    assert oracle.speedup(model, "prefill", 750) / oracle.speedup(model, "prefill", 400) == 1.8
    assert 750 / 400 == pytest.approx(1.875)
    # P:289 decode plateau 1.3-1.5x
    assert 1.3 <= oracle.speedup(model, "decode", 750) <= 1.5
    # P:156 TTFT flattens after 700 W: marginal gain per W 700->750 below 400->700
    g1 = (oracle.speedup(model, "prefill", 700) - 1.0) / 300
    g2 = (oracle.speedup(model, "prefill", 750) - oracle.speedup(model, "prefill", 700)) / 50
    assert g2 < g1


def test_speedup_monotone_1w_grid(model):
    # non-decreasing over a 1 W grid; S:43 exact at anchors
    for ph in ("prefill", "decode"):
        vals = [oracle.speedup(model, ph, w) for w in range(400, 751)]
        assert all(b >= a for a, b in zip(vals, vals[1:]))
        for w, s in model[ph]:
            assert oracle.speedup(model, ph, w) == s


def test_latency_pins(model):
    for T, b, w, v in GOLD["prefill_lat"]["rows"]:
        assert oracle.prefill_lat(model, T, b, w) == v
    for n, w, v in GOLD["decode_lat"]["rows"]:
        assert oracle.decode_lat(model, n, w) == v
    for T, v in GOLD["kv_lat"]["rows"]:
        assert oracle.kv_lat(model, T) == v


def test_spec_approximate_examples(model):
    # SPEC S:56-57, S:64-66, S:72 printed approximations
    assert oracle.prefill_lat(model, 8192, 1, 750) == pytest.approx(0.350, abs=1e-3)
    assert oracle.prefill_lat(model, 8192, 1, 400) == pytest.approx(0.630, abs=1e-3)
    assert 0 < oracle.prefill_lat(model, 1, 1, 750) < 1e-3
    assert oracle.decode_lat(model, 32, 600) == pytest.approx(0.0114, abs=1e-4)
    assert oracle.decode_lat(model, 1, 400) == pytest.approx(0.00825, rel=1e-12)
    r = oracle.decode_lat(model, 32, 750) / oracle.decode_lat(model, 32, 600)
    assert r == pytest.approx(1.4 / 1.45, rel=1e-15)
    assert oracle.kv_lat(model, 8192) == pytest.approx(0.0229, abs=1e-4)


def test_kv_affine_and_bandwidth_halving(model):
    # S:74 doubling fabric bandwidth halves the variable term exactly; S:89 affine
    m2 = dict(model, bw=model["bw"] * 2)
    for T in (1, 500, 4096, 8192):
        v1 = oracle.kv_lat(model, T) - model["ovh"]
        v2 = oracle.kv_lat(m2, T) - model["ovh"]
        assert v2 == pytest.approx(v1 / 2, rel=1e-15)
    xs = [oracle.kv_lat(model, T) for T in (1000, 2000, 3000)]
    assert xs[2] - xs[1] == pytest.approx(xs[1] - xs[0], rel=1e-12)


def test_prefill_batch_form(model):
    # batch efficiency: same tokens split over b requests gets faster with b
    a = oracle.prefill_lat(model, 16384, 1, 600)
    b = oracle.prefill_lat(model, 16384, 2, 600)
    assert b == pytest.approx(a / 1.15, rel=1e-15)


def test_decode_ctx_term(model):
    m2 = dict(model, dec_per_ctx=1e-7)
    assert oracle.decode_lat(m2, 4, 600, ctx=10000) == pytest.approx(
        (0.008 + 0.00025 * 4 + 1e-7 * 10000) / 1.4, rel=1e-15)


def test_p90():
    assert oracle.p90([0.2 * k for k in range(1, 11)]) == pytest.approx(1.8)
    assert oracle.p90(list(range(1, 11))) == 9.0
    assert oracle.p90([3.5]) == 3.5
    assert oracle.p90([]) == 0.0
    rng = np.random.default_rng(1)
    for n in (1, 2, 9, 10, 11, 99, 100, 101, 257):
        v = rng.random(n)
        k = int(np.ceil(0.9 * n))                     # nearest rank, 1-based
        assert oracle.p90(v) == np.sort(v)[k - 1]


def _brute_count(N, B, step, exact, lo=400, hi=750):
    rows = []
    for x in range(1, N):
        for p in range(lo, hi + 1, step):
            for d in range(lo, hi + 1, step):
                t = x * p + (N - x) * d
                if (t == B) if exact else (t <= B):
                    rows.append((x, p, d))
    return rows


@pytest.mark.parametrize("row", GOLD["enumeration"]["rows"])
def test_enumeration_counts(row):
    N, B, step, exact, count = row
    got = oracle.enumerate_pool_uniform(N, B, 400, 750, step, exact)
    assert len(got) == count
    if N <= 8:
        assert [tuple(r) for r in got] == _brute_count(N, B, step, exact)


def test_enumeration_per_x_and_cfg1():
    got = oracle.enumerate_pool_uniform(8, 4800, 400, 750, 25)
    per_x = [int((got[:, 0] == x).sum()) for x in range(1, 8)]
    assert per_x == GOLD["enumeration"]["per_x_8_4800_25"]
    g1 = oracle.enumerate_pool_uniform(8, 4800, 400, 750, 100)
    assert int((g1[:, 0] == 4).sum()) == GOLD["enumeration"]["cfg1_4p4d_100w"]


def test_percentile_nearest_rank():
    # nearest rank = value at 1-based index ceil(p/100 * n)
    assert oracle.percentile(list(range(1, 11)), 90) == 9.0
    assert oracle.percentile([7.5], 50) == 7.5
    rng = np.random.default_rng(3)
    for n in (1, 2, 3, 10, 99, 100, 101, 2000):
        v = rng.random(n)
        for p in (50, 90, 99, 100):
            k = int(np.ceil(p / 100 * n))
            assert oracle.percentile(v, p) == np.sort(v)[k - 1]
