"""Oracle pins for the static replay (c.2) — CPU only.

Pins: hand-worked single- and two-request examples (golden/appendix_a.json),
the Lindley recursion (single FIFO server, batch 1, any trace), the low-load
limit, M/D/1 Pollaczek-Khinchine (statistical), SPEC routing/batching
examples, out=1.
"""
import json
import math
import os

import numpy as np
import pytest

import oracle
from workloads import DEFAULT_POLICY, DEFAULT_SLO, make_trace, static_candidates

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "appendix_a.json")))
BIG_SLO = {"ttft": 1e9, "tpot": (1e9, 1e9)}


def run(model, n, xpd, tr, qps=1.0, slo=DEFAULT_SLO, policy=DEFAULT_POLICY, budget=None):
    role, cap = static_candidates(n, [xpd])
    budget = budget if budget is not None else 750 * n
    return oracle.replay(model, role[0], cap[0], policy, budget, slo, tr, qps)


def trace(arr, ins, outs, phase=None):
    return dict(s_unit=np.asarray(arr, float), in_tok=np.asarray(ins, np.int32),
                out_tok=np.asarray(outs, np.int32),
                phase=np.zeros(len(arr), np.uint8) if phase is None else np.asarray(phase, np.uint8))


@pytest.mark.parametrize("row", GOLD["single_request"]["rows"])
def test_single_request(model, row):
    r = run(model, 8, (4, row["p"], row["d"]), trace([0.0], [row["in"]], [row["out"]]), budget=6000)
    assert r["prefill_end"][0] == row["prefill_end"]
    assert r["ttft"][0] == row["prefill_end"]
    assert r["transfer_end"][0] == row["transfer_end"]
    assert r["completion"][0] == row["completion"]
    assert r["tpot"][0] == row["tpot"]
    # closed form of an isolated request: completion = te + (out-1)*L (A14)
    assert r["completion"][0] == row["transfer_end"] + float(row["out"] - 1) * row["L"]


def test_T1_two_at_zero_batch_together(model):
    g = GOLD["T1"]
    r = run(model, 2, (1, 600, 600), trace([0.0, 0.0], [8192, 8192], [128, 128]))
    assert list(r["prefill_end"]) == [g["prefill_end"]] * 2
    assert list(r["transfer_end"]) == [g["transfer_end"]] * 2
    assert list(r["completion"]) == [g["completion"]] * 2
    assert list(r["tpot"]) == [g["tpot"]] * 2


def test_T2_queue_and_join(model):
    g = GOLD["T2"]
    # 1P1D, q=1 -> lambda = 2, s_unit 0.2 -> arrival 0.1
    r = run(model, 2, (1, 600, 600), trace([0.0, 0.2], [8192, 8192], [128, 128]))
    assert r["prefill_end"][0] == g["pe0"] and r["prefill_end"][1] == g["pe1"]
    assert r["transfer_end"][1] == g["te1"]
    assert r["completion"][0] == g["comp0"] and r["tpot"][0] == g["tpot0"]
    assert r["completion"][1] == g["comp1"] and r["tpot"][1] == g["tpot1"]
    # independent re-derivation of the join step (first boundary >= te1)
    te0 = r["transfer_end"][0]
    L1 = oracle.decode_lat(model, 1, 600)
    k = math.ceil((g["te1"] - te0) / L1)
    assert k == g["join_k"] and te0 + float(k) * L1 == g["join_t"]


def test_out1_completes_at_transfer_end(model):
    r = run(model, 8, (4, 600, 600), trace([0.0, 0.5], [8192, 100], [1, 1]))
    assert np.array_equal(r["completion"], r["transfer_end"])
    assert np.all(r["tpot"] == 0.0)
    assert r["met"] == 2


def test_lindley_single_server_batch1(model):
    # x=1, max_prefill_batch=1: pe_i = max(a_i, pe_{i-1}) + S_i exactly (FIFO single server)
    m = dict(model, max_pb=1)
    tr = make_trace("lb", 3, 400)
    for q in (0.3, 1.0, 3.0):
        r = run(m, 2, (1, 650, 550), tr, qps=q)
        inv = 1.0 / (q * 2.0)
        a = tr["s_unit"] * inv
        pe_prev = -math.inf
        for i in range(len(a)):
            start = max(a[i], pe_prev)
            pe = start + oracle.prefill_lat(m, int(tr["in_tok"][i]), 1, 650)
            assert r["prefill_end"][i] == pe, (q, i)
            pe_prev = pe


def test_low_load_limit(model):
    # gaps far larger than any service: TTFT = prefill_latency alone
    tr = trace(np.arange(1, 21) * 1000.0, np.full(20, 4096), np.full(20, 32))
    r = run(model, 8, (3, 700, 500), tr, qps=1.0 / 8)
    S = oracle.prefill_lat(model, 4096, 1, 700)
    for i in range(20):
        a = tr["s_unit"][i] * (1.0 / ((1.0 / 8) * 8.0))
        assert r["prefill_end"][i] == a + S
        assert r["ttft"][i] == (a + S) - a


@pytest.mark.slow
@pytest.mark.parametrize("lam", [0.5, 1.0, 1.5])
def test_md1_pollaczek_khinchine(model, lam):
    # 1P, batch 1, deterministic 8192-token prompts at 600 W: M/D/1 waiting time
    m = dict(model, max_pb=1)
    S = oracle.prefill_lat(m, 8192, 1, 600)
    rho = lam * S
    wq = lam * S * S / (2 * (1 - rho))
    R = 400_000
    g = np.random.default_rng(7)
    s_unit = np.cumsum(g.standard_exponential(R))
    tr = trace(s_unit, np.full(R, 8192), np.ones(R, np.int32))
    r = run(m, 2, (1, 600, 600), tr, qps=lam / 2.0, slo=BIG_SLO)
    w = (r["ttft"] - S)[R // 20:]          # drop warm-up
    nb = 100
    means = w[: (len(w) // nb) * nb].reshape(nb, -1).mean(axis=1)
    se = means.std(ddof=1) / math.sqrt(nb)
    assert abs(w.mean() - wq) < 4 * se + 1e-12, (w.mean(), wq, se)


def test_spec_routing_example(model):
    # outstanding [1000, 200, 200, 5000] -> worker 1 (least, lowest id)
    tr = trace([0.0, 0.0, 0.0, 0.0, 1e-6], [1000, 200, 200, 5000, 300], [2] * 5)
    r = run(model, 8, (4, 600, 600), tr, qps=1.0 / 8)
    s200 = oracle.prefill_lat(model, 200, 1, 600)
    # request 4 waits behind worker 1's 200-token batch
    assert r["prefill_end"][1] == s200
    assert r["prefill_end"][4] == s200 + oracle.prefill_lat(model, 300, 1, 600)
    # S:219 all queues empty -> worker 0 (request 0 starts at once on worker 0)
    assert r["prefill_end"][0] == oracle.prefill_lat(model, 1000, 1, 600)


def test_spec_batching_example(model):
    # queue [8192, 8192, 512], budget 16384, max 4 -> batch of the first two
    m = dict(model, max_pb=4)
    tr = trace([0.0, 0.0, 0.0], [8192, 8192, 512], [2, 2, 2])
    r = run(m, 2, (1, 600, 600), tr)
    b = oracle.prefill_lat(m, 16384, 2, 600)
    assert r["prefill_end"][0] == b and r["prefill_end"][1] == b
    assert r["prefill_end"][2] == b + oracle.prefill_lat(m, 512, 1, 600)
    # S:228 max_prefill_batch=1 -> singleton batches
    m1 = dict(model, max_pb=1)
    r1 = run(m1, 2, (1, 600, 600), tr)
    assert r1["prefill_end"][0] == oracle.prefill_lat(m1, 8192, 1, 600)


def test_two_at_zero_on_2p(model):
    # two arrivals at t=0 on 2P -> workers 0 and 1, each alone
    tr = trace([0.0, 0.0], [8192, 8192], [128, 128])
    r = run(model, 4, (2, 600, 600), tr, qps=1.0)
    s = oracle.prefill_lat(model, 8192, 1, 600)
    assert list(r["prefill_end"]) == [s, s]


def test_transfer_buffer_bound(model):
    # 48 one-token-output prompts finish prefill at one instant (4 identical
    # batches of 12): 32 transfers start at once, the other 16 wait for a slot
    # and start when the first 32 end ("request buffer of size 32")
    n = 48
    tr = trace(np.zeros(n), np.full(n, 64), np.ones(n, np.int32))
    r = run(model, 8, (4, 600, 600), tr, qps=1.0)
    pe, te = r["prefill_end"], r["transfer_end"]
    assert np.all(pe == pe[0])
    kv = oracle.kv_lat(model, 64)
    first = pe[0] + kv
    assert int((te == first).sum()) == 32
    assert int((te == first + kv).sum()) == 16
    assert np.array_equal(r["completion"], te)
