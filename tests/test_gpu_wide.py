"""GPU ↔ oracle parity of the wide-node factorized path (8 < N ≤ 64: one warp
per replay, wide_path.cuh) through the C ABI: per-request records bit-exact,
and identical to the joint kernel's (padsim_tuning.wide_path = 0) on the same
inputs.  Shapes follow BASELINE cfg 5 (64 GPUs, 38.4 kW, long-prompt /
long-output mixes), scaled down so the oracle finishes in seconds."""
import numpy as np
import pytest

import oracle
from gpu_helpers import compare_records
from workloads import DEFAULT_MODEL, DEFAULT_SLO, PHASE_SLO, make_trace, policy, static_candidates

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pkg():
    from paper_2601_12241_b200.build import build
    build()
    import paper_2601_12241_b200 as p
    return p


# x prefill GPUs at p W, N − x decode GPUs at d W: every worker-slot boundary of
# the two-workers-per-lane layout (x or N − x = 1, 31, 32, 33, 63)
XPD64 = [(1, 750, 575), (31, 600, 600), (32, 600, 600), (33, 700, 450), (63, 600, 400),
         (40, 675, 475), (10, 750, 550), (16, 400, 400)]


@pytest.mark.parametrize("chunk", [0, 1], ids=["auto-chunk", "chunk1"])
def test_wide_records_exact_n64(pkg, chunk):
    role, cap = static_candidates(64, XPD64)
    pols = [policy("static")] * len(XPD64)
    traces = [make_trace("long_prompt", 4, 700), make_trace("long_output", 5, 500),
              make_trace("lb_bursty", 6, 600)]
    qps = [0.25, 1.0, 2.5]
    n = compare_records(traces, qps, DEFAULT_MODEL, role, cap, pols, DEFAULT_SLO, 38400,
                        tuning=dict(wide_chunk=chunk))
    assert n == len(XPD64) * len(qps) * 1800


@pytest.mark.parametrize("N,B", [(16, 9600), (12, 7200), (40, 24000)])
def test_wide_records_exact_other_sizes(pkg, N, B):
    xpd = [(1, 700, 550), (N // 2, 600, 600), (N - 1, 600, 450), (N // 3, 750, 500)]
    role, cap = static_candidates(N, xpd)
    traces = [make_trace("lb", 11, 500), make_trace("long_output", 12, 300)]
    compare_records(traces, [0.5, 1.5, 4.0], DEFAULT_MODEL, role, cap, [policy("static")] * len(xpd),
                    DEFAULT_SLO, B)


@pytest.mark.parametrize("N,B", [(8, 4800), (4, 2400)])
def test_wide_path_forced_small_nodes(pkg, N, B):
    # padsim_tuning.wide_path = 1 sends N <= 8 static candidates down the wide path
    # (the planner's choice for tiny workloads such as cfg 1): records = oracle
    xpd = [(1, 700, 550), (N // 2, 600, 600), (N - 1, 600, 450), (N // 2, 400, 700)]
    role, cap = static_candidates(N, xpd)
    traces = [make_trace("lb", 13, 300), make_trace("phase", 14, 200)]
    for w in (1, 0):
        compare_records(traces, [0.5, 1.5, 4.0], DEFAULT_MODEL, role, cap, [policy("static")] * len(xpd),
                        PHASE_SLO, B, tuning=dict(wide_path=w))


def test_wide_non_uniform_caps_and_small_kv_buffer(pkg):
    # arbitrary per-GPU cap vectors and interleaved roles (the ABI takes full
    # vectors), a 4-slot KV buffer (waiting FIFO exercised), small batch limits
    rng = np.random.default_rng(7)
    N = 24
    role = np.zeros((3, N), np.uint8)
    cap = np.zeros((3, N), np.int32)
    for c in range(3):
        role[c] = rng.permutation(np.r_[np.zeros(9 + c, np.uint8), np.ones(N - 9 - c, np.uint8)])
        cap[c] = rng.integers(0, 15, N) * 25 + 400
    B = int(cap.sum(1).max())
    model = dict(DEFAULT_MODEL, slots=4, max_pb=3, max_db=8)
    traces = [make_trace("lb", 21, 400), make_trace("lb_bursty", 22, 400)]
    compare_records(traces, [1.0, 3.0], model, role, cap, [policy("static")] * 3, DEFAULT_SLO, B)


def test_wide_matches_joint_kernel_and_extras(pkg):
    # the same static N = 64 candidates through the wide stages and the joint kernel:
    # records, replays, SLO sweep, provisioned power and Fig. 6 sums identical
    role, cap = static_candidates(64, XPD64[:5])
    pols = [policy("static")] * 5
    traces = [make_trace("long_prompt", 31, 400), make_trace("long_output", 32, 300)]
    qps = [0.5, 2.0]
    sweep = [{"ttft": 0.5, "tpot": (0.025, 0.025)}, {"ttft": 2.0, "tpot": (0.08, 0.08)}]
    outs = []
    for wide in (1, 0):
        ctx = pkg.Context(0, tuning=dict(wide_path=wide))
        try:
            ctx.plan(traces, qps, DEFAULT_MODEL, role, cap, pols, DEFAULT_SLO, 38400, records=True)
            ctx.set_slo_sweep(sweep)
            ctx.run()
            outs.append((ctx.fetch(), ctx.fetch_replays(), ctx.fetch_records(), ctx.fetch_extras(),
                         ctx.fetch_decomposition()))
        finally:
            ctx.close()
    for a, b in zip(outs[0], outs[1]):
        for k in a:
            if k == "events":        # DES instants: the factorized path counts stage C's only
                continue
            if k in ("rep_queue", "rep_exec", "sum_queue", "sum_exec"):
                # Fig. 6 sums: stage A adds member by member, the joint kernel batch by
                # batch (A38; test_gpu_decomposition.py holds both to the oracle at 1e-9)
                assert np.allclose(np.asarray(a[k]), np.asarray(b[k]), rtol=1e-9, atol=0), k
                continue
            assert np.array_equal(np.asarray(a[k]), np.asarray(b[k])), k
    ref = oracle.evaluate(DEFAULT_MODEL, role, cap, pols, 38400, DEFAULT_SLO, traces, qps, n_threads=8)
    assert np.array_equal(outs[0][0]["met"], ref["met"])
    assert np.array_equal(outs[0][0]["argmax"], ref["argmax"])


def test_wide_with_dynamic_candidates(pkg):
    # static N = 16 candidates on the wide path next to dynamic ones on the joint kernel
    role, cap = static_candidates(16, [(8, 600, 600), (10, 600, 600), (8, 600, 600)])
    pols = [policy("static"), policy("static"), policy("dyn-both", cooldown_s=2.0)]
    traces = [make_trace("phase", 8, 800)]
    compare_records(traces, [1.5, 2.5], DEFAULT_MODEL, role, cap, pols, PHASE_SLO, 9600)


def test_wide_empty_and_single_request(pkg):
    role, cap = static_candidates(16, [(8, 600, 600), (1, 750, 560)])
    pols = [policy("static")] * 2
    empty = make_trace("lb", 0, 0)
    one = make_trace("lb", 1, 1)
    compare_records([empty, one, make_trace("lb", 2, 40)], [0.5, 8.0], DEFAULT_MODEL, role, cap, pols,
                    DEFAULT_SLO, 9600)


def test_planner_static_path_choice(pkg):
    # padsim_static_path: thread-per-replay stages for large N <= 8 workloads, the
    # warp-per-replay stages for small ones (<= 8 static replays per SM) and for
    # N > 8, the joint kernel when asked (records-only joint flag)
    role, cap = static_candidates(8, [(4, 600, 600), (3, 700, 540)])
    pols = [policy("static")] * 2
    small = [make_trace("lb", 1, 50)]
    ctx = pkg.Context(0)
    try:
        ctx.plan(small, [1.0], DEFAULT_MODEL, role, cap, pols, DEFAULT_SLO, 4800)
        assert ctx.static_path() == "warp"
        big = [make_trace("lb", s, 20) for s in range(16)]
        many = [0.1 * k for k in range(1, 81)]          # 2 x 80 x 16 = 2560 > 8 per SM
        ctx.plan(big, many, DEFAULT_MODEL, role, cap, pols, DEFAULT_SLO, 4800)
        assert ctx.static_path() == "thread"
        ctx.plan(small, [1.0], DEFAULT_MODEL, role, cap, pols, DEFAULT_SLO, 4800, joint=True)
        assert ctx.static_path() == "joint"
        r64, c64 = static_candidates(64, [(32, 600, 600)])
        ctx.plan(small, [1.0], DEFAULT_MODEL, r64, c64, [policy("static")], DEFAULT_SLO, 38400)
        assert ctx.static_path() == "warp"
        ctx.plan(small, [1.0], DEFAULT_MODEL, role, cap, [policy("dyn-both")] * 2, DEFAULT_SLO, 4800)
        assert ctx.static_path() == "none"
    finally:
        ctx.close()
    ctx = pkg.Context(0, tuning=dict(wide_path=0))
    try:
        ctx.plan(small, [1.0], DEFAULT_MODEL, role, cap, pols, DEFAULT_SLO, 4800)
        assert ctx.static_path() == "thread"
    finally:
        ctx.close()
