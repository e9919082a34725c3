"""GPU ↔ oracle parity for the context-growing decode cost (SURVEY §8(f) row 4,
reading A40) on every replay kernel: stage C (static, N ≤ 8), the joint
kernel (dynamic; static under PADSIM_JOINT and for N > 8) and the coalesced
kernel.  Records bit-exact (same closed-form boundary expression on both
sides)."""
import numpy as np
import pytest

from gpu_helpers import compare_records
from workloads import DEFAULT_MODEL, DEFAULT_SLO, PHASE_SLO, make_trace, policy, static_candidates

pytestmark = pytest.mark.gpu

GROW = dict(DEFAULT_MODEL, dec_per_ctx=2e-7, ctx_growth=1)


@pytest.fixture(scope="module")
def pkg():
    from paper_2601_12241_b200.build import build
    build()
    import paper_2601_12241_b200 as p
    return p


XPD = [(1, 750, 575), (3, 675, 525), (4, 600, 600), (6, 550, 700)]


@pytest.mark.parametrize("family", ["lb", "long_output"])
def test_growth_static_stage_c(pkg, family):
    role, cap = static_candidates(8, XPD)
    traces = [make_trace(family, 50 + s, 300) for s in range(2)]
    compare_records(traces, [0.5, 2.0, 4.0], GROW, role, cap, [policy("static")] * len(XPD), DEFAULT_SLO, 4800)


def test_growth_dynamic_and_coalesced(pkg):
    role, cap = static_candidates(8, [(4, 600, 600), (3, 600, 600), (4, 600, 600)])
    pols = [policy("dyn-both", cooldown_s=2.0), policy("dyn-power", step_w=25), policy("coalesced")]
    traces = [make_trace("phase", s, 600) for s in range(2)]
    compare_records(traces, [1.5, 3.0], GROW, role, cap, pols, PHASE_SLO, 4800)


def test_growth_joint_paths(pkg):
    # static through the joint kernel (PADSIM_JOINT) must equal stage C and the oracle
    role, cap = static_candidates(8, XPD[:2])
    traces = [make_trace("lb", 60, 300)]
    outs = []
    for joint in (False, True):
        ctx = pkg.Context(0)
        try:
            ctx.plan(traces, [1.0, 3.0], GROW, role, cap, [policy("static")] * 2, DEFAULT_SLO, 4800,
                     records=True, joint=joint)
            ctx.run()
            outs.append(ctx.fetch_records())
        finally:
            ctx.close()
    for k in outs[0]:
        assert np.array_equal(outs[0][k], outs[1][k]), k
    # N = 16: the shared-memory-table joint kernel (NG = 64)
    r16, c16 = static_candidates(16, [(8, 600, 600), (6, 700, 540)])
    compare_records([make_trace("lb", 61, 400)], [1.0, 2.5], GROW, r16, c16,
                    [policy("static"), policy("dyn-both", cooldown_s=2.0)], DEFAULT_SLO, 9600)
