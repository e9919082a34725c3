"""Thin ctypes binding over libpadsim.so (include/padsim.h).

Argument marshalling only: every step of the evaluation runs in the CUDA
kernels of the library.  There is no CPU fallback — if the library or a CUDA
device is missing, every call raises ``PadsimError``.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
# PADSIM_LIB: load another build of the same library (A/B experiments only)
LIB_PATH = os.environ.get("PADSIM_LIB") or os.path.join(HERE, "libpadsim.so")

MAX_GPUS = 64
MAX_ANCHORS = 8
MAX_PCT = 16
RECORDS = 1
JOINT = 2

STATUS = {0: "OK", -1: "EINVAL", -2: "ERANGE", -3: "EBUDGET", -4: "EROLE", -5: "EMODEL",
          -6: "EDOMAIN", -7: "ECUDA", -8: "ENOMEM"}


class PadsimError(RuntimeError):
    def __init__(self, rc: int, msg: str = ""):
        super().__init__(f"padsim {STATUS.get(rc, rc)} ({rc}): {msg}")
        self.rc = rc


class Trace(C.Structure):
    _fields_ = [("n_req", C.c_int32), ("s_unit", C.POINTER(C.c_double)),
                ("in_tok", C.POINTER(C.c_int32)), ("out_tok", C.POINTER(C.c_int32)),
                ("phase", C.POINTER(C.c_uint8))]


class Curve(C.Structure):
    _fields_ = [("n", C.c_int32), ("w", C.c_int32 * MAX_ANCHORS), ("s", C.c_double * MAX_ANCHORS)]


class Model(C.Structure):
    _fields_ = [("min_w", C.c_int32), ("max_w", C.c_int32), ("prefill", Curve), ("decode", Curve),
                ("prefill_base_rate", C.c_double), ("prefill_batch_eff", C.c_double),
                ("decode_fixed_s", C.c_double), ("decode_per_seq_s", C.c_double),
                ("decode_per_ctx_tok_s", C.c_double), ("kv_bytes_per_token", C.c_double),
                ("fabric_bw_Bps", C.c_double), ("transfer_overhead_s", C.c_double),
                ("max_prefill_batch", C.c_int32), ("prefill_token_budget", C.c_int32),
                ("max_decode_batch", C.c_int32), ("transfer_slots", C.c_int32),
                ("prefill_chunk_tokens", C.c_int32), ("decode_ctx_growth", C.c_int32)]


class Policy(C.Structure):
    _fields_ = [("kind", C.c_int32), ("queue_threshold", C.c_int32), ("power_step_w", C.c_int32),
                ("decode_ceiling_w", C.c_int32), ("window_stamp", C.c_int32), ("cooldown_s", C.c_double),
                ("tick_s", C.c_double),
                ("window_s", C.c_double), ("settle_s", C.c_double), ("reassign_s", C.c_double)]


class Candidates(C.Structure):
    _fields_ = [("n_gpus", C.c_int32), ("n_cand", C.c_int32), ("role", C.POINTER(C.c_uint8)),
                ("cap_w", C.POINTER(C.c_int32)), ("policy", C.POINTER(Policy))]


class Slo(C.Structure):
    _fields_ = [("ttft_s", C.c_double), ("tpot_s", C.c_double * 2)]


class Budget(C.Structure):
    _fields_ = [("budget_w", C.c_int32), ("cand_budget_w", C.POINTER(C.c_int32))]


class Result(C.Structure):
    _fields_ = [("met", C.POINTER(C.c_int64)), ("goodput", C.POINTER(C.c_double)),
                ("near_boundary", C.POINTER(C.c_int64)), ("argmax", C.POINTER(C.c_int32)),
                ("bad_index", C.c_int32)]


class DeviceResults(C.Structure):
    _fields_ = [("d_met", C.c_void_p), ("d_goodput", C.c_void_p), ("d_near", C.c_void_p),
                ("d_argmax", C.c_void_p), ("d_rep_met", C.c_void_p), ("d_rep_near", C.c_void_p),
                ("d_rep_duration", C.c_void_p), ("d_rep_goodput", C.c_void_p),
                ("d_rep_events", C.c_void_p), ("n_cand", C.c_int32), ("n_qps", C.c_int32),
                ("n_traces", C.c_int32), ("d_aux_events", C.c_void_p), ("n_aux_events", C.c_int32)]


class CtrlState(C.Structure):
    _fields_ = [("role", C.c_uint8 * MAX_GPUS), ("draining", C.c_uint8 * MAX_GPUS),
                ("cmd_cap_w", C.c_int32 * MAX_GPUS), ("eff_cap_w", C.c_int32 * MAX_GPUS),
                ("pending_raise_w", C.c_int32 * MAX_GPUS), ("settle_deadline_s", C.c_double * MAX_GPUS),
                ("flip_deadline_s", C.c_double * MAX_GPUS), ("n_gpus", C.c_int32),
                ("last_move_s", C.c_double)]


class WindowStats(C.Structure):
    _fields_ = [("ttft_stat_s", C.c_double), ("tpot_stat_s", C.c_double),
                ("ttft_slo_s", C.c_double), ("tpot_slo_s", C.c_double), ("rate_p", C.c_double),
                ("rate_d", C.c_double), ("q_prefill", C.c_int32), ("q_decode", C.c_int32),
                ("load", C.c_int32 * MAX_GPUS), ("drained_empty_s", C.c_double * MAX_GPUS)]


class Tuning(C.Structure):
    _fields_ = [("stage_a_threads", C.c_int32), ("stage_c_classes", C.c_int32),
                ("stage_c_batch_lists", C.c_int32), ("joint_threads", C.c_int32),
                ("joint_reg_cap", C.c_int32), ("joint_lanes_per_warp", C.c_int32),
                ("joint_after_stage_a", C.c_int32), ("serialize", C.c_int32),
                ("joint_groups", C.c_int32), ("wide_path", C.c_int32), ("wide_chunk", C.c_int32)]


TUNING_AUTO = dict(stage_a_threads=0, stage_c_classes=0, stage_c_batch_lists=-1, joint_threads=0,
                   joint_reg_cap=-1, joint_lanes_per_warp=0, joint_after_stage_a=-1, serialize=0,
                   joint_groups=-1, wide_path=-1, wide_chunk=0)


class Action(C.Structure):
    _fields_ = [("kind", C.c_int32), ("direction", C.c_int32), ("gpu", C.c_int32),
                ("new_cap_w", C.c_int32 * MAX_GPUS)]


EXPORTS = ["padsim_create", "padsim_destroy", "padsim_last_error", "padsim_version",
           "padsim_evaluate_allocations", "padsim_plan", "padsim_run", "padsim_fetch",
           "padsim_get_device_results", "padsim_fetch_replays", "padsim_fetch_records",
           "padsim_argmax_device", "padsim_step_controller", "padsim_controller_decide_device",
           "padsim_set_tuning", "padsim_launch_count", "padsim_static_path", "padsim_enumerate_pool_uniform",
           "padsim_replay_kernel_ms", "padsim_kernel_times_ms", "padsim_set_slo_sweep",
           "padsim_fetch_extras", "padsim_fetch_decomposition", "padsim_fetch_percentiles",
           "padsim_replay_records"]

_lib = None
_P = C.POINTER


def load(path: str = LIB_PATH):
    """Load libpadsim.so; raises if it is missing (no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise PadsimError(-7, f"{path} not built: run paper_2601_12241_b200.build.build()")
    L = C.CDLL(path)
    vp = C.c_void_p
    L.padsim_create.argtypes = [C.c_int32, vp, _P(vp)]
    L.padsim_destroy.argtypes = [vp]
    L.padsim_destroy.restype = None
    L.padsim_last_error.argtypes = [vp]
    L.padsim_last_error.restype = C.c_char_p
    L.padsim_version.restype = C.c_char_p
    L.padsim_evaluate_allocations.argtypes = [vp, _P(Trace), C.c_int32, _P(C.c_double), C.c_int32,
                                              _P(Model), _P(Candidates), _P(Slo), _P(Budget),
                                              _P(Result)]
    L.padsim_plan.argtypes = [vp, _P(Trace), C.c_int32, _P(C.c_double), C.c_int32, _P(Model),
                              _P(Candidates), _P(Slo), _P(Budget), C.c_uint32, _P(C.c_int32)]
    L.padsim_run.argtypes = [vp, vp]
    L.padsim_replay_records.argtypes = [vp, _P(Trace), C.c_double, _P(Model), _P(Candidates), _P(Slo),
                                        _P(Budget)] + [_P(C.c_double)] * 4
    L.padsim_fetch.argtypes = [vp, vp, _P(Result)]
    L.padsim_get_device_results.argtypes = [vp, _P(DeviceResults)]
    L.padsim_replay_kernel_ms.argtypes = [vp, _P(C.c_float)]
    L.padsim_kernel_times_ms.argtypes = [vp, _P(C.c_float)]
    L.padsim_set_slo_sweep.argtypes = [vp, _P(Slo), C.c_int32]
    L.padsim_fetch_extras.argtypes = [vp, vp, _P(C.c_int64), _P(C.c_double), _P(C.c_double),
                                      _P(C.c_int32)]
    L.padsim_fetch_replays.argtypes = [vp, vp, _P(C.c_int32), _P(C.c_int32), _P(C.c_double),
                                       _P(C.c_double), _P(C.c_int64)]
    L.padsim_fetch_records.argtypes = [vp, vp] + [_P(C.c_double)] * 5 + [_P(C.c_int32)]
    L.padsim_fetch_decomposition.argtypes = [vp, vp] + [_P(C.c_double)] * 4
    L.padsim_fetch_percentiles.argtypes = [vp, vp, _P(C.c_int32), C.c_int32, _P(C.c_double)]
    L.padsim_argmax_device.argtypes = [vp, vp, vp, vp, C.c_int32, C.c_int32, vp]
    L.padsim_step_controller.argtypes = [_P(Policy), _P(Budget), _P(Model), _P(CtrlState),
                                         _P(WindowStats), C.c_double, _P(Action)]
    L.padsim_controller_decide_device.argtypes = [vp, _P(Policy), _P(Budget), _P(Model), _P(CtrlState),
                                                  _P(WindowStats), C.c_double, _P(Action)]
    L.padsim_set_tuning.argtypes = [vp, _P(Tuning)]
    L.padsim_launch_count.argtypes = [vp, _P(C.c_int32)]
    L.padsim_static_path.argtypes = [vp, _P(C.c_int32)]
    L.padsim_enumerate_pool_uniform.argtypes = [C.c_int32] * 6 + [_P(C.c_int32), C.c_int32,
                                                                  _P(C.c_int32)]
    _lib = L
    return L


# ---------------------------------------------------------------------------
# marshalling
# ---------------------------------------------------------------------------
def _curve(anchors) -> Curve:
    c = Curve()
    c.n = len(anchors)
    for k, (w, s) in enumerate(anchors):
        c.w[k], c.s[k] = int(w), float(s)
    return c


def make_model(m: dict) -> Model:
    M = Model()
    M.min_w, M.max_w = int(m["min_w"]), int(m["max_w"])
    M.prefill, M.decode = _curve(m["prefill"]), _curve(m["decode"])
    M.prefill_base_rate, M.prefill_batch_eff = float(m["rate"]), float(m["eff"])
    M.decode_fixed_s, M.decode_per_seq_s = float(m["dec_fixed"]), float(m["dec_per_seq"])
    M.decode_per_ctx_tok_s = float(m["dec_per_ctx"])
    M.kv_bytes_per_token, M.fabric_bw_Bps = float(m["kvb"]), float(m["bw"])
    M.transfer_overhead_s = float(m["ovh"])
    M.max_prefill_batch, M.prefill_token_budget = int(m["max_pb"]), int(m["pb_tokens"])
    M.max_decode_batch, M.transfer_slots = int(m["max_db"]), int(m["slots"])
    M.prefill_chunk_tokens = int(m.get("chunk", 512))     # coalesced mode
    M.decode_ctx_growth = int(m.get("ctx_growth", 0))     # A40
    return M


def make_policy(p: dict) -> Policy:
    P = Policy()
    P.kind, P.queue_threshold = int(p["kind"]), int(p["threshold"])
    P.power_step_w, P.decode_ceiling_w = int(p["step_w"]), int(p["dec_ceiling_w"])
    P.window_stamp = int(p.get("window_stamp", 0))
    P.cooldown_s, P.tick_s, P.window_s = float(p["cooldown_s"]), float(p["tick_s"]), float(p["window_s"])
    P.settle_s, P.reassign_s = float(p["settle_s"]), float(p["reassign_s"])
    return P


def make_slo(s: dict) -> Slo:
    S = Slo()
    S.ttft_s = float(s["ttft"])
    S.tpot_s[0], S.tpot_s[1] = float(s["tpot"][0]), float(s["tpot"][1])
    return S


def _p(a, ct):
    return a.ctypes.data_as(_P(ct))


def make_budget(budget_w, cand_budget_w=None, keep=None) -> Budget:
    """padsim_budget: the node budget, or one budget per candidate."""
    if cand_budget_w is None:
        return Budget(int(budget_w), None)
    cb = np.ascontiguousarray(cand_budget_w, dtype=np.int32)
    if keep is not None:
        keep.objs.append(cb)
    b = Budget(int(budget_w), _p(cb, C.c_int32))
    b._cb = cb                                  # keep the array alive with the struct
    return b


class _Keep:
    """Holds numpy arrays alive while ctypes structs point into them."""

    def __init__(self):
        self.objs = []

    def arr(self, a, dtype):
        a = np.ascontiguousarray(a, dtype=dtype)
        self.objs.append(a)
        return a


def make_traces(traces, keep: _Keep):
    arr = (Trace * len(traces))()
    for k, t in enumerate(traces):
        s = keep.arr(t["s_unit"], np.float64)
        i = keep.arr(t["in_tok"], np.int32)
        o = keep.arr(t["out_tok"], np.int32)
        ph = keep.arr(t.get("phase", np.zeros(s.size, np.uint8)), np.uint8)
        arr[k].n_req = s.size
        arr[k].s_unit, arr[k].in_tok = _p(s, C.c_double), _p(i, C.c_int32)
        arr[k].out_tok, arr[k].phase = _p(o, C.c_int32), _p(ph, C.c_uint8)
    return arr


def make_candidates(role, cap, policies, keep: _Keep):
    role = keep.arr(role, np.uint8)
    cap = keep.arr(cap, np.int32)
    Cn, N = role.shape
    pols = (Policy * Cn)(*[make_policy(p) for p in policies])
    keep.objs.append(pols)
    cands = Candidates(N, Cn, _p(role, C.c_uint8), _p(cap, C.c_int32),
                       C.cast(pols, _P(Policy)))
    return cands


class Context:
    """One padsim_ctx bound to a CUDA device."""

    def __init__(self, device: int = 0, stream=None, tuning: dict | None = None):
        self.L = load()
        self.ptr = C.c_void_p()
        rc = self.L.padsim_create(int(device), C.c_void_p(stream or 0), C.byref(self.ptr))
        if rc != 0:
            raise PadsimError(rc, "padsim_create (no CUDA device?)")
        self.shape = None
        self._keep = None
        self.n_sweep = 0
        if tuning:
            self.set_tuning(tuning)

    def set_tuning(self, tuning: dict | None):
        """Launch-configuration overrides (padsim_set_tuning); results never depend on them."""
        t = dict(TUNING_AUTO, **(tuning or {}))
        self._check(self.L.padsim_set_tuning(self.ptr, C.byref(Tuning(**t))), "set_tuning")

    def static_path(self) -> str:
        """The planner's path for the static candidates: "none", "thread" (stageA_kernel /
        stageC_kernel), "warp" (the wide stages) or "joint" (padsim_static_path)."""
        n = C.c_int32(0)
        self._check(self.L.padsim_static_path(self.ptr, C.byref(n)), "static_path")
        return ("none", "thread", "warp", "joint")[n.value]

    def launch_count(self) -> int:
        n = C.c_int32(0)
        self._check(self.L.padsim_launch_count(self.ptr, C.byref(n)), "launch_count")
        return int(n.value)

    def decide_device(self, policy: dict, model: dict, budget_w: int, state: dict, stats: dict, now: float):
        """padsim_controller_decide_device: the kernel's Alg. 1 decision (no state change)."""
        st, ws = _ctrl_structs(state, stats)
        act = Action()
        self._check(self.L.padsim_controller_decide_device(
            self.ptr, C.byref(make_policy(policy)), C.byref(make_budget(budget_w)), C.byref(make_model(model)),
            C.byref(st), C.byref(ws), float(now), C.byref(act)), "controller_decide_device")
        n = st.n_gpus
        return dict(kind=act.kind, direction=act.direction, gpu=act.gpu,
                    new_cap=[act.new_cap_w[g] for g in range(n)])

    def close(self):
        if self.ptr:
            self.L.padsim_destroy(self.ptr)
            self.ptr = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, rc, what):
        if rc != 0:
            msg = self.L.padsim_last_error(self.ptr)
            raise PadsimError(rc, f"{what}: {msg.decode() if msg else ''}")

    def plan(self, traces, qps, model, role, cap, policies, slo, budget_w, records=False,
             joint=False, cand_budget_w=None):
        keep = _Keep()
        tr = make_traces(traces, keep)
        q = keep.arr(qps, np.float64)
        cands = make_candidates(role, cap, policies, keep)
        bad = C.c_int32(-1)
        self.n_sweep = 0                           # padsim_plan clears the SLO sweep
        rc = self.L.padsim_plan(self.ptr, tr, len(traces), _p(q, C.c_double), q.size,
                                C.byref(make_model(model)), C.byref(cands), C.byref(make_slo(slo)),
                                C.byref(make_budget(budget_w, cand_budget_w, keep)),
                                (RECORDS if records else 0) | (JOINT if joint else 0), C.byref(bad))
        if rc != 0:
            e = PadsimError(rc, self.L.padsim_last_error(self.ptr).decode())
            e.bad_index = bad.value
            raise e
        self.shape = (cands.n_cand, q.size, len(traces), max([t["s_unit"].size for t in traces] + [0]))
        self._keep = keep
        return self

    def run(self, stream=None):
        self._check(self.L.padsim_run(self.ptr, C.c_void_p(stream or 0)), "padsim_run")

    def fetch(self, stream=None):
        Cn, Q, S, _ = self.shape
        met = np.zeros((Cn, Q), np.int64)
        good = np.zeros((Cn, Q), np.float64)
        near = np.zeros((Cn, Q), np.int64)
        am = np.zeros(Q, np.int32)
        res = Result(_p(met, C.c_int64), _p(good, C.c_double), _p(near, C.c_int64),
                     _p(am, C.c_int32), -1)
        self._check(self.L.padsim_fetch(self.ptr, C.c_void_p(stream or 0), C.byref(res)), "fetch")
        return {"met": met, "goodput": good, "near_boundary": near, "argmax": am}

    def replay_kernel_ms(self) -> float:
        ms = C.c_float(0.0)
        self._check(self.L.padsim_replay_kernel_ms(self.ptr, C.byref(ms)), "replay_kernel_ms")
        return float(ms.value)

    def set_slo_sweep(self, slos):
        """Score up to 8 extra SLO sets on the same replays (padsim_set_slo_sweep)."""
        arr = (Slo * max(len(slos), 1))(*[make_slo(x) for x in slos])
        self._check(self.L.padsim_set_slo_sweep(self.ptr, arr, len(slos)), "set_slo_sweep")
        self.n_sweep = len(slos)

    def fetch_extras(self, stream=None):
        """SLO-sweep met counts, QPS/W, mean provisioned W, max QPS index at ≥80 %."""
        Cn, Q, S, _ = self.shape
        K = 8
        metk = np.zeros((Cn, Q, K), np.int64)
        qpw = np.zeros((Cn, Q), np.float64)
        watts = np.zeros((Cn, Q), np.float64)
        m80 = np.zeros((Cn, K + 1), np.int32)
        self._check(self.L.padsim_fetch_extras(self.ptr, C.c_void_p(stream or 0), _p(metk, C.c_int64),
                                               _p(qpw, C.c_double), _p(watts, C.c_double),
                                               _p(m80, C.c_int32)), "fetch_extras")
        n = getattr(self, "n_sweep", 0)
        return {"met_sweep": metk[:, :, :n], "qps_per_watt": qpw, "watts_sum": watts,
                "max_qps80": m80[:, : n + 1]}

    def kernel_times_ms(self):
        """[stage A, stage C, joint] device ms of the last run."""
        ms = (C.c_float * 3)()
        self._check(self.L.padsim_kernel_times_ms(self.ptr, ms), "kernel_times_ms")
        return [float(v) for v in ms]

    def fetch_replays(self, stream=None):
        Cn, Q, S, _ = self.shape
        out = {"met": np.zeros((Cn, Q, S), np.int32), "near_boundary": np.zeros((Cn, Q, S), np.int32),
               "duration": np.zeros((Cn, Q, S), np.float64), "goodput": np.zeros((Cn, Q, S), np.float64),
               "events": np.zeros((Cn, Q, S), np.int64)}
        self._check(self.L.padsim_fetch_replays(
            self.ptr, C.c_void_p(stream or 0), _p(out["met"], C.c_int32),
            _p(out["near_boundary"], C.c_int32), _p(out["duration"], C.c_double),
            _p(out["goodput"], C.c_double), _p(out["events"], C.c_int64)), "fetch_replays")
        return out

    def fetch_records(self, stream=None):
        Cn, Q, S, R = self.shape
        R = max(R, 1)
        names = ("ttft", "tpot", "prefill_end", "completion", "transfer_end")
        out = {k: np.zeros((Cn, Q, S, R), np.float64) for k in names}
        rmax = C.c_int32(0)
        self._check(self.L.padsim_fetch_records(self.ptr, C.c_void_p(stream or 0),
                                                *[_p(out[k], C.c_double) for k in names],
                                                C.byref(rmax)), "fetch_records")
        return out

    def fetch_decomposition(self, stream=None):
        """Fig. 6 split of TTFT: per-replay Σ queueing delay / Σ prefill
        execution time [C,Q,S] and their Σ over traces [C,Q]."""
        Cn, Q, S, _ = self.shape
        rq = np.zeros((Cn, Q, S), np.float64)
        re = np.zeros((Cn, Q, S), np.float64)
        sq = np.zeros((Cn, Q), np.float64)
        se = np.zeros((Cn, Q), np.float64)
        self._check(self.L.padsim_fetch_decomposition(self.ptr, C.c_void_p(stream or 0), _p(rq, C.c_double),
                                                      _p(re, C.c_double), _p(sq, C.c_double),
                                                      _p(se, C.c_double)), "fetch_decomposition")
        return {"rep_queue": rq, "rep_exec": re, "sum_queue": sq, "sum_exec": se}

    def fetch_percentiles(self, pcts, stream=None):
        """Nearest-rank TTFT/TPOT percentiles per replay (records mode):
        returns {"ttft": [C,Q,S,n_pct], "tpot": [C,Q,S,n_pct]}."""
        Cn, Q, S, _ = self.shape
        p = np.ascontiguousarray(np.asarray(pcts, np.int32))
        out = np.zeros((Cn, Q, S, 2, max(p.size, 1)), np.float64)
        self._check(self.L.padsim_fetch_percentiles(self.ptr, C.c_void_p(stream or 0), _p(p, C.c_int32),
                                                    int(p.size), _p(out, C.c_double)), "fetch_percentiles")
        return {"ttft": out[..., 0, :], "tpot": out[..., 1, :]}

    def device_results(self):
        d = DeviceResults()
        self._check(self.L.padsim_get_device_results(self.ptr, C.byref(d)), "device_results")
        return d

    def argmax_device(self, d_met_ptr: int, n_cand: int, n_qps: int, d_argmax_ptr: int, stream=None,
                      d_capsum_ptr: int | None = None):
        """Argmax kernel on a device met array [n_cand, n_qps] (d_capsum_ptr: device
        int32 Σcaps per candidate; None = the planned candidates')."""
        self._check(self.L.padsim_argmax_device(self.ptr, C.c_void_p(stream or 0), C.c_void_p(d_met_ptr),
                                                C.c_void_p(d_capsum_ptr or 0), n_cand, n_qps,
                                                C.c_void_p(d_argmax_ptr)), "argmax")



def _ctrl_structs(state: dict, stats: dict):
    n = len(state["role"])
    st = CtrlState()
    st.n_gpus = n
    for g in range(n):
        st.role[g] = int(state["role"][g])
        st.draining[g] = int(state.get("draining", [0] * n)[g])
        st.cmd_cap_w[g] = int(state["cmd"][g])
        st.eff_cap_w[g] = int(state.get("eff", state["cmd"])[g])
        st.pending_raise_w[g] = int(state.get("raise", [0] * n)[g])
        st.settle_deadline_s[g] = float(state.get("settle_deadline", [-1.0] * n)[g])
        st.flip_deadline_s[g] = float(state.get("flip_deadline", [-1.0] * n)[g])
    st.last_move_s = float(state.get("last_move", 0.0))
    ws = WindowStats()
    ws.ttft_stat_s, ws.tpot_stat_s = float(stats["ttft_stat"]), float(stats["tpot_stat"])
    ws.ttft_slo_s, ws.tpot_slo_s = float(stats["ttft_slo"]), float(stats["tpot_slo"])
    ws.q_prefill = int(stats.get("q_prefill", 0))
    for g, l in enumerate(stats.get("load", [0] * n)):
        ws.load[g] = int(l)
    for g in range(MAX_GPUS):
        ws.drained_empty_s[g] = -1.0
    for g, e in enumerate(stats.get("drained_empty", [-1.0] * n)):
        ws.drained_empty_s[g] = float(e)
    return st, ws


def step_controller(policy: dict, model: dict, budget_w: int, state: dict, stats: dict, now: float):
    """padsim_step_controller — pure host Alg. 1 step on the full node state.

    state: role, cmd, eff, raise, settle_deadline, flip_deadline, draining, last_move
    (lists of n_gpus; missing optional keys default to no pending transition).
    Returns (action dict, new state dict)."""
    L = load()
    st, ws = _ctrl_structs(state, stats)
    act = Action()
    rc = L.padsim_step_controller(C.byref(make_policy(policy)), C.byref(make_budget(budget_w)),
                                  C.byref(make_model(model)), C.byref(st), C.byref(ws), float(now),
                                  C.byref(act))
    if rc != 0:
        raise PadsimError(rc, "padsim_step_controller")
    n = st.n_gpus
    a = dict(kind=act.kind, direction=act.direction, gpu=act.gpu, new_cap=[act.new_cap_w[g] for g in range(n)])
    s = dict(role=[st.role[g] for g in range(n)], draining=[st.draining[g] for g in range(n)],
             cmd=[st.cmd_cap_w[g] for g in range(n)], eff=[st.eff_cap_w[g] for g in range(n)],
             raise_=[st.pending_raise_w[g] for g in range(n)],
             settle_deadline=[st.settle_deadline_s[g] for g in range(n)],
             flip_deadline=[st.flip_deadline_s[g] for g in range(n)], last_move=st.last_move_s)
    s["raise"] = s.pop("raise_")
    return a, s


def replay_records(trace, qps_per_gpu, model, role, cap, policy, slo, budget_w, device=0,
                   ctx: Context | None = None):
    """padsim_replay_records: one candidate (role[N], cap[N], policy) on one trace at
    one QPS point → per-request ttft, tpot, prefill_end, completion (marshalling only)."""
    own = ctx is None
    ctx = ctx or Context(device)
    try:
        keep = _Keep()
        tr = make_traces([trace], keep)
        cands = make_candidates(np.asarray(role).reshape(1, -1), np.asarray(cap).reshape(1, -1),
                                [policy], keep)
        R = int(np.asarray(trace["s_unit"]).size)
        out = {k: np.zeros(max(R, 1), np.float64) for k in ("ttft", "tpot", "prefill_end", "completion")}
        ctx._check(ctx.L.padsim_replay_records(ctx.ptr, tr, float(qps_per_gpu), C.byref(make_model(model)),
                                               C.byref(cands), C.byref(make_slo(slo)),
                                               C.byref(make_budget(budget_w, None, keep)),
                                               *[_p(out[k], C.c_double) for k in out]), "replay_records")
        ctx.shape = None                 # the ctx was re-planned for this one replay
        return {k: v[:R] for k, v in out.items()}
    finally:
        if own:
            ctx.close()


def evaluate_allocations(traces, qps, model, role, cap, policies, slo, budget_w, device=0,
                         ctx: Context | None = None, cand_budget_w=None):
    """One-shot padsim_evaluate_allocations (host buffers in, host results out).

    With ``ctx`` the call re-plans that context: its shape / kept arrays are
    updated so later fetch* calls on it size their buffers from this plan."""
    own = ctx is None
    ctx = ctx or Context(device)
    keep = _Keep()
    tr = make_traces(traces, keep)
    q = keep.arr(qps, np.float64)
    cands = make_candidates(role, cap, policies, keep)
    Cn, Q = cands.n_cand, q.size
    met = np.zeros((Cn, Q), np.int64)
    good = np.zeros((Cn, Q), np.float64)
    near = np.zeros((Cn, Q), np.int64)
    am = np.zeros(Q, np.int32)
    res = Result(_p(met, C.c_int64), _p(good, C.c_double), _p(near, C.c_int64), _p(am, C.c_int32), -1)
    rc = ctx.L.padsim_evaluate_allocations(ctx.ptr, tr, len(traces), _p(q, C.c_double), Q,
                                           C.byref(make_model(model)), C.byref(cands),
                                           C.byref(make_slo(slo)),
                                           C.byref(make_budget(budget_w, cand_budget_w, keep)),
                                           C.byref(res))
    if not own:                        # the context now holds this plan
        ctx.shape = (Cn, Q, len(traces), max([t["s_unit"].size for t in traces] + [0]))
        ctx._keep = keep
        ctx.n_sweep = 0
    try:
        if rc != 0:
            e = PadsimError(rc, ctx.L.padsim_last_error(ctx.ptr).decode())
            e.bad_index = res.bad_index
            raise e
        return {"met": met, "goodput": good, "near_boundary": near, "argmax": am}
    finally:
        if own:
            ctx.close()


def enumerate_pool_uniform(n_gpus, budget_w, min_w, max_w, step_w, exact=False) -> np.ndarray:
    L = load()
    n = C.c_int32(0)
    rc = L.padsim_enumerate_pool_uniform(n_gpus, budget_w, min_w, max_w, step_w, int(exact), None, 0,
                                         C.byref(n))
    if rc != 0:
        raise PadsimError(rc, "enumerate")
    out = np.zeros((max(n.value, 1), 3), np.int32)
    rc = L.padsim_enumerate_pool_uniform(n_gpus, budget_w, min_w, max_w, step_w, int(exact),
                                         _p(out, C.c_int32), n.value, C.byref(n))
    if rc != 0:
        raise PadsimError(rc, "enumerate")
    return out[: n.value]
