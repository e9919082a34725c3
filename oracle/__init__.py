"""CPU oracle for the power-aware disaggregation what-if evaluator.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package.  The product (``paper_2601_12241_b200``) never imports it and shares
no code, header, table or constant with it; see ``padsim_oracle.h``.

This module is a thin ctypes wrapper (argument marshalling only) over the
plain C discrete-event simulator in ``padsim_oracle.c``.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "padsim_oracle.c")
_HDR = os.path.join(_HERE, "padsim_oracle.h")
_SO = os.path.join(_HERE, "libpadsim_oracle.so")
_lock = threading.Lock()
_lib = None

MAX_ANCHORS = 8
MAX_GPUS = 64


def build(force: bool = False) -> str:
    """Compile the oracle with -O2 -ffp-contract=off (no FMA, no fast-math)."""
    newest = max(os.path.getmtime(_SRC), os.path.getmtime(_HDR))
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < newest:
        cmd = ["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared",
               "-pthread", "-o", _SO + ".tmp", _SRC, "-lm"]
        subprocess.check_call(cmd)
        os.replace(_SO + ".tmp", _SO)
    return _SO


class Curve(C.Structure):
    _fields_ = [("n", C.c_int32), ("w", C.c_int32 * MAX_ANCHORS), ("s", C.c_double * MAX_ANCHORS)]


class Model(C.Structure):
    _fields_ = [("min_w", C.c_int32), ("max_w", C.c_int32), ("prefill", Curve), ("decode", Curve),
                ("rate", C.c_double), ("eff", C.c_double), ("dec_fixed", C.c_double),
                ("dec_per_seq", C.c_double), ("dec_per_ctx", C.c_double), ("kvb", C.c_double),
                ("bw", C.c_double), ("ovh", C.c_double), ("max_pb", C.c_int32),
                ("pb_tokens", C.c_int32), ("max_db", C.c_int32), ("slots", C.c_int32),
                ("chunk", C.c_int32), ("ctx_growth", C.c_int32)]


class Policy(C.Structure):
    _fields_ = [("kind", C.c_int32), ("threshold", C.c_int32), ("step_w", C.c_int32),
                ("dec_ceiling_w", C.c_int32), ("window_stamp", C.c_int32), ("cooldown_s", C.c_double), ("tick_s", C.c_double),
                ("window_s", C.c_double), ("settle_s", C.c_double), ("reassign_s", C.c_double)]


class Slo(C.Structure):
    _fields_ = [("ttft", C.c_double), ("tpot", C.c_double * 2)]


class Summary(C.Structure):
    _fields_ = [("met", C.c_int32), ("near_boundary", C.c_int32), ("n_req", C.c_int32),
                ("pad", C.c_int32), ("duration", C.c_double), ("goodput", C.c_double),
                ("events", C.c_int64), ("n_moves_power", C.c_int32), ("n_moves_gpu", C.c_int32),
                ("n_saturated", C.c_int32), ("n_flips", C.c_int32), ("avg_watts", C.c_double),
                ("qps_per_watt", C.c_double), ("sum_queue", C.c_double), ("sum_exec", C.c_double)]


class LogRec(C.Structure):
    _fields_ = [("t", C.c_double), ("type", C.c_int32), ("gpu", C.c_int32), ("a", C.c_int32),
                ("b", C.c_int32)]


class TickRec(C.Structure):
    _fields_ = [("t", C.c_double), ("ttft_stat", C.c_double), ("tpot_stat", C.c_double),
                ("ttft_slo", C.c_double), ("tpot_slo", C.c_double), ("q_prefill", C.c_int32),
                ("kind", C.c_int32), ("direction", C.c_int32), ("gpu", C.c_int32),
                ("load", C.c_int32 * MAX_GPUS), ("drained_empty", C.c_double * MAX_GPUS),
                ("role", C.c_uint8 * MAX_GPUS), ("draining", C.c_uint8 * MAX_GPUS),
                ("cmd", C.c_int32 * MAX_GPUS), ("eff", C.c_int32 * MAX_GPUS),
                ("raise_to", C.c_int32 * MAX_GPUS), ("last_move", C.c_double)]


class Log(C.Structure):
    _fields_ = [("cap", C.c_int32), ("n", C.c_int32), ("recs", C.POINTER(LogRec)),
                ("tcap", C.c_int32), ("tn", C.c_int32), ("ticks", C.POINTER(TickRec))]


class CtlState(C.Structure):
    _fields_ = [("role", C.c_uint8 * MAX_GPUS), ("draining", C.c_uint8 * MAX_GPUS),
                ("cmd", C.c_int32 * MAX_GPUS), ("n_gpus", C.c_int32),
                ("drain_pending", C.c_int32), ("last_move", C.c_double)]


class CtlObs(C.Structure):
    _fields_ = [("ttft_stat", C.c_double), ("tpot_stat", C.c_double), ("ttft_slo", C.c_double),
                ("tpot_slo", C.c_double), ("q_prefill", C.c_int32), ("load", C.c_int32 * MAX_GPUS)]


class CtlAction(C.Structure):
    _fields_ = [("kind", C.c_int32), ("direction", C.c_int32), ("gpu", C.c_int32),
                ("new_cap", C.c_int32 * MAX_GPUS)]


LOG_MOVE_POWER, LOG_MOVE_GPU, LOG_SATURATED, LOG_SETTLE, LOG_FLIP, LOG_BUDGET, LOG_ROLES, LOG_CAPS = \
    1, 2, 3, 4, 5, 6, 7, 8

_P = C.POINTER


def lib():
    global _lib
    with _lock:
        if _lib is None:
            build()
            L = C.CDLL(_SO)
            L.or_speedup.restype = C.c_double
            L.or_speedup.argtypes = [_P(Curve), C.c_int32]
            L.or_prefill_lat.restype = C.c_double
            L.or_prefill_lat.argtypes = [_P(Model), C.c_int64, C.c_int32, C.c_int32]
            L.or_decode_lat.restype = C.c_double
            L.or_decode_lat.argtypes = [_P(Model), C.c_int32, C.c_int64, C.c_int32]
            L.or_kv_lat.restype = C.c_double
            L.or_kv_lat.argtypes = [_P(Model), C.c_int32]
            L.or_p90.restype = C.c_double
            L.or_p90.argtypes = [_P(C.c_double), C.c_int32]
            L.or_percentile.restype = C.c_double
            L.or_percentile.argtypes = [_P(C.c_double), C.c_int32, C.c_int32]
            L.or_enumerate.restype = C.c_int
            L.or_enumerate.argtypes = [C.c_int32] * 6 + [_P(C.c_int32), C.c_int32, _P(C.c_int32)]
            L.or_replay.restype = C.c_int
            L.or_replay.argtypes = [_P(Model), C.c_int32, _P(C.c_uint8), _P(C.c_int32), _P(Policy),
                                    C.c_int32, _P(Slo), C.c_int32, _P(C.c_double), _P(C.c_int32),
                                    _P(C.c_int32), _P(C.c_uint8), C.c_double, _P(C.c_double),
                                    _P(C.c_double), _P(C.c_double), _P(C.c_double), _P(C.c_double),
                                    _P(C.c_double), _P(Summary), _P(Log)]
            L.or_evaluate.restype = C.c_int
            L.or_evaluate.argtypes = [_P(Model), C.c_int32, C.c_int32, _P(C.c_uint8), _P(C.c_int32),
                                      _P(Policy), C.c_int32, _P(C.c_int32), _P(Slo), C.c_int32, _P(C.c_int32),
                                      _P(_P(C.c_double)), _P(_P(C.c_int32)), _P(_P(C.c_int32)),
                                      _P(_P(C.c_uint8)), C.c_int32, _P(C.c_double), C.c_int32,
                                      _P(C.c_int64), _P(C.c_double), _P(C.c_int64), _P(C.c_int32),
                                      _P(C.c_int32), _P(C.c_double), _P(C.c_double)]
            L.or_met_for_slos.restype = C.c_int
            L.or_met_for_slos.argtypes = [C.c_int32, _P(C.c_double), _P(C.c_double), _P(C.c_uint8),
                                          C.c_int32, _P(Slo), _P(C.c_int32)]
            L.or_step_controller.restype = C.c_int
            L.or_step_controller.argtypes = [_P(Policy), _P(Model), C.c_int32, _P(CtlState),
                                             _P(CtlObs), C.c_double, _P(CtlAction)]
            _lib = L
    return _lib


# --------------------------------------------------------------------------
# marshalling helpers
# --------------------------------------------------------------------------
def _curve(anchors) -> Curve:
    c = Curve()
    c.n = len(anchors)
    for k, (w, s) in enumerate(anchors):
        c.w[k] = int(w)
        c.s[k] = float(s)
    return c


def make_model(m: dict) -> Model:
    M = Model()
    M.min_w, M.max_w = int(m["min_w"]), int(m["max_w"])
    M.prefill = _curve(m["prefill"])
    M.decode = _curve(m["decode"])
    for k in ("rate", "eff", "dec_fixed", "dec_per_seq", "dec_per_ctx", "kvb", "bw", "ovh"):
        setattr(M, k, float(m[k]))
    for k in ("max_pb", "pb_tokens", "max_db", "slots"):
        setattr(M, k, int(m[k]))
    M.chunk = int(m.get("chunk", 512))      # S:264 default chunk
    M.ctx_growth = int(m.get("ctx_growth", 0))   # A40
    return M


def make_policy(p: dict) -> Policy:
    P = Policy()
    for k in ("kind", "threshold", "step_w", "dec_ceiling_w"):
        setattr(P, k, int(p[k]))
    P.window_stamp = int(p.get("window_stamp", 0))
    for k in ("cooldown_s", "tick_s", "window_s", "settle_s", "reassign_s"):
        setattr(P, k, float(p[k]))
    return P


def make_slo(s: dict) -> Slo:
    S = Slo()
    S.ttft = float(s["ttft"])
    S.tpot[0] = float(s["tpot"][0])
    S.tpot[1] = float(s["tpot"][1])
    return S


def _ptr(a, ct):
    return a.ctypes.data_as(_P(ct))


def speedup(model: dict, phase: str, w: int) -> float:
    M = make_model(model)
    return lib().or_speedup(C.byref(M.prefill if phase == "prefill" else M.decode), int(w))


def prefill_lat(model: dict, tokens: int, b: int, w: int) -> float:
    return lib().or_prefill_lat(C.byref(make_model(model)), int(tokens), int(b), int(w))


def decode_lat(model: dict, n: int, w: int, ctx: int = 0) -> float:
    return lib().or_decode_lat(C.byref(make_model(model)), int(n), int(ctx), int(w))


def kv_lat(model: dict, tokens: int) -> float:
    return lib().or_kv_lat(C.byref(make_model(model)), int(tokens))


def p90(values) -> float:
    v = np.ascontiguousarray(values, dtype=np.float64)
    return lib().or_p90(_ptr(v, C.c_double), int(v.size))


def percentile(values, p: int) -> float:
    v = np.ascontiguousarray(values, dtype=np.float64)
    return lib().or_percentile(_ptr(v, C.c_double), int(v.size), int(p))


def enumerate_pool_uniform(n_gpus, budget_w, min_w, max_w, step_w, exact=False) -> np.ndarray:
    n = C.c_int32(0)
    rc = lib().or_enumerate(n_gpus, budget_w, min_w, max_w, step_w, int(exact), None, 0, C.byref(n))
    assert rc == 0
    out = np.zeros((max(n.value, 1), 3), dtype=np.int32)
    rc = lib().or_enumerate(n_gpus, budget_w, min_w, max_w, step_w, int(exact),
                            _ptr(out, C.c_int32), n.value, C.byref(n))
    assert rc == 0
    return out[: n.value]


class OracleError(RuntimeError):
    def __init__(self, rc):
        super().__init__(f"oracle rc={rc}")
        self.rc = rc


def _trace_arrays(tr):
    s = np.ascontiguousarray(tr["s_unit"], dtype=np.float64)
    i = np.ascontiguousarray(tr["in_tok"], dtype=np.int32)
    o = np.ascontiguousarray(tr["out_tok"], dtype=np.int32)
    p = np.ascontiguousarray(tr.get("phase", np.zeros(len(s), np.uint8)), dtype=np.uint8)
    return s, i, o, p


def replay(model: dict, role, cap, policy: dict, budget_w: int, slo: dict, trace: dict,
           qps_per_gpu: float, log_cap: int = 0, tick_cap: int = 0):
    """One replay; returns dict with per-request arrays, summary and log."""
    role = np.ascontiguousarray(role, dtype=np.uint8)
    cap = np.ascontiguousarray(cap, dtype=np.int32)
    s, i, o, p = _trace_arrays(trace)
    R = s.size
    outs = {k: np.zeros(max(R, 1), dtype=np.float64)
            for k in ("ttft", "tpot", "prefill_end", "completion", "transfer_end", "prefill_start")}
    sm = Summary()
    lg = None
    recs = None
    ticks = None
    if log_cap or tick_cap:
        recs = (LogRec * max(log_cap, 1))()
        ticks = (TickRec * tick_cap)() if tick_cap else None
        lg = Log(log_cap, 0, C.cast(recs, _P(LogRec)), tick_cap, 0,
                 C.cast(ticks, _P(TickRec)) if ticks is not None else None)
    M, P, S = make_model(model), make_policy(policy), make_slo(slo)
    rc = lib().or_replay(C.byref(M), role.size, _ptr(role, C.c_uint8), _ptr(cap, C.c_int32),
                         C.byref(P), int(budget_w), C.byref(S), R, _ptr(s, C.c_double),
                         _ptr(i, C.c_int32), _ptr(o, C.c_int32), _ptr(p, C.c_uint8),
                         float(qps_per_gpu), _ptr(outs["ttft"], C.c_double),
                         _ptr(outs["tpot"], C.c_double), _ptr(outs["prefill_end"], C.c_double),
                         _ptr(outs["completion"], C.c_double),
                         _ptr(outs["transfer_end"], C.c_double), _ptr(outs["prefill_start"], C.c_double),
                         C.byref(sm),
                         C.byref(lg) if lg is not None else None)
    if rc != 0:
        raise OracleError(rc)
    res = {k: v[:R] for k, v in outs.items()}
    res.update(met=sm.met, near_boundary=sm.near_boundary, duration=sm.duration,
               goodput=sm.goodput, events=sm.events, n_moves_power=sm.n_moves_power,
               n_moves_gpu=sm.n_moves_gpu, n_saturated=sm.n_saturated, n_flips=sm.n_flips,
               avg_watts=sm.avg_watts, qps_per_watt=sm.qps_per_watt, sum_queue=sm.sum_queue,
               sum_exec=sm.sum_exec)
    if lg is not None:
        n = min(lg.n, log_cap)
        res["log"] = [(recs[k].t, recs[k].type, recs[k].gpu, recs[k].a, recs[k].b) for k in range(n)]
        res["log_overflow"] = lg.n > log_cap
        if ticks is not None:
            n = len(role)
            res["ticks"] = [dict(t=x.t, ttft_stat=x.ttft_stat, tpot_stat=x.tpot_stat, ttft_slo=x.ttft_slo,
                                 tpot_slo=x.tpot_slo, q_prefill=x.q_prefill, kind=x.kind,
                                 direction=x.direction, gpu=x.gpu, load=list(x.load[:n]),
                                 drained_empty=list(x.drained_empty[:n]), role=list(x.role[:n]),
                                 draining=list(x.draining[:n]), cmd=list(x.cmd[:n]), eff=list(x.eff[:n]),
                                 raise_to=list(x.raise_to[:n]), last_move=x.last_move)
                            for x in ticks[: min(lg.tn, tick_cap)]]
            res["ticks_overflow"] = lg.tn > tick_cap
    return res


def evaluate(model: dict, role, cap, policies, budget_w: int, slo: dict, traces, qps,
             n_threads: int = 1, per_replay: bool = False, cand_budget_w=None):
    """Full evaluation: candidates x QPS x traces. role/cap: [C][N]."""
    role = np.ascontiguousarray(role, dtype=np.uint8)
    cap = np.ascontiguousarray(cap, dtype=np.int32)
    Cn, N = role.shape
    pols = (Policy * Cn)(*[make_policy(p) for p in policies])
    arrs = [_trace_arrays(t) for t in traces]
    S = len(arrs)
    nreq = np.array([a[0].size for a in arrs], dtype=np.int32)
    sp = (_P(C.c_double) * S)(*[_ptr(a[0], C.c_double) for a in arrs])
    ip = (_P(C.c_int32) * S)(*[_ptr(a[1], C.c_int32) for a in arrs])
    op = (_P(C.c_int32) * S)(*[_ptr(a[2], C.c_int32) for a in arrs])
    pp = (_P(C.c_uint8) * S)(*[_ptr(a[3], C.c_uint8) for a in arrs])
    qps = np.ascontiguousarray(qps, dtype=np.float64)
    Q = qps.size
    met = np.zeros((Cn, Q), np.int64)
    good = np.zeros((Cn, Q), np.float64)
    near = np.zeros((Cn, Q), np.int64)
    am = np.zeros(Q, np.int32)
    rm = np.zeros((Cn, Q, S), np.int32) if per_replay else None
    rg = np.zeros((Cn, Q, S), np.float64) if per_replay else None
    rd = np.zeros((Cn, Q, S), np.float64) if per_replay else None
    M, SL = make_model(model), make_slo(slo)
    cb = None if cand_budget_w is None else np.ascontiguousarray(cand_budget_w, dtype=np.int32)
    rc = lib().or_evaluate(C.byref(M), N, Cn, _ptr(role, C.c_uint8), _ptr(cap, C.c_int32), pols,
                           int(budget_w), _ptr(cb, C.c_int32) if cb is not None else None, C.byref(SL), S, _ptr(nreq, C.c_int32), sp, ip, op, pp, Q,
                           _ptr(qps, C.c_double), int(n_threads), _ptr(met, C.c_int64),
                           _ptr(good, C.c_double), _ptr(near, C.c_int64), _ptr(am, C.c_int32),
                           _ptr(rm, C.c_int32) if per_replay else None,
                           _ptr(rg, C.c_double) if per_replay else None,
                           _ptr(rd, C.c_double) if per_replay else None)
    if rc != 0:
        raise OracleError(rc)
    out = dict(met=met, goodput=good, near_boundary=near, argmax=am)
    if per_replay:
        out.update(rep_met=rm, rep_goodput=rg, rep_duration=rd)
    return out


def met_for_slos(ttft, tpot, phase, slos) -> np.ndarray:
    """Met counts of one replay's records against several SLO sets."""
    t1 = np.ascontiguousarray(ttft, dtype=np.float64)
    t2 = np.ascontiguousarray(tpot, dtype=np.float64)
    ph = np.ascontiguousarray(phase, dtype=np.uint8)
    arr = (Slo * max(len(slos), 1))(*[make_slo(s) for s in slos])
    out = np.zeros(max(len(slos), 1), np.int32)
    rc = lib().or_met_for_slos(t1.size, _ptr(t1, C.c_double), _ptr(t2, C.c_double), _ptr(ph, C.c_uint8),
                               len(slos), arr, _ptr(out, C.c_int32))
    if rc != 0:
        raise OracleError(rc)
    return out[: len(slos)]


def step_controller(policy: dict, model: dict, budget_w: int, state: dict, obs: dict, now: float):
    """Alg. 1 pure step; returns (action dict, new state dict)."""
    n = len(state["role"])
    st = CtlState()
    st.n_gpus = n
    for g in range(n):
        st.role[g] = int(state["role"][g])
        st.draining[g] = int(state.get("draining", [0] * n)[g])
        st.cmd[g] = int(state["cmd"][g])
    st.drain_pending = int(state.get("drain_pending", 0))
    st.last_move = float(state.get("last_move", 0.0))
    ob = CtlObs()
    ob.ttft_stat, ob.tpot_stat = float(obs["ttft_stat"]), float(obs["tpot_stat"])
    ob.ttft_slo, ob.tpot_slo = float(obs["ttft_slo"]), float(obs["tpot_slo"])
    ob.q_prefill = int(obs.get("q_prefill", 0))
    for g, l in enumerate(obs.get("load", [0] * n)):
        ob.load[g] = int(l)
    act = CtlAction()
    rc = lib().or_step_controller(C.byref(make_policy(policy)), C.byref(make_model(model)),
                                  int(budget_w), C.byref(st), C.byref(ob), float(now), C.byref(act))
    if rc != 0:
        raise OracleError(rc)
    a = dict(kind=act.kind, direction=act.direction, gpu=act.gpu,
             new_cap=[act.new_cap[g] for g in range(n)])
    s = dict(role=[st.role[g] for g in range(n)], draining=[st.draining[g] for g in range(n)],
             cmd=[st.cmd[g] for g in range(n)], drain_pending=st.drain_pending,
             last_move=st.last_move)
    return a, s
