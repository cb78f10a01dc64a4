"""ctypes wrapper of the fp64 CPU oracle (oracle/idm_oracle.c).

TEST INFRASTRUCTURE ONLY -- may be imported solely by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / ``--impl reference`` legs.  It shares no code with the CUDA path
(paper_2412_16750_b200/) and imports nothing from it.

Every function here is argument marshalling around the C oracle; the arithmetic and its
citations to the paper (PAPER.md lines) live in idm_oracle.c.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "idm_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

NPAR = 6
PARAM_NAMES = ("a_max", "a_pref", "s_min", "T_pref", "v_targ", "delta")

_dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_ip = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (plain -O2, no fast-math, no FMA contraction)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(
            ["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-ffp-contract=off",
             "-fno-fast-math", _SRC, "-o", tmp, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        L = C.CDLL(build())
        d, i64, i32, vp = C.c_double, C.c_int64, C.c_int32, C.c_void_p
        L.ora_softplus.restype = d
        L.ora_softplus.argtypes = [d]
        L.ora_sigmoid.restype = d
        L.ora_sigmoid.argtypes = [d]
        L.ora_optimal_spacing.restype = d
        L.ora_optimal_spacing.argtypes = [d] * 6
        L.ora_accel.restype = d
        L.ora_accel.argtypes = [_dp, d, d, d, C.c_int, d, d]
        L.ora_accel_partials.restype = None
        L.ora_accel_partials.argtypes = [_dp, d, d, d, C.c_int, C.c_int, d, d, _dp]
        L.ora_rollout.restype = C.c_int
        L.ora_rollout.argtypes = [i64, _ip, _dp, _dp, _dp, _dp, i64, i32, d, d, d, _dp, _dp, vp]
        L.ora_loss.restype = d
        L.ora_loss.argtypes = [C.c_int, i64, i32, _dp, _dp, vp, vp, _dp]
        L.ora_backward.restype = C.c_int
        L.ora_backward.argtypes = [i64, _ip, _dp, _dp, i64, i32, d, d, d, _dp, _dp, _dp, _dp,
                                   vp, vp, vp, vp, vp]
        L.ora_rollout_tangent.restype = C.c_int
        L.ora_rollout_tangent.argtypes = [i64, _ip, _dp, _dp, _dp, _dp, i64, i32, d, d, d,
                                          vp, vp, vp, _dp, _dp]
        L.ora_rollout_vl.restype = C.c_int
        L.ora_rollout_vl.argtypes = [i64, _dp, _dp, _dp, i64, i32, d, d, d, _dp, _dp, _dp, _dp]
        L.ora_backward_vl.restype = C.c_int
        L.ora_backward_vl.argtypes = [i64, _dp, i64, i32, d, d, d, _dp, _dp, _dp, _dp, _dp, _dp,
                                      vp, _dp, _dp, vp, vp, vp, vp]
        L.ora_rollout_vl_tangent.restype = C.c_int
        L.ora_rollout_vl_tangent.argtypes = [i64, _dp, _dp, _dp, i64, i32, d, d, d, _dp, _dp,
                                             vp, vp, vp, vp, vp, _dp, _dp]
        L.ora_lr.restype = d
        L.ora_lr.argtypes = [i32, i32, d, d]
        L.ora_adam_step.restype = None
        L.ora_adam_step.argtypes = [i64, _dp, _dp, _dp, _dp, i32, d, d, d, d, vp]
        L.ora_project.restype = None
        L.ora_project.argtypes = [i64, _dp]
        _lib = L
    return _lib


def _f64(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


def _ptr(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


class OracleError(RuntimeError):
    pass


# ------------------------------------------------------------------ scalar API
def softplus(x: float) -> float:
    return lib().ora_softplus(float(x))


def sigmoid(x: float) -> float:
    return lib().ora_sigmoid(float(x))


def optimal_spacing(a_max, a_pref, s_min, T_pref, v, dv) -> float:
    return lib().ora_optimal_spacing(a_max, a_pref, s_min, T_pref, v, dv)


def accel(theta, v, dp, dv, has_leader=True, dt=0.1, a_min=-10.0) -> float:
    return lib().ora_accel(_f64(theta), v, dp, dv, int(has_leader), dt, a_min)


def accel_partials(theta, v, dp, dv, has_leader=True, dp_clamped=False, dt=0.1, a_min=-10.0):
    """Returns (a*, da/dv|dv, da/ddp, da/ddv, da/dtheta[6])."""
    out = np.zeros(10)
    lib().ora_accel_partials(_f64(theta), v, dp, dv, int(has_leader), int(dp_clamped), dt,
                             a_min, out)
    return out[0], out[1], out[2], out[3], out[4:].copy()


# ------------------------------------------------------------------ array API
def leader_from_lanes(lane_offsets) -> np.ndarray:
    """Leader index h(i) of lane-sorted vehicles: i+1 inside the lane, -1 for
    the lane head (free road, reading R#8)."""
    off = np.asarray(lane_offsets, dtype=np.int64)
    n = int(off[-1])
    h = np.arange(1, n + 1, dtype=np.int32)
    heads = off[1:] - 1
    heads = heads[off[1:] > off[:-1]]
    h[heads] = -1
    return h


def _params2d(params, n):
    p = _f64(params)
    if p.ndim == 1:
        p = p.reshape(NPAR, 1)
    assert p.shape[0] == NPAR and p.shape[1] in (1, n), p.shape
    return np.ascontiguousarray(p)


def rollout(leader, length, p0, v0, params, K, dt=0.1, a_min=-10.0, eps_gap=0.1,
            want_accel=False):
    """Eq. 3 rollout.  Returns P, V [(K+1), n] (and A [K, n] if want_accel)."""
    leader = np.ascontiguousarray(leader, dtype=np.int32)
    n = leader.shape[0]
    prm = _params2d(params, n)
    P = np.empty((K + 1, n))
    V = np.empty((K + 1, n))
    A = np.empty((K, n)) if want_accel else None
    rc = lib().ora_rollout(n, leader, _f64(length), _f64(p0), _f64(v0), prm, prm.shape[1],
                           K, dt, a_min, eps_gap, P, V, _ptr(A))
    if rc:
        raise OracleError(f"non-finite state at step {rc - 1}")
    return (P, V, A) if want_accel else (P, V)


def loss(P, obs, kind="l1", mask=None, sign_override=None):
    """Eq. 4.  Returns (L, dL/dP)."""
    P = _f64(P)
    obs = _f64(obs)
    K1, n = P.shape
    gP = np.empty_like(P)
    m = None if mask is None else np.ascontiguousarray(mask, dtype=np.uint8)
    s = None if sign_override is None else np.ascontiguousarray(sign_override, dtype=np.int8)
    L = lib().ora_loss(0 if kind == "l1" else 1, n, K1 - 1, P, obs, _ptr(m), _ptr(s), gP)
    return L, gP


def backward(leader, length, params, P, V, gP, dt=0.1, a_min=-10.0, eps_gap=0.1):
    """Reverse-mode adjoint.  Returns dict(g_params [6, n_par], g_abs, g_p0, g_v0, g_p0_abs,
    g_v0_abs); the *_abs arrays are the condition scales (sum of |terms|) of the gradients."""
    leader = np.ascontiguousarray(leader, dtype=np.int32)
    n = leader.shape[0]
    prm = _params2d(params, n)
    K = P.shape[0] - 1
    g = np.empty_like(prm)
    ga = np.empty_like(prm)
    gp0 = np.empty(n)
    gv0 = np.empty(n)
    gp0a = np.empty(n)
    gv0a = np.empty(n)
    rc = lib().ora_backward(n, leader, _f64(length), prm, prm.shape[1], K, dt, a_min, eps_gap,
                            _f64(P), _f64(V), _f64(gP), g, _ptr(ga), _ptr(gp0), _ptr(gv0),
                            _ptr(gp0a), _ptr(gv0a))
    if rc:
        raise OracleError(f"non-finite adjoint at step {rc - 1}")
    return {"g_params": g, "g_abs": ga, "g_p0": gp0, "g_v0": gv0, "g_p0_abs": gp0a,
            "g_v0_abs": gv0a}


def rollout_tangent(leader, length, p0, v0, params, K, tp0=None, tv0=None, tparams=None,
                    dt=0.1, a_min=-10.0, eps_gap=0.1):
    """Forward-mode (dual number) rollout.  Returns P, dP [(K+1), n]."""
    leader = np.ascontiguousarray(leader, dtype=np.int32)
    n = leader.shape[0]
    prm = _params2d(params, n)
    tp0 = None if tp0 is None else _f64(tp0)
    tv0 = None if tv0 is None else _f64(tv0)
    tpr = None if tparams is None else np.ascontiguousarray(
        _f64(tparams).reshape(prm.shape))
    P = np.empty((K + 1, n))
    dP = np.empty((K + 1, n))
    rc = lib().ora_rollout_tangent(n, leader, _f64(length), _f64(p0), _f64(v0), prm,
                                   prm.shape[1], K, dt, a_min, eps_gap, _ptr(tp0), _ptr(tv0),
                                   _ptr(tpr), P, dP)
    if rc:
        raise OracleError(f"non-finite tangent at step {rc - 1}")
    return P, dP


# ---------------------------------------------------------- virtual-leader mode
def rollout_vl(p0, v0, params, dp, dv, dt=0.1, a_min=-10.0, eps_gap=0.1):
    """Virtual-leader rollout: dp, dv [K, n] free leader terms.  Returns P, V."""
    dp = _f64(dp)
    K, n = dp.shape
    prm = _params2d(params, n)
    P = np.empty((K + 1, n))
    V = np.empty((K + 1, n))
    rc = lib().ora_rollout_vl(n, _f64(p0), _f64(v0), prm, prm.shape[1], K, dt, a_min, eps_gap,
                              dp, _f64(dv), P, V)
    if rc:
        raise OracleError(f"non-finite state at step {rc - 1}")
    return P, V


def backward_vl(params, dp, dv, P, V, gP, dt=0.1, a_min=-10.0, eps_gap=0.1):
    """Adjoint of rollout_vl.  Returns dict(g_params, g_abs, g_dp, g_dv, g_p0, g_v0)."""
    dp = _f64(dp)
    K, n = dp.shape
    prm = _params2d(params, n)
    g = np.empty_like(prm)
    ga = np.empty_like(prm)
    gdp = np.empty((K, n))
    gdv = np.empty((K, n))
    gp0 = np.empty(n)
    gv0 = np.empty(n)
    gp0a = np.empty(n)
    gv0a = np.empty(n)
    rc = lib().ora_backward_vl(n, prm, prm.shape[1], K, dt, a_min, eps_gap, dp, _f64(dv),
                               _f64(P), _f64(V), _f64(gP), g, _ptr(ga), gdp, gdv, _ptr(gp0),
                               _ptr(gv0), _ptr(gp0a), _ptr(gv0a))
    if rc:
        raise OracleError("non-finite adjoint")
    return {"g_params": g, "g_abs": ga, "g_dp": gdp, "g_dv": gdv, "g_p0": gp0, "g_v0": gv0,
            "g_p0_abs": gp0a, "g_v0_abs": gv0a}


def rollout_vl_tangent(p0, v0, params, dp, dv, tp0=None, tv0=None, tparams=None, tdp=None,
                       tdv=None, dt=0.1, a_min=-10.0, eps_gap=0.1):
    dp = _f64(dp)
    K, n = dp.shape
    prm = _params2d(params, n)
    arr = [None if x is None else _f64(x) for x in (tp0, tv0)]
    tpr = None if tparams is None else np.ascontiguousarray(_f64(tparams).reshape(prm.shape))
    tdp_ = None if tdp is None else _f64(tdp)
    tdv_ = None if tdv is None else _f64(tdv)
    P = np.empty((K + 1, n))
    dP = np.empty((K + 1, n))
    rc = lib().ora_rollout_vl_tangent(n, _f64(p0), _f64(v0), prm, prm.shape[1], K, dt, a_min,
                                      eps_gap, dp, _f64(dv), _ptr(arr[0]), _ptr(arr[1]),
                                      _ptr(tpr), _ptr(tdp_), _ptr(tdv_), P, dP)
    if rc:
        raise OracleError("non-finite tangent")
    return P, dP


def lr(it, total=500, lr0=0.1, lr1=0.01) -> float:
    return lib().ora_lr(it, total, lr0, lr1)


def adam_step(x, g, m1, m2, t, lr_, beta1=0.9, beta2=0.999, eps=1e-8, mask=None):
    """In-place Adam step on float64 arrays (t is 1-based)."""
    for a in (x, m1, m2):
        assert a.dtype == np.float64 and a.flags.c_contiguous
    mk = None if mask is None else np.ascontiguousarray(mask, dtype=np.uint8)
    lib().ora_adam_step(x.size, x, _f64(g), m1, m2, t, lr_, beta1, beta2, eps, _ptr(mk))


def project(params):
    """In-place box clamp of SoA [6, n_par] float64 params."""
    assert params.dtype == np.float64 and params.flags.c_contiguous
    lib().ora_project(params.shape[1] if params.ndim == 2 else 1, params)


def param_mask(opt_mask: int, n_par: int) -> np.ndarray:
    """Element mask [6, n_par] from the 6-bit parameter mask (bit k = parameter k optimized)."""
    m = np.zeros((NPAR, n_par), dtype=np.uint8)
    for k in range(NPAR):
        if opt_mask >> k & 1:
            m[k, :] = 1
    return m


def fit_iteration(state, obs, it, total=500, lr0=0.1, lr1=0.01, kind="l1", mask=None,
                  opt_mask=0b011111, dt=0.1, a_min=-10.0, eps_gap=0.1, sign_override=None):
    """One optimizer iteration of the paper's fitting loop:
    rollout -> Eq. 4 loss -> adjoint -> Adam (lr schedule) -> box clamp.  `state` is a dict
    with leader, length, p0, v0, params [6, n_par] f64, m1, m2 (mutated).  Returns (L, grads)."""
    P, V = rollout(state["leader"], state["length"], state["p0"], state["v0"], state["params"],
                   obs.shape[0] - 1, dt, a_min, eps_gap)
    L, gP = loss(P, obs, kind, mask, sign_override)
    g = backward(state["leader"], state["length"], state["params"], P, V, gP, dt, a_min, eps_gap)
    pm = param_mask(opt_mask, state["params"].shape[1])
    adam_step(state["params"], g["g_params"], state["m1"], state["m2"], it + 1,
              lr(it, total, lr0, lr1), mask=pm)
    project(state["params"])
    return L, g
