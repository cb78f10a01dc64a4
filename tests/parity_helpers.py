"""Shared helpers for the GPU-vs-oracle parity tests (test infrastructure).

Tolerances (north_star, BASELINE.json):
  * states: |x_gpu - x_ora| <= max(1e-4 |x_ora|, 1e-3)  (m, m/s) at every step
  * gradients: |g_gpu - g_ora| <= 1e-3 |g_ora| + 1e-3 G_abs, G_abs = sum_t |q da/dtheta|
    (condition-aware 1e-3 relative; plain 1e-3 relative pass rate is reported too); the state
    gradients dL/dp0, dL/dv0 likewise, with G_abs = the oracle's sum of |terms| added into
    the state adjoint (g_p0_abs, g_v0_abs)
  * L1 kinks: the oracle backward is fed the GPU's sign pattern (sign(0) = 0); every sign
    mismatch must have |residual| < 1e-3 m.
"""
from __future__ import annotations

import numpy as np

STATE_REL, STATE_ABS = 1e-4, 1e-3
GRAD_REL = 1e-3


def state_violation(gpu, ora):
    """max over elements of |gpu - ora| / max(1e-4 |ora|, 1e-3) (<= 1 passes)."""
    tol = np.maximum(STATE_REL * np.abs(ora), STATE_ABS)
    return float(np.max(np.abs(np.asarray(gpu, np.float64) - ora) / tol))


def grad_check(g_gpu, g_ora, g_abs, rel=GRAD_REL):
    """Returns (max ratio to the condition-aware tolerance, plain-1e-3 pass fraction)."""
    g_gpu = np.asarray(g_gpu, np.float64)
    err = np.abs(g_gpu - g_ora)
    tol = rel * np.abs(g_ora) + rel * g_abs + 1e-30
    plain = err <= rel * np.abs(g_ora) + 1e-12
    return float(np.max(err / tol)), float(np.mean(plain))


def oracle_truth_obs(oracle, w, sigma=0.3, seed=None):
    """Observations = oracle rollout with theta_true + N(0, sigma^2) (rounded to f32)."""
    from paper_2412_16750_b200 import synth
    h = oracle.leader_from_lanes(w.lane_offsets)
    P, _ = oracle.rollout(h, w.length, w.p0, w.v0, w.theta_true, w.K, w.dt)
    return synth.add_noise(P, sigma, w.seed if seed is None else seed)


def state_grad_check(g_state0, g, rel=GRAD_REL, label=""):
    """dL/dp0 and dL/dv0 of the GPU ([2, n]: rows p0, v0) against the oracle's g_p0, g_v0
    with the condition-aware bar (g_p0_abs, g_v0_abs).  Returns the worst ratio to the
    tolerance over both rows and prints the plain-1e-3 pass rates and, for the elements that
    fail the plain bar, the smallest |g| / G_abs (a cancellation: the gradient is a small
    difference of larger terms)."""
    g_state0 = np.asarray(g_state0, np.float64)
    worst = 0.0
    for row, (key, akey) in enumerate((("g_p0", "g_p0_abs"), ("g_v0", "g_v0_abs"))):
        w, plain = grad_check(g_state0[row], g[key], g[akey], rel)
        err = np.abs(g_state0[row] - g[key])
        fail = err > rel * np.abs(g[key]) + 1e-12
        canc = (np.abs(g[key][fail]) / np.maximum(g[akey][fail], 1e-300)).max() if fail.any() \
            else float("nan")
        print(f"{label} {key}: worst/tol = {w:.3f}, plain-1e-3 pass = {plain:.5f}, "
              f"plain failures {int(fail.sum())}, max |g|/G_abs among them = {canc:.3g}")
        worst = max(worst, w)
    return worst


def sign_mismatch_residual(obs, P_ora, gpu_grad_traj):
    """The L1 sign protocol: where the GPU's dL/dP = -sign(obs - P) differs
    from the oracle's own sign on its fp64 trajectory, obs lies between the two trajectories,
    so the oracle's residual there is at most |P_gpu - P_ora| -- which the state parity bounds
    by the position tolerance max(1e-4 |P|, 1e-3 m) (north_star; 1e-3 m up to 10 km, DESIGN.md
    section 7).  Both signs are then correct to the tolerance.  Returns the largest residual /
    tolerance over the mismatches (0 if the patterns agree; <= 1 passes)."""
    r = np.asarray(obs, np.float64) - P_ora
    own = -np.sign(np.where(np.isnan(r), 0.0, r))
    mism = own != np.asarray(gpu_grad_traj, np.float64)
    if not mism.any():
        return 0.0
    tol = np.maximum(STATE_REL * np.abs(P_ora), STATE_ABS)
    return float((np.abs(r) / tol)[mism].max())


def near_kink_vehicles(V, dt=0.1, a_min=-10.0, tol=1e-4):
    """Vehicles whose (oracle) speed comes within `tol` m/s of the a_lb tie v = dt |a_min|
    at some step (R#5: a_lb = max(-v/dt, a_min) switches branch there, so its derivative jumps;
    SURVEY.md 8(c) parity protocol: such vehicles are reported separately, not failed)."""
    V = np.asarray(V, np.float64)
    return np.where((np.abs(V[:-1] - dt * abs(a_min)) < tol).any(axis=0))[0]
