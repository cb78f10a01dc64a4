"""Shared helpers for the GPU-vs-oracle parity tests (test infrastructure).

Tolerances (north_star, BASELINE.json):
  * states: |x_gpu - x_ora| <= max(1e-4 |x_ora|, 1e-3)  (m, m/s) at every step
  * gradients: |g_gpu - g_ora| <= 1e-3 |g_ora| + 1e-3 G_abs, G_abs = sum_t |q da/dtheta|
    (condition-aware 1e-3 relative; plain 1e-3 relative pass rate is reported too)
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
