"""Trajectory filtering / reconstruction bookkeeping around the hot path (host side).

* `dense_observations`: the paper's nearest-step alignment ("for each time stamp
  T_j ... we can find the nearest time step k_j * dt") of timestamped 1-D observations into the
  step-major [(K+1), N] array the kernels read, NaN = not observed (sparse reconstruction,
  PAPER.md:259: >= 1 s sampling; dt = 1.0 s there).
* `table1_metrics`: the paper's evaluation criteria computed on the device
  from the recorded trajectory and speeds (evaluation, not part of the hot path).
"""
from __future__ import annotations

import numpy as np
import torch


def nearest_steps(T, dt: float) -> np.ndarray:
    """k_j = round(T_j / dt), ties half up; a 1e-9 relative guard makes
    decimal ties such as 0.35 / 0.1 round up despite binary representation."""
    q = np.asarray(T, dtype=np.float64) / dt
    return np.floor(q + 0.5 + 1e-9 * np.maximum(1.0, np.abs(q))).astype(np.int64)


def dense_observations(vehicle, T, P, n: int, K: int, dt: float) -> np.ndarray:
    """Scatter observations (vehicle index, timestamp, position) to a float32 [(K+1), n] array
    with NaN where nothing is observed.  Raises if two observations of a vehicle fall on the
    same step (Eq. 4 would need both terms) or a timestamp lies outside [0, K dt]."""
    vehicle = np.asarray(vehicle, dtype=np.int64)
    k = nearest_steps(T, dt)
    if np.any(k < 0) or np.any(k > K):
        raise ValueError("observation timestamp outside the simulated horizon")
    if np.any(vehicle < 0) or np.any(vehicle >= n):
        raise ValueError("observation vehicle index out of range")
    flat = k * n + vehicle
    if np.unique(flat).size != flat.size:
        raise ValueError("two observations of one vehicle map to the same step; use dt smaller "
                         "than the sampling interval")
    obs = np.full((K + 1) * n, np.nan, dtype=np.float32)
    obs[flat] = np.asarray(P, dtype=np.float32)
    return obs.reshape(K + 1, n)


IMP_THRESHOLD = 10.0  # PAPER.md:291 "absolute acceleration exceeds 10"
IMP_ATOL = 1e-4       # fp32 rounding of the recorded speeds: (v' - v)/dt of a step at exactly
                      # |a*| = 10 reads up to ~1e-6 m/s^2 beyond it


@torch.no_grad()
def table1_metrics(traj: torch.Tensor, vel_traj: torch.Tensor, obs: torch.Tensor, dt: float,
                   steps: int | None = None) -> dict:
    """Pos. (%), Acc. (mean/std of |a|, m/s^2) and Imp. (fraction of trajectories with any
    |a| > 10, with an IMP_ATOL allowance for fp32 state rounding) of fitted trajectories
    (PAPER.md:287-292).  traj, vel_traj, obs: [(K+1), N] on the device; accelerations are the
    Euler increments (v(t+dt) - v(t)) / dt of Eq. 3; `acc_max` is reported too."""
    K = traj.shape[0] - 1 if steps is None else steps
    P = traj[:K + 1].double()
    V = vel_traj[:K + 1].double()
    O = obs[:K + 1].double()
    seen = torch.isfinite(O)
    length = (P[-1] - P[0]).clamp_min(1e-300)
    ratio = torch.where(seen, (O - P).abs() / length, torch.zeros_like(P))
    pos = 100.0 * ratio.sum() / seen.sum().clamp_min(1)
    acc = (V[1:] - V[:-1]).abs() / dt
    return {"pos_pct": float(pos), "acc_mean": float(acc.mean()),
            "acc_std": float(acc.std(unbiased=False)),
            "acc_max": float(acc.max()),
            "imp_frac": float((acc > IMP_THRESHOLD + IMP_ATOL).any(dim=0).double().mean())}
