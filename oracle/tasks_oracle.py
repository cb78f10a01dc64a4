"""Plain reference of the trajectory-reconstruction bookkeeping and the Table-I metrics.

TEST INFRASTRUCTURE ONLY (see oracle/oracle.py).  Pure Python/numpy, written from the paper:
  * nearest time step k_j of each timestamp T_j (round half up);
  * Eq. 4 over observation lists, L = sum_j |P_j - P[k_j]|;
  * the fit's initial state from the first two data points (R#13);
  * Table I criteria: Pos. = mean over data points of |P_j - P[k_j]| divided
    by the total trajectory length (spatial P_last - P_first), Acc. = mean / std
    of |a| over all steps, Imp. = fraction of trajectories with any |a| > 10 (strict).
"""
from __future__ import annotations

import math
from decimal import ROUND_HALF_UP, Decimal


def nearest_step(T: float, dt: float) -> int:
    """k = round(T / dt), exact half-up decided in decimal (0.35 / 0.1 -> 4)."""
    q = Decimal(repr(T)) / Decimal(repr(dt))
    return int(q.quantize(Decimal(1), rounding=ROUND_HALF_UP))


def loss_sparse(P, obs):
    """Eq. 4 over a list of observations (vehicle i, time T_j, position P_j): returns
    (L, dL/dP as a dict {(k, i): -sign}) with the nearest-step alignment above; dt given per
    call through `obs` entries (i, T, Pj, dt)."""
    L = 0.0
    grad = {}
    for i, T, Pj, dt in obs:
        k = nearest_step(T, dt)
        r = float(Pj) - float(P[k][i])
        L += abs(r)
        grad[(k, i)] = grad.get((k, i), 0.0) - ((r > 0) - (r < 0))
    return L, grad


def positional_error_rate(P, obs_by_vehicle, dt):
    """per data point |P_j - P[k_j]| / trajectory length, averaged (in %)."""
    terms = []
    for i, pts in obs_by_vehicle.items():
        length = P[-1][i] - P[0][i]
        if length <= 0:
            raise ValueError("zero-length trajectory")
        for T, Pj in pts:
            terms.append(abs(Pj - P[nearest_step(T, dt)][i]) / length)
    return 100.0 * sum(terms) / len(terms)


def acceleration_stats(acc):
    """Population mean and std of |a| (Table I caption)."""
    a = [abs(x) for x in acc]
    m = sum(a) / len(a)
    return m, math.sqrt(sum((x - m) ** 2 for x in a) / len(a))


def implausible(acc) -> bool:
    """any |a| exceeding 10 (strict)."""
    return any(abs(x) > 10.0 for x in acc)


def state_from_obs(obs, dt):
    """"the initial position p(0) and speed v(0) for each trajectory were set to
    0 and (Delta P) / Delta t, where Delta P is the distance between the first two data
    points".  obs: rows t = 0..K of per-vehicle positions (NaN = not observed).  With lanes the
    position is the vehicle's own (R#13): p0 = the first data point carried back to step 0 at
    speed v0 (itself when observed at step 0); v0 clamped at 0 (no backward motion).
    One data point: v0 = 0; none: (0, 0).  Returns lists (p0, v0)."""
    n = len(obs[0])
    p0, v0 = [], []
    for i in range(n):
        pts = [(t, float(row[i])) for t, row in enumerate(obs) if math.isfinite(float(row[i]))]
        if not pts:
            p0.append(0.0)
            v0.append(0.0)
            continue
        (t1, P1) = pts[0]
        v = 0.0
        if len(pts) > 1:
            (t2, P2) = pts[1]
            v = max(0.0, (P2 - P1) / ((t2 - t1) * dt))
        p0.append(P1 - t1 * dt * v)
        v0.append(v)
    return p0, v0
