"""Plain reference of the trajectory-reconstruction bookkeeping and the Table-I metrics.

TEST INFRASTRUCTURE ONLY (see oracle/oracle.py).  Pure Python/numpy, written from the paper:
  * nearest time step k_j of each timestamp T_j (round half up);
  * Eq. 4 over observation lists, L = sum_j |P_j - P[k_j]|;
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
