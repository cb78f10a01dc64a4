"""Seeded synthetic workload generator shared by the CUDA path's tests/bench and the oracle.

This module holds NONE of the method's arithmetic (no IDM, no Euler step, no loss): it only
draws random numbers with the shapes and value ranges of the paper's workloads and rounds
them to fp32 once, so both sides consume identical inputs.  Recipe: DESIGN.md "Input recipe".

Layout conventions:
  * vehicles are lane-sorted: lane l owns [lane_offsets[l], lane_offsets[l+1]), ascending
    position; the leader h(i) of vehicle i is i+1 inside the lane, none for the
    lane head;
  * params are SoA [6][n_par] in the order (a_max, a_pref, s_min, T_pref, v_targ, delta).
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

PARAM_NAMES = ("a_max", "a_pref", "s_min", "T_pref", "v_targ", "delta")
# initial (a_max, a_pref, T_pref, s_min, v_targ) = (10, 2, 1, 5, 50); delta is
# never given (reading R#1: 4).  Stored in our parameter order.
PAPER_INIT = (10.0, 2.0, 5.0, 1.0, 50.0, 4.0)
A_MIN = -10.0  # PAPER.md:208 "a_min is set to -10"


@dataclass
class Workload:
    name: str
    lane_offsets: np.ndarray  # int32 [L+1]
    length: np.ndarray        # f32 [N] body lengths
    p0: np.ndarray            # f32 [N] initial positions (lane-local, m)
    v0: np.ndarray            # f32 [N] initial speeds (m/s)
    theta_true: np.ndarray    # f32 [6, N] "true" driver parameters (for truth rollouts)
    K: int                    # simulated steps
    dt: float = 0.1
    seed: int = 0
    meta: dict = field(default_factory=dict)

    @property
    def n(self) -> int:
        return int(self.lane_offsets[-1])

    @property
    def n_lanes(self) -> int:
        return int(self.lane_offsets.shape[0] - 1)


# BASELINE.json configs (names C1..C5 as in SURVEY.md section 8(d)).
CONFIGS = {
    "C1": dict(lanes=1, per_lane=10, K=100, seed=1),
    "C2": dict(lanes=1000, per_lane=100, K=300, seed=2),
    "C3": dict(lanes=6, per_lane=333, K=27000, seed=3),
    "C4": dict(lanes=20000, per_lane=100, K=300, seed=4),
    "C5": dict(scenes=100000, K=10, seed=5),
    # not a BASELINE.json config: C4's 2M vehicles in 2,000 lanes of 1,000 (each over a 2-CTA
    # thread-block cluster), to measure the long-lane path against C4's whole-lane tiles
    "C4L": dict(lanes=2000, per_lane=1000, K=300, seed=4),
}


def lane_sizes_for(name: str, rng: np.random.Generator) -> np.ndarray:
    c = CONFIGS[name]
    if "scenes" in c:
        # Waymo-shaped: per scene 4-12 lanes, each with 1 + Binomial(7, 0.2) vehicles.
        lanes_per_scene = rng.integers(4, 13, size=c["scenes"])
        return 1 + rng.binomial(7, 0.2, size=int(lanes_per_scene.sum()))
    return np.full(c["lanes"], c["per_lane"], dtype=np.int64)


def make_workload(name: str = "C1", lane_sizes=None, K: int | None = None, seed: int | None = None,
                  dt: float = 0.1) -> Workload:
    """Draw a lane-sorted platoon workload.

    Per vehicle: theta_true ~ a_max U[5,10], a_pref U[1,3], s_min U[1.5,4], T U[0.8,2],
    v_targ U[25,40], delta = 4 (inside the paper's boxes); length U[4,5.5] m.
    Per lane: cruise speed v_e ~ U[8,25] m/s; v_i(0) = max(0, v_e (1 + 0.05 xi)).
    Gaps (bumper to bumper): g_i = g0_i + v_i(0) h_i with jam distance g0 ~ U[2,5] m and time
    headway h ~ U[1.0,2.0] s (a traffic-count style draw, independent of the IDM).
    Positions: lane tail at 0, p_{i+1} = p_i + g_i + length_{i+1}.
    """
    c = CONFIGS.get(name, {})
    seed = c.get("seed", 0) if seed is None else seed
    K = c.get("K", 100) if K is None else K
    rng = np.random.Generator(np.random.PCG64(seed))
    sizes = np.asarray(lane_sizes if lane_sizes is not None else lane_sizes_for(name, rng),
                       dtype=np.int64)
    L = sizes.shape[0]
    off = np.zeros(L + 1, dtype=np.int64)
    np.cumsum(sizes, out=off[1:])
    n = int(off[-1])
    lane_of = np.repeat(np.arange(L), sizes)

    theta = np.empty((6, n))
    theta[0] = rng.uniform(5.0, 10.0, n)
    theta[1] = rng.uniform(1.0, 3.0, n)
    theta[2] = rng.uniform(1.5, 4.0, n)
    theta[3] = rng.uniform(0.8, 2.0, n)
    theta[4] = rng.uniform(25.0, 40.0, n)
    theta[5] = 4.0
    length = rng.uniform(4.0, 5.5, n)
    v_e = rng.uniform(8.0, 25.0, L)
    v0 = np.maximum(0.0, v_e[lane_of] * (1.0 + 0.05 * rng.standard_normal(n)))
    gap = rng.uniform(2.0, 5.0, n) + v0 * rng.uniform(1.0, 2.0, n)
    # p_{i+1} = p_i + gap_i + len_{i+1}; lane tail (first vehicle of the lane) at 0.
    step = np.zeros(n)
    step[1:] = gap[:-1] + length[1:]
    starts = off[:-1][sizes > 0]
    step[starts] = 0.0
    csum = np.cumsum(step)
    p0 = csum - np.repeat(csum[starts], sizes[sizes > 0])

    return Workload(name=name, lane_offsets=off.astype(np.int32),
                    length=length.astype(np.float32), p0=p0.astype(np.float32),
                    v0=v0.astype(np.float32), theta_true=theta.astype(np.float32), K=K, dt=dt,
                    seed=seed)


def init_params(n_par: int) -> np.ndarray:
    """The paper's initial parameter values as f32 SoA [6, n_par]."""
    return np.repeat(np.asarray(PAPER_INIT, dtype=np.float32)[:, None], n_par, axis=1).copy()


def add_noise(P_true: np.ndarray, sigma: float, seed: int) -> np.ndarray:
    """Observation noise N(0, sigma^2) (sigma = 0.3 m), rounded to f32; row 0
    (the initial positions) is left exact."""
    rng = np.random.Generator(np.random.PCG64(seed + 7919))
    obs = np.asarray(P_true, dtype=np.float64).copy()
    obs[1:] += sigma * rng.standard_normal(obs[1:].shape)
    return obs.astype(np.float32)


def kinematic_obs(w: Workload, sigma: float = 0.3, seed: int | None = None) -> np.ndarray:
    """Synthetic 'measured' trajectories that do not come from any simulator: each vehicle
    moves with its initial speed plus a small constant acceleration U[-0.3, 0.3] m/s^2
    (speed floored at 0), plus N(0, sigma^2) noise.  f32 [(K+1), N]."""
    seed = w.seed if seed is None else seed
    rng = np.random.Generator(np.random.PCG64(seed + 104729))
    acc = rng.uniform(-0.3, 0.3, w.n)
    t = (np.arange(w.K + 1) * w.dt)[:, None]
    v0 = w.v0.astype(np.float64)[None, :]
    # time at which the speed would hit 0 (only for decelerating vehicles)
    t_stop = np.where(acc < 0, -v0 / np.minimum(acc, -1e-12), np.inf)
    te = np.minimum(t, t_stop)
    disp = v0 * te + 0.5 * acc[None, :] * te * te
    obs = w.p0.astype(np.float64)[None, :] + disp
    obs[1:] += sigma * rng.standard_normal(obs[1:].shape)
    return obs.astype(np.float32)


def lane_subset(w: Workload, lanes) -> Workload:
    """The workload restricted to the given lane indices (lanes are independent units)."""
    lanes = np.asarray(lanes, dtype=np.int64)
    off = w.lane_offsets.astype(np.int64)
    idx = np.concatenate([np.arange(off[l], off[l + 1]) for l in lanes]) if len(lanes) else \
        np.zeros(0, dtype=np.int64)
    sizes = off[lanes + 1] - off[lanes]
    new_off = np.zeros(len(lanes) + 1, dtype=np.int64)
    np.cumsum(sizes, out=new_off[1:])
    return Workload(name=f"{w.name}[subset]", lane_offsets=new_off.astype(np.int32),
                    length=w.length[idx].copy(), p0=w.p0[idx].copy(), v0=w.v0[idx].copy(),
                    theta_true=w.theta_true[:, idx].copy(), K=w.K, dt=w.dt, seed=w.seed,
                    meta={"vehicle_index": idx, "lanes": lanes})
