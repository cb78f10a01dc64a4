"""Pins of the fp64 oracle (oracle/idm_oracle.c) against things other than itself:
worked values (tests/golden, cited), closed forms of the modified IDM's steady states,
invariants the paper states, central finite differences, and an independent dual-number
forward mode.  Each pin is chosen so that a plausible mistake fails it (noted per test).
"""
import math
import os

import numpy as np
import pytest

from paper_2412_16750_b200 import synth

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "spec_worked_examples.txt")
DEFAULT = np.array([10.0, 2.0, 5.0, 1.0, 50.0, 4.0])  # PAPER.md:208 init, delta = 4 (R#1)
DT, A_MIN, EPS = 0.1, -10.0, 0.1


def _golden_rows():
    rows = []
    with open(GOLDEN) as f:
        for line in f:
            if line.startswith("#") or not line.strip():
                continue
            rows.append(line.split())
    return rows


@pytest.mark.parametrize("row", _golden_rows(), ids=lambda r: r[0])
def test_golden_worked_examples(oracle, row):
    kind = row[0]
    nums = []
    for tok in row[1:]:
        try:
            nums.append(float(tok))
        except ValueError:
            break
    if kind == "softplus":
        x, exp, tol = nums
        assert abs(oracle.softplus(x) - exp) <= tol
    elif kind == "optimal_spacing":
        a, b, s0, T, v, dv, exp, tol = nums
        assert abs(oracle.optimal_spacing(a, b, s0, T, v, dv) - exp) <= tol
    elif kind == "accel":
        th = nums[:6]
        v, dp, dv, dt, amin, exp, tol = nums[6:]
        assert abs(oracle.accel(th, v, dp, dv, True, dt, amin) - exp) <= tol
    elif kind == "gather":
        # 2-vehicle lane: follower 0 at p_i, leader 1 at p_h; one rollout step uses the
        # gathered (dp, dv) -- compare the follower's a* to accel() at the expected (dp, dv).
        p_i, p_h, len_h, v_i, v_h, exp_dp, exp_dv, _tol = nums
        P, V, A = oracle.rollout(np.array([1, -1], np.int32), np.array([4.0, len_h]),
                                 np.array([p_i, p_h]), np.array([v_i, v_h]), DEFAULT, 1, DT,
                                 A_MIN, EPS, want_accel=True)
        assert A[0, 0] == oracle.accel(DEFAULT, v_i, exp_dp, exp_dv, True, DT, A_MIN)
        # the sign of dv matters: swapping it gives a different acceleration
        assert A[0, 0] != oracle.accel(DEFAULT, v_i, exp_dp, -exp_dv, True, DT, A_MIN)
    elif kind == "loss_l1":
        if len(nums) == 5:  # obs P -> L g tol
            o, p, expL, expg, _ = nums
            L, g = oracle.loss(np.array([[0.0], [p]]), np.array([[0.0], [o]]), "l1")
            assert L == expL and g[1, 0] == expg and g[0, 0] == 0.0
        else:
            r1, _, r2, _, expL = nums[0], nums[1], nums[2], nums[3], nums[4]
            P = np.zeros((2, 2))
            obs = np.array([[0.0, 0.0], [r1, r2]])
            L, _ = oracle.loss(P, obs, "l1")
            assert L == expL
    elif kind == "lr":
        it, total, lr0, lr1, exp, tol = nums
        assert abs(oracle.lr(int(it), int(total), lr0, lr1) - exp) <= tol
    else:
        raise AssertionError(kind)


# ----------------------------------------------------------------- scalar math
def test_softplus_identities(oracle):
    # softplus(x) - softplus(-x) = x ; softplus >= max(x, 0); sigmoid = d softplus
    for x in np.linspace(-60, 60, 241):
        assert abs(oracle.softplus(x) - oracle.softplus(-x) - x) <= 1e-12 * max(1, abs(x))
        assert oracle.softplus(x) >= max(x, 0.0)
        assert abs(oracle.sigmoid(x) + oracle.sigmoid(-x) - 1.0) <= 1e-15


def test_accel_is_log_sum_exp(oracle):
    """Sec. III-C: a* = a_lb + log(1+exp(a - a_lb)) = log(e^a + e^a_lb).  Pinned with the
    free-road closed form a_f = a_max (1 - (v/v_targ)^delta) (north_star) and numpy's
    logaddexp: a wrong softplus composition or a_lb fails."""
    rng = np.random.default_rng(0)
    for _ in range(500):
        th = np.array([rng.uniform(5, 10), rng.uniform(0.1, 5), rng.uniform(1, 10),
                       rng.uniform(0.1, 5), rng.uniform(20, 60), 4.0])
        v = rng.uniform(0, 45)
        a_f = th[0] * (1 - (v / th[4]) ** 4)
        a_lb = max(-v / DT, A_MIN)
        got = oracle.accel(th, v, math.inf, 0.0, False, DT, A_MIN)
        assert abs(got - np.logaddexp(a_f, a_lb)) <= 1e-12 * max(1, abs(got))
        # and it matches the north_star's free-road a(1 - (v/v0)^delta) within
        # log(1 + e^(a_lb - a_f)) (the softplus slack)
        assert 0 <= got - a_f <= math.log1p(math.exp(a_lb - a_f)) + 1e-12


def test_accel_bounds_and_monotonicity(oracle):
    """a_lb < a* <= log(e^a_max + e^a_lb) (R#4), v + dt a* >= 0,
    braking increases with approach rate dv and with shrinking gap."""
    rng = np.random.default_rng(1)
    for _ in range(2000):
        th = np.array([rng.uniform(5, 10), rng.uniform(0.1, 5), rng.uniform(1, 10),
                       rng.uniform(0.1, 5), rng.uniform(20, 60), 4.0])
        v = rng.uniform(0, 40)
        dp = rng.uniform(0.1, 200)
        dv = rng.uniform(-10, 10)
        a = oracle.accel(th, v, dp, dv, True, DT, A_MIN)
        a_lb = max(-v / DT, A_MIN)
        assert a > a_lb - 1e-12
        assert a <= np.logaddexp(th[0], a_lb) + 1e-12
        assert v + DT * a >= -1e-12
        assert oracle.accel(th, v, dp, dv + 1.0, True, DT, A_MIN) <= a + 1e-12
        assert oracle.accel(th, v, dp * 0.9, dv, True, DT, A_MIN) <= a + 1e-12


def test_classic_idm_limit(oracle):
    """a_min -> -inf with s_opt >> 0 reduces to Treiber's IDM (Treiber 2000, cited at
    PAPER.md:103): a* -> a_raw, within log(1 + e^(a_lb - a_raw)) and the s_opt softplus slack."""
    th = DEFAULT
    for v, dp, dv in [(10, 30, 0), (20, 40, 2), (5, 12, -1), (30, 80, 3)]:
        a_min = -1e4
        dt = 1e-3  # -v/dt << 0 as well
        s_star = th[2] + v * th[3] + v * dv / (2 * math.sqrt(th[0] * th[1]))
        a_textbook = th[0] * (1 - (v / th[4]) ** 4 - (s_star / dp) ** 2)
        got = oracle.accel(th, v, dp, dv, True, dt, a_min)
        # the only other difference is the s_opt softplus slack ds = log(1 + e^-s_opt)
        ds = math.log1p(math.exp(-s_star))
        bound = th[0] * ((s_star + ds) ** 2 - s_star ** 2) / dp ** 2
        assert abs(got - a_textbook) <= bound + 1e-12
        assert bound < 1e-3


def _fd(f, x, h):
    d1 = (f(x + h) - f(x - h)) / (2 * h)
    d2 = (f(x + h / 2) - f(x - h / 2)) / h
    return (4 * d2 - d1) / 3  # Richardson


def test_accel_partials_vs_finite_differences(oracle):
    """Every hand partial of a* against Richardson-extrapolated central FD of
    accel() on 1000 random inputs, 10% leaderless; catches a dropped chain term or sign."""
    rng = np.random.default_rng(2)
    worst = 0.0
    for trial in range(1000):
        th = np.array([rng.uniform(5, 10), rng.uniform(0.1, 5), rng.uniform(1, 10),
                       rng.uniform(0.1, 5), rng.uniform(20, 60), rng.uniform(2, 6)])
        v = rng.uniform(0.5, 40)
        if abs(-v / DT - A_MIN) < 1e-3:
            continue
        hl = trial % 10 != 0
        dp = rng.uniform(2, 150) if hl else math.inf
        dv = rng.uniform(-8, 8) if hl else 0.0
        a, d_v, d_dp, d_dv, d_th = oracle.accel_partials(th, v, dp, dv, hl, False, DT, A_MIN)
        assert a == oracle.accel(th, v, dp, dv, hl, DT, A_MIN)

        def num(g, x):
            return _fd(g, x, 1e-4 * max(1.0, abs(x)))

        checks = [(d_v, num(lambda x: oracle.accel(th, x, dp, dv, hl, DT, A_MIN), v))]
        if hl:
            checks.append((d_dp, num(lambda x: oracle.accel(th, v, x, dv, hl, DT, A_MIN), dp)))
            checks.append((d_dv, num(lambda x: oracle.accel(th, v, dp, x, hl, DT, A_MIN), dv)))
        for k in range(6):
            def fk(x, k=k):
                t2 = th.copy()
                t2[k] = x
                return oracle.accel(t2, v, dp, dv, hl, DT, A_MIN)
            checks.append((d_th[k], num(fk, th[k])))
        for an, nu in checks:
            err = abs(an - nu) / max(1e-3, abs(nu))
            worst = max(worst, err)
    assert worst < 1e-6, worst


def test_partials_clamped_gap_and_zero_speed(oracle):
    """R#7: a clamped gap has zero gap-derivative; R#24: at v = 0 the delta- and
    v_targ-derivatives vanish and d a*/d T_pref = 0."""
    _, _, d_dp, _, _ = oracle.accel_partials(DEFAULT, 10, EPS, 0, True, True, DT, A_MIN)
    assert d_dp == 0.0
    _, _, _, _, d_th = oracle.accel_partials(DEFAULT, 0.0, 20.0, 0.0, True, False, DT, A_MIN)
    assert d_th[3] == 0.0 and d_th[4] == 0.0 and d_th[5] == 0.0


# --------------------------------------------------------- closed-form steady states
def free_road_equilibrium_speed(th, a_min=A_MIN):
    """a* = 0 for a leaderless vehicle <=> a_max(1 - (v/v_targ)^delta) = log(1 - e^a_lb),
    a_lb = a_min (v > -a_min dt):  v_f = v_targ (1 - log(1 - e^a_min)/a_max)^(1/delta)."""
    return th[4] * (1.0 - math.log(-math.expm1(a_min)) / th[0]) ** (1.0 / th[5])


def equilibrium_gap(th, v, a_min=A_MIN):
    """a* = 0 with dv = 0 and a leader: softplus(s_min + v T) / dp = sqrt(1 - (v/v_targ)^delta
    - log(1 - e^a_min)/a_max)."""
    s_star = math.log1p(math.exp(th[2] + v * th[3]))
    return s_star / math.sqrt(1.0 - (v / th[4]) ** th[5] - math.log(-math.expm1(a_min)) / th[0])


def test_equilibrium_gap_values():
    """Closed-form equilibrium spacing of the modified model (SURVEY.md 8(c) values)."""
    for v, exp in [(5, 10.000522735), (10, 15.011980593), (20, 25.326219075),
                   (30, 37.515217658)]:
        assert abs(equilibrium_gap(DEFAULT, v) - exp) < 2e-9
    assert abs(free_road_equilibrium_speed(DEFAULT) - 50.0000567511) < 1e-9


def test_free_road_vehicle_is_steady_at_closed_form_speed(oracle):
    """A lone vehicle at v_f keeps v_f (a* = 0 to rounding) and moves dt v_f per step (Eq. 3):
    pins the free-road branch, the a_lb/softplus composition and the Euler update."""
    th = np.array([7.0, 1.5, 2.0, 1.2, 30.0, 4.0])
    vf = free_road_equilibrium_speed(th)
    P, V = oracle.rollout(np.array([-1], np.int32), np.array([4.5]), np.array([3.0]),
                          np.array([vf]), th, 200, DT, A_MIN, EPS)
    assert np.max(np.abs(V - vf)) < 1e-12
    assert np.max(np.abs(P[:, 0] - (3.0 + DT * vf * np.arange(201)))) < 1e-9


def test_platoon_at_equilibrium_spacing_is_steady(oracle):
    """Platoon of heterogeneous drivers at the closed-form equilibrium gaps behind a lane head
    at its free-road equilibrium speed: every speed and gap stays constant for 300 steps.
    Pins Eq. 1 (v T term + softplus), Eq. 2's interaction term, the gather with the LEADER's
    length and the synchronous update; a wrong length index or exponent breaks it."""
    rng = np.random.default_rng(3)
    n = 12
    th = np.empty((6, n))
    th[0] = rng.uniform(5, 10, n)
    th[1] = rng.uniform(0.5, 3, n)
    th[2] = rng.uniform(1.5, 4, n)
    th[3] = rng.uniform(0.8, 2, n)
    th[4] = rng.uniform(25, 40, n)
    th[5] = 4.0
    length = rng.uniform(4, 5.5, n)
    # head (last index) has no leader; choose its v_targ so that v_f(head) = v_e
    v_e = 18.0
    head = th[:, n - 1].copy()
    head[4] = 1.0
    th[4, n - 1] = v_e / free_road_equilibrium_speed(head)
    assert abs(free_road_equilibrium_speed(th[:, n - 1]) - v_e) < 1e-12
    p = np.zeros(n)
    for i in range(1, n):
        p[i] = p[i - 1] + equilibrium_gap(th[:, i - 1], v_e) + length[i]
    leader = np.append(np.arange(1, n), -1).astype(np.int32)
    P, V = oracle.rollout(leader, length, p, np.full(n, v_e), th, 300, DT, A_MIN, EPS)
    assert np.max(np.abs(V - v_e)) < 1e-10
    gaps = P[:, 1:] - P[:, :-1] - length[None, 1:]
    assert np.max(np.abs(gaps - gaps[0])) < 1e-8
    # Perturbing the length convention (own length instead of leader's) breaks steadiness
    p_bad = np.zeros(n)
    for i in range(1, n):
        p_bad[i] = p_bad[i - 1] + equilibrium_gap(th[:, i - 1], v_e) + length[i - 1]
    _, Vb = oracle.rollout(leader, length, p_bad, np.full(n, v_e), th, 50, DT, A_MIN, EPS)
    assert np.max(np.abs(Vb - v_e)) > 1e-4


def test_explicit_euler_uses_old_speed(oracle):
    """Eq. 3 (R#6): p(t+dt) = p + dt v(t) -- a vehicle starting at rest does not move in the
    first step although it accelerates; SPEC.md:154 p=0, v=10, a=0 -> (1.0, 10.0)."""
    P, V, A = oracle.rollout(np.array([-1], np.int32), np.array([4.0]), np.array([0.0]),
                             np.array([0.0]), DEFAULT, 1, DT, A_MIN, EPS, want_accel=True)
    assert P[1, 0] == 0.0 and V[1, 0] == DT * A[0, 0] and A[0, 0] > 0
    th = DEFAULT.copy()
    th[4] = 10.0 / free_road_equilibrium_speed(np.r_[th[:4], 1.0, th[5]])
    P, V = oracle.rollout(np.array([-1], np.int32), np.array([4.0]), np.array([0.0]),
                          np.array([10.0]), th, 1, DT, A_MIN, EPS)
    assert abs(P[1, 0] - 1.0) < 1e-15 and abs(V[1, 0] - 10.0) < 1e-12


# ---------------------------------------------------------------------- invariants
def _c1_like(seed=11, sizes=(10,), K=100):
    return synth.make_workload("C1", lane_sizes=list(sizes), K=K, seed=seed)


def test_no_backward_motion_under_hard_braking(oracle):
    """speeds never go negative, positions never decrease, even when a
    follower runs into a stopped queue (a_raw << a_min)."""
    n = 6
    p = np.array([0.0, 30.0, 40.0, 50.0, 60.0, 70.0])
    v = np.array([25.0, 0.0, 0.0, 0.0, 0.0, 0.0])
    th = np.repeat(DEFAULT[:, None], n, axis=1)
    th[4, 1:] = 20.0
    leader = np.append(np.arange(1, n), -1).astype(np.int32)
    P, V = oracle.rollout(leader, np.full(n, 4.5), p, v, th, 400, DT, A_MIN, EPS)
    assert V.min() >= -1e-12
    assert np.all(np.diff(P, axis=0) >= -1e-12)
    assert V[:, 0].min() < 1.0  # it really braked to (near) standstill


def test_invariants_on_generated_workload(oracle):
    """v >= 0, non-decreasing positions, lane order / positive gaps preserved and
    |a*| <= 10 (+softplus slack) when a_max <= 10 (Imp. = 0)."""
    w = synth.make_workload("C2", lane_sizes=[100] * 30, K=300, seed=5)
    h = oracle.leader_from_lanes(w.lane_offsets)
    P, V, A = oracle.rollout(h, w.length, w.p0, w.v0, w.theta_true, w.K, want_accel=True)
    m = h >= 0
    gaps = P[:, h[m]] - P[:, m] - w.length[h[m]].astype(np.float64)
    assert gaps.min() > EPS
    assert V.min() >= 0
    assert np.all(np.diff(P, axis=0) >= 0)
    assert np.abs(A).max() <= 10.0 + 1e-6


def test_permutation_equivariance_and_lane_independence(oracle):
    """permuting vehicle indices (leader indices remapped) permutes the outputs
    bit-identically; a lane simulated alone equals the same lane inside a batch."""
    w = synth.make_workload("C2", lane_sizes=[7, 1, 12, 5], K=60, seed=9)
    h = oracle.leader_from_lanes(w.lane_offsets)
    P, V = oracle.rollout(h, w.length, w.p0, w.v0, w.theta_true, w.K)
    rng = np.random.default_rng(0)
    perm = rng.permutation(w.n)            # new index j holds old vehicle perm[j]
    inv = np.argsort(perm)
    h2 = np.where(h[perm] >= 0, inv[np.maximum(h[perm], 0)], -1).astype(np.int32)
    P2, V2 = oracle.rollout(h2, w.length[perm], w.p0[perm], w.v0[perm],
                            w.theta_true[:, perm], w.K)
    assert np.array_equal(P2, P[:, perm]) and np.array_equal(V2, V[:, perm])
    sub = synth.lane_subset(w, [2])
    Ps, Vs = oracle.rollout(oracle.leader_from_lanes(sub.lane_offsets), sub.length, sub.p0,
                            sub.v0, sub.theta_true, w.K)
    idx = sub.meta["vehicle_index"]
    assert np.array_equal(Ps, P[:, idx]) and np.array_equal(Vs, V[:, idx])


# ------------------------------------------------------------------------ gradients
def _grad_dot(g, tp0, tv0, tth):
    return float(np.sum(g["g_p0"] * tp0) + np.sum(g["g_v0"] * tv0) +
                 np.sum(g["g_params"] * tth))


@pytest.mark.parametrize("kind", ["l2", "l1"])
def test_adjoint_matches_dual_number_forward_mode(oracle, kind):
    """The hand adjoint (reverse mode) against forward-mode dual numbers: for random
    directions d, <grad L, d> = sum dL/dP . dP/d(eps) exactly (to rounding).  Independent
    derivations; a dropped leader term, wrong sign or transposed index fails."""
    w = synth.make_workload("C1", lane_sizes=[6, 1, 4], K=80, seed=21)
    h = oracle.leader_from_lanes(w.lane_offsets)
    th = w.theta_true.astype(np.float64)
    th[5] = np.random.default_rng(0).uniform(3, 5, w.n)  # general delta
    P, V = oracle.rollout(h, w.length, w.p0, w.v0, th, w.K)
    obs = synth.add_noise(P, 0.3, 3)
    L, gP = oracle.loss(P, obs, kind)
    g = oracle.backward(h, w.length, th, P, V, gP)
    rng = np.random.default_rng(4)
    for _ in range(6):
        tp0 = rng.standard_normal(w.n)
        tv0 = rng.standard_normal(w.n)
        tth = rng.standard_normal(th.shape)
        _, dP = oracle.rollout_tangent(h, w.length, w.p0, w.v0, th, w.K, tp0, tv0, tth)
        fwd = float(np.sum(gP * dP))
        rev = _grad_dot(g, tp0, tv0, tth)
        assert abs(fwd - rev) <= 1e-10 * max(1.0, abs(fwd)), (fwd, rev)


def test_adjoint_matches_central_fd_whole_rollout(oracle):
    """whole-rollout FD on all parameters and the initial state (L2 loss,
    4 vehicles x 40 steps): within 1e-6 relative of Richardson central differences."""
    w = synth.make_workload("C1", lane_sizes=[4], K=40, seed=5)
    h = oracle.leader_from_lanes(w.lane_offsets)
    th = w.theta_true.astype(np.float64)
    P, V = oracle.rollout(h, w.length, w.p0, w.v0, th, w.K)
    obs = synth.add_noise(P, 0.3, 1).astype(np.float64) + 0.5

    def Lof(p0, v0, t):
        P_, _ = oracle.rollout(h, w.length, p0, v0, t, w.K)
        return oracle.loss(P_, obs, "l2")[0]

    _, gP = oracle.loss(P, obs, "l2")
    g = oracle.backward(h, w.length, th, P, V, gP)
    p0 = w.p0.astype(np.float64)
    v0 = w.v0.astype(np.float64)
    for i in range(w.n):
        for name, base, grad in (("p0", p0, g["g_p0"]), ("v0", v0, g["g_v0"])):
            def f(x, i=i, name=name):
                a = (p0 if name == "p0" else v0).copy()
                a[i] = x
                return Lof(a, v0, th) if name == "p0" else Lof(p0, a, th)
            num = _fd(f, base[i], 1e-4)
            assert abs(grad[i] - num) <= 1e-6 * max(1.0, abs(num)), (name, i, grad[i], num)
        for k in range(6):
            def f(x, i=i, k=k):
                t2 = th.copy()
                t2[k, i] = x
                return Lof(p0, v0, t2)
            num = _fd(f, th[k, i], 1e-4 * abs(th[k, i]))
            assert abs(g["g_params"][k, i] - num) <= 1e-6 * max(1.0, abs(num)), (k, i)


def test_adjoint_linearity_and_k1(oracle):
    """zero upstream gradient => all gradients exactly zero; K = 1 with
    L = p_1: dL/dv0 = dt, dL/dp0 = 1."""
    w = synth.make_workload("C1", lane_sizes=[5], K=30, seed=2)
    h = oracle.leader_from_lanes(w.lane_offsets)
    P, V = oracle.rollout(h, w.length, w.p0, w.v0, w.theta_true, w.K)
    g = oracle.backward(h, w.length, w.theta_true, P, V, np.zeros_like(P))
    assert not np.any(g["g_params"]) and not np.any(g["g_p0"]) and not np.any(g["g_v0"])
    P, V = oracle.rollout(np.array([-1], np.int32), np.array([4.0]), np.array([0.0]),
                          np.array([10.0]), DEFAULT, 1)
    gP = np.array([[0.0], [1.0]])
    g = oracle.backward(np.array([-1], np.int32), np.array([4.0]), DEFAULT, P, V, gP)
    assert g["g_v0"][0] == DT and g["g_p0"][0] == 1.0


def test_state_gradient_condition_scales(oracle):
    """The condition scales of dL/dp0, dL/dv0 (sum of |terms| added into the state adjoint, the
    analogue of g_abs; SURVEY.md 8(c) parity protocol): closed forms at K = 1 and K = 2, the
    exact cancellation of a lone vehicle's L = P_2 - P_1 (dL/dp0 = 0 at scale 2), the triangle
    inequality |g| <= scale on coupled lanes (lane and virtual-leader adjoints), and linearity
    in the upstream gradient."""
    lone, ln = np.array([-1], np.int32), np.array([4.0])
    P, V = oracle.rollout(lone, ln, np.array([0.0]), np.array([10.0]), DEFAULT, 1)
    g = oracle.backward(lone, ln, DEFAULT, P, V, np.array([[0.0], [1.0]]))
    assert g["g_p0_abs"][0] == 1.0 and g["g_v0_abs"][0] == DT
    # L = P_2 - P_1 = dt v_1: p0 cancels exactly; its scale counts both observations
    P, V = oracle.rollout(lone, ln, np.array([0.0]), np.array([10.0]), DEFAULT, 2)
    g = oracle.backward(lone, ln, DEFAULT, P, V, np.array([[0.0], [-1.0], [1.0]]))
    assert g["g_p0"][0] == 0.0 and g["g_p0_abs"][0] == 2.0
    assert g["g_v0_abs"][0] >= abs(g["g_v0"][0]) > 0.0
    w = synth.make_workload("C1", lane_sizes=[7, 1, 5], K=60, seed=9)
    h = oracle.leader_from_lanes(w.lane_offsets)
    P, V = oracle.rollout(h, w.length, w.p0, w.v0, w.theta_true, w.K)
    for kind in ("l1", "l2"):
        _, gP = oracle.loss(P, synth.add_noise(P, 0.3, 4), kind)
        g = oracle.backward(h, w.length, w.theta_true, P, V, gP)
        for a, b in (("g_p0", "g_p0_abs"), ("g_v0", "g_v0_abs")):
            assert np.all(np.abs(g[a]) <= g[b] * (1 + 1e-12))
        g3 = oracle.backward(h, w.length, w.theta_true, P, V, -3.0 * gP)
        assert np.allclose(g3["g_p0_abs"], 3 * g["g_p0_abs"], rtol=1e-12)
        assert np.allclose(g3["g_v0_abs"], 3 * g["g_v0_abs"], rtol=1e-12)
    dp = np.random.default_rng(2).uniform(5, 40, (w.K, w.n))
    dv = np.random.default_rng(3).uniform(-2, 2, (w.K, w.n))
    Pv, Vv = oracle.rollout_vl(w.p0, w.v0, w.theta_true, dp, dv)
    _, gP = oracle.loss(Pv, synth.add_noise(Pv, 0.3, 5), "l1")
    g = oracle.backward_vl(w.theta_true, dp, dv, Pv, Vv, gP)
    for a, b in (("g_p0", "g_p0_abs"), ("g_v0", "g_v0_abs")):
        assert np.all(np.abs(g[a]) <= g[b] * (1 + 1e-12))


def test_shared_parameter_gradient_is_sum_of_per_vehicle(oracle):
    """Shared mode (north_star): with identical per-vehicle parameters, the shared gradient
    equals the sum of the per-vehicle gradients."""
    w = synth.make_workload("C1", lane_sizes=[6, 3], K=50, seed=8)
    h = oracle.leader_from_lanes(w.lane_offsets)
    shared = np.array([8.0, 1.7, 3.0, 1.4, 33.0, 4.0])
    per = np.repeat(shared[:, None], w.n, axis=1)
    P, V = oracle.rollout(h, w.length, w.p0, w.v0, per, w.K)
    Ps, Vs = oracle.rollout(h, w.length, w.p0, w.v0, shared, w.K)
    assert np.array_equal(P, Ps)
    obs = synth.add_noise(P, 0.3, 2)
    _, gP = oracle.loss(P, obs, "l1")
    g1 = oracle.backward(h, w.length, per, P, V, gP)
    g2 = oracle.backward(h, w.length, shared, Ps, Vs, gP)
    assert np.allclose(g1["g_params"].sum(axis=1), g2["g_params"][:, 0], rtol=1e-12, atol=1e-12)


# --------------------------------------------------------------------- optimizer
def test_adam_matches_torch_adam_and_linear_lr(oracle):
    """Adam (Kingma & Ba) reduces to torch.optim.Adam (fp64, defaults) with a
    LinearLR 0.1 -> 0.01 schedule over 500 iterations; clamp per PAPER.md:208."""
    torch = pytest.importorskip("torch")
    rng = np.random.default_rng(0)
    x0 = rng.standard_normal(40)
    xt = torch.tensor(x0.copy(), dtype=torch.float64, requires_grad=True)
    opt = torch.optim.Adam([xt], lr=0.1)
    sched = torch.optim.lr_scheduler.LinearLR(opt, start_factor=1.0, end_factor=0.1,
                                              total_iters=499)
    x = x0.copy()
    m1 = np.zeros_like(x)
    m2 = np.zeros_like(x)
    for it in range(500):
        g = rng.standard_normal(40) * (1 + it % 7)
        assert abs(opt.param_groups[0]["lr"] - oracle.lr(it, 500, 0.1, 0.01)) < 1e-15
        xt.grad = torch.tensor(g)
        opt.step()
        sched.step()
        oracle.adam_step(x, g, m1, m2, it + 1, oracle.lr(it, 500, 0.1, 0.01))
    assert np.allclose(x, xt.detach().numpy(), rtol=1e-12, atol=1e-12)
    assert abs(oracle.lr(249, 499, 0.1, 0.01) - 0.055) < 1e-15  # midpoint


def test_adam_first_step_and_mask(oracle):
    """the bias-corrected first step moves lr*g/(|g|+eps) ~ lr*sign(g); masked
    (frozen) entries such as delta (PAPER.md:208 optimizes five) stay untouched."""
    x = np.array([1.0, 2.0, 3.0])
    g = np.array([0.5, -3.0, 7.0])
    m1 = np.zeros(3)
    m2 = np.zeros(3)
    oracle.adam_step(x, g, m1, m2, 1, 0.1, mask=np.array([1, 1, 0], np.uint8))
    assert np.allclose(x[:2], [1.0 - 0.1, 2.0 + 0.1], atol=1e-8) and x[2] == 3.0


def test_projection_boxes(oracle):
    """PAPER.md:208 boxes, matched positionally (R#15); idempotent."""
    p = np.array([[12.3, 4.0], [0.05, 9.0], [0.5, 11.0], [0.05, 6.0], [70.0, 10.0],
                  [4.0, -3.0]])
    oracle.project(p)
    assert p.tolist() == [[10.0, 5.0], [0.1, 5.0], [1.0, 10.0], [0.1, 5.0], [60.0, 20.0],
                          [4.0, -3.0]]
    q = p.copy()
    oracle.project(q)
    assert np.array_equal(p, q)


def test_fit_reduces_loss_c1(oracle):
    """The paper's fitting recipe on C1 (1 lane x 10 vehicles, 100 steps,
    noise-free truth): 500 iterations cut the Eq. 4 loss substantially and keep every
    parameter inside its box."""
    w = synth.make_workload("C1")
    h = oracle.leader_from_lanes(w.lane_offsets)
    P_true, _ = oracle.rollout(h, w.length, w.p0, w.v0, w.theta_true, w.K)
    obs = P_true.astype(np.float32).astype(np.float64)
    st = dict(leader=h, length=w.length, p0=w.p0, v0=w.v0,
              params=synth.init_params(w.n).astype(np.float64), m1=np.zeros((6, w.n)),
              m2=np.zeros((6, w.n)))
    losses = []
    for it in range(500):
        L, _ = oracle.fit_iteration(st, obs, it)
        losses.append(L)
    assert losses[-1] < losses[0] / 20
    p = st["params"]
    for k, (lo, hi) in enumerate([(5, 10), (0.1, 5), (1, 10), (0.1, 5), (20, 60)]):
        assert p[k].min() >= lo and p[k].max() <= hi
    assert np.all(p[5] == 4.0)


# ------------------------------------------------------------ virtual-leader mode
def test_virtual_leader_reproduces_lane_rollout(oracle):
    """fed the (dp, dv) a real leader produced, the virtual-leader rollout of the
    follower is the lane rollout's follower trajectory exactly (same arithmetic)."""
    w = synth.make_workload("C1", lane_sizes=[2], K=120, seed=4)
    h = oracle.leader_from_lanes(w.lane_offsets)
    th = w.theta_true.astype(np.float64)
    P, V = oracle.rollout(h, w.length, w.p0, w.v0, th, w.K)
    dp = (P[:-1, 1] - P[:-1, 0] - w.length[1].astype(np.float64))[:, None]
    dv = (V[:-1, 0] - V[:-1, 1])[:, None]
    Pv, Vv = oracle.rollout_vl(w.p0[:1], w.v0[:1], th[:, :1], dp, dv)
    assert np.array_equal(Pv[:, 0], P[:, 0]) and np.array_equal(Vv[:, 0], V[:, 0])


def test_virtual_leader_far_gap_is_free_road(oracle):
    """A virtual leader 1e9 m ahead at the same speed is the free road to rounding: the lone
    vehicle at its closed-form equilibrium speed v_f stays there."""
    th = np.array([7.0, 1.5, 2.0, 1.2, 30.0, 4.0])
    vf = free_road_equilibrium_speed(th)
    K = 200
    P, V = oracle.rollout_vl([0.0], [vf], th, np.full((K, 1), 1e9), np.zeros((K, 1)))
    assert np.max(np.abs(V - vf)) < 1e-9


def test_virtual_leader_paper_init_accelerates_from_rest(oracle):
    """dp = 10, dv = 0 (the paper's init) with default parameters and
    v0 = 0: speeds never go negative and rise toward the equilibrium of the 10 m gap."""
    K = 300
    P, V = oracle.rollout_vl([0.0], [0.0], DEFAULT, np.full((K, 1), 10.0), np.zeros((K, 1)))
    v = V[:, 0]
    assert v.min() >= 0.0
    i_peak = int(np.argmax(v))
    assert np.all(np.diff(v[:i_peak + 1]) >= -1e-12) and v[i_peak] > 1.0


@pytest.mark.parametrize("kind", ["l2", "l1"])
def test_virtual_leader_adjoint_matches_dual_numbers(oracle, kind):
    """Hand adjoint of the virtual-leader rollout vs forward-mode dual numbers, in the
    directions of p0, v0, all parameters and every dp_k, dv_k (clamped steps included)."""
    rng = np.random.default_rng(7)
    n, K = 5, 60
    th = np.stack([rng.uniform(5, 10, n), rng.uniform(0.5, 3, n), rng.uniform(1.5, 4, n),
                   rng.uniform(0.8, 2, n), rng.uniform(25, 40, n), rng.uniform(3, 5, n)])
    p0 = rng.uniform(0, 50, n)
    v0 = rng.uniform(5, 20, n)
    dp = rng.uniform(5, 40, (K, n))
    dp[3, 1] = 0.05  # a clamped gap (R#7)
    dv = rng.uniform(-3, 3, (K, n))
    P, V = oracle.rollout_vl(p0, v0, th, dp, dv)
    obs = P + rng.normal(0, 0.3, P.shape)
    L, gP = oracle.loss(P, obs, kind)
    g = oracle.backward_vl(th, dp, dv, P, V, gP)
    assert g["g_dp"][3, 1] == 0.0
    for _ in range(5):
        d = [rng.standard_normal(x.shape) for x in (p0, v0, th, dp, dv)]
        _, dP = oracle.rollout_vl_tangent(p0, v0, th, dp, dv, *d)
        fwd = float(np.sum(gP * dP))
        rev = float(np.sum(g["g_p0"] * d[0]) + np.sum(g["g_v0"] * d[1]) +
                    np.sum(g["g_params"] * d[2]) + np.sum(g["g_dp"] * d[3]) +
                    np.sum(g["g_dv"] * d[4]))
        assert abs(fwd - rev) <= 1e-10 * max(1.0, abs(fwd)), (fwd, rev)


# ------------------------------------------------------- reconstruction bookkeeping
def test_nearest_step_and_table1_worked_values():
    """SPEC.md:300-302 (alignment), :421-441 (metrics) worked values."""
    from oracle import tasks_oracle as T
    assert T.nearest_step(0.34, 0.1) == 3
    assert T.nearest_step(0.35, 0.1) == 4  # half-up tie
    assert T.nearest_step(0.0, 0.7) == 0
    assert T.nearest_step(2.5, 1.0) == 3 and T.nearest_step(2.49, 1.0) == 2
    # exact fit -> 0 %; one data point off by 1 m on a 1000 m trajectory, 10 points -> 0.01 %
    P = [[0.0], [100.0], [200.0], [300.0], [400.0], [500.0], [600.0], [700.0], [800.0],
         [900.0], [1000.0]]
    pts = {0: [(0.1 * k, P[k][0]) for k in range(1, 11)]}
    assert T.positional_error_rate(P, pts, 0.1) == 0.0
    pts[0][3] = (0.4, P[4][0] + 1.0)
    assert abs(T.positional_error_rate(P, pts, 0.1) - 0.01) < 1e-12
    assert T.acceleration_stats([0.0, 0.0]) == (0.0, 0.0)
    assert T.acceleration_stats([1.0, -1.0]) == (1.0, 0.0)
    assert T.acceleration_stats([0.0, 2.0]) == (1.0, 1.0)
    assert T.implausible([66.0]) and not T.implausible([10.0]) and not T.implausible([3, -3])
    L, g = T.loss_sparse([[0.0], [8.0]], [(0, 0.1, 10.0, 0.1)])
    assert L == 2.0 and g == {(1, 0): -1.0}


def test_product_alignment_agrees_with_oracle_alignment():
    """The host-side alignment of the product (tasks.nearest_steps) against the decimal
    half-up oracle on random and tie timestamps."""
    from oracle import tasks_oracle as T
    from paper_2412_16750_b200 import tasks
    rng = np.random.default_rng(0)
    for dt in (0.1, 1.0, 0.25):
        Ts = list(np.round(rng.uniform(0, 300, 500), 3)) + [dt * (k + 0.5) for k in range(50)]
        got = tasks.nearest_steps(Ts, dt)
        exp = [T.nearest_step(float(t), dt) for t in Ts]
        assert list(got) == exp


def test_rollout_converges_to_the_ode_at_first_order(oracle):
    """The multi-step rollout (leader gather, synchronous update, explicit Euler of Eq. 3,
    PAPER.md:121-128) against an independent integrator: scipy's adaptive RK45 on the ODE
    dp/dt = v, dv/dt = a*(v, Delta p, Delta v) of the same lane, with a* from the oracle's
    scalar accel (pinned on its own above) at a step so small that a_lb = a_min.  Euler is
    first order, so the error at T = 3 s halves with dt (ratio 2 +- 0.3) and is small."""
    from scipy.integrate import solve_ivp

    theta = np.array([[7.0, 1.5, 2.5, 1.2, 30.0, 4.0],
                      [8.5, 2.0, 3.0, 1.0, 33.0, 4.0],
                      [6.0, 1.8, 2.0, 1.5, 28.0, 4.0]]).T.copy()  # [6][3]
    length = np.array([4.5, 5.0, 4.2])
    p0 = np.array([0.0, 22.0, 47.0])   # lane-sorted, vehicle 2 leads
    v0 = np.array([14.0, 12.0, 10.0])
    leader = oracle.leader_from_lanes([0, 3])
    T = 3.0

    def rhs(_, y):
        p, v = y[:3], y[3:]
        a = np.empty(3)
        for i in range(3):
            h = leader[i]
            if h < 0:
                a[i] = oracle.accel(theta[:, i], v[i], 0.0, 0.0, has_leader=False, dt=1e-9)
            else:
                a[i] = oracle.accel(theta[:, i], v[i], p[h] - p[i] - length[h], v[i] - v[h],
                                    has_leader=True, dt=1e-9)
        return np.concatenate([v, a])

    ref = solve_ivp(rhs, (0.0, T), np.concatenate([p0, v0]), method="RK45", rtol=1e-11,
                    atol=1e-11).y[:, -1]
    errs = []
    for dt in (0.01, 0.005, 0.0025):
        K = int(round(T / dt))
        P, V = oracle.rollout(leader, length, p0, v0, theta, K, dt=dt)
        errs.append(max(np.max(np.abs(P[K] - ref[:3])), np.max(np.abs(V[K] - ref[3:]))))
    r1, r2 = errs[0] / errs[1], errs[1] / errs[2]
    assert 1.7 < r1 < 2.3 and 1.7 < r2 < 2.3, (errs, r1, r2)
    assert errs[2] < 0.05


def test_state_from_obs_worked_values():
    """PAPER.md:267 initialisation (v(0) = Delta P / Delta t of the first two data points), by
    hand: vehicle 0 first seen at step 1 (5.0) then step 3 (6.0), dt = 0.5 -> v0 = 1 / 1.0 = 1,
    p0 = 5 - 0.5 * 1 = 4.5; vehicle 1 at steps 0, 1 -> v0 = 1 / 0.5 = 2, p0 = 0; vehicle 2
    moving backwards -> v0 clamped to 0 (no backward motion), p0 = its first
    point; vehicle 3 seen once -> (its point, 0); vehicle 4 never -> (0, 0)."""
    from oracle import tasks_oracle as TO
    nan = float("nan")
    obs = [[nan, 0.0, 7.0, nan, nan],
           [5.0, 1.0, 6.0, nan, nan],
           [nan, 2.5, 5.0, 3.0, nan],
           [6.0, nan, nan, nan, nan]]
    p0, v0 = TO.state_from_obs(obs, 0.5)
    assert p0 == [4.5, 0.0, 7.0, 3.0, 0.0]
    assert v0 == [1.0, 2.0, 0.0, 0.0, 0.0]
