/*
 * idm_oracle.c -- plain, slow, fp64 CPU ORACLE for the differentiable IDM hot path
 * of arXiv 2412.16750 ("parallel differentiable traffic simulator").
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  The product path
 * (paper_2412_16750_b200/, libidm.so) never calls, links or includes anything here,
 * and nothing here includes or calls the product path.
 *
 * Citations "PAPER.md:N" are lines of the paper's LaTeX;
 * "SPEC.md:N" lines of the CPU-program spec written from it.  Where the paper is
 * silent the DESIGN.md reading number is given as "R#n".
 *
 * What it computes (literal, in the paper's order and notation):
 *   gather   dp = p_{h(i)} - p_i - length_{h(i)},  dv = v_i - v_{h(i)}   (Sec. III-A)
 *   Eq. 1    s_opt = s_min + v T_pref + v dv / (2 sqrt(a_max a_pref))
 *   III-C    s* = log(1 + exp(s_opt))
 *   Eq. 2    a = a_max [1 - (v/v_targ)^delta - (s_star/dp)^2]
 *   III-C    a_lb = max(-v/dt, a_min);  a* = a_lb + log(1+exp(a - a_lb))
 *   Eq. 3    p(t+dt) = p + dt v(t);  v(t+dt) = v + dt a*
 *   III-B    all vehicles updated from the same pre-step snapshot
 *   Eq. 4    L = sum |P_obs - P[k]|
 *   Adam     (Kingma & Ba), lr linear 0.1 -> 0.01, box clamp
 * plus the exact reverse-mode derivative of that discrete map (PAPER.md:134
 * "implemented in a differentiable manner"; the paper uses autograd),
 * derived here by hand in position form, and an independent forward-mode
 * (dual-number) derivative used to pin the hand adjoint.
 *
 * Readings of silent/ambiguous points:
 *   R#1 delta is an input (default 4);  R#5 a_lb tie -> a_min branch (zero v-derivative);
 *   R#7 dp < eps_gap is clamped to eps_gap with zero gradient;  R#8 no leader (h(i) = -1)
 *   => exact free road: the (s_star/dp)^2 term is absent and dv = 0;  R#6 explicit Euler with v(t);
 *   R#11 Eq. 4 is a sum, sign(0) = 0;  R#24 at v = 0, (v/v_targ)^delta = 0 with zero
 *   derivatives in v and delta.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define NPAR 6 /* parameter order: a_max, a_pref, s_min, T_pref, v_targ, delta */
enum { P_AMAX = 0, P_APREF = 1, P_SMIN = 2, P_T = 3, P_VTARG = 4, P_DELTA = 5 };

/* ------------------------------------------------------------------ scalars */

/* softplus(x) = log(1 + exp(x)), overflow-safe form */
double ora_softplus(double x) { return (x > 0.0 ? x : 0.0) + log1p(exp(-fabs(x))); }

/* d softplus / dx */
double ora_sigmoid(double x)
{
    if (x >= 0.0) return 1.0 / (1.0 + exp(-x));
    double e = exp(x);
    return e / (1.0 + e);
}

/* Eq. 1: raw optimal spacing */
double ora_optimal_spacing(double a_max, double a_pref, double s_min, double T_pref, double v,
                           double dv)
{
    return s_min + v * T_pref + v * dv / (2.0 * sqrt(a_max * a_pref));
}

/* Eq. 2 with the Sec. III-C softplus bounds.
   th = (a_max, a_pref, s_min, T_pref, v_targ, delta).  dp must already be clamped (R#7). */
double ora_accel(const double th[NPAR], double v, double dp, double dv, int has_leader, double dt,
                 double a_min)
{
    double a_max = th[P_AMAX], v_targ = th[P_VTARG], delta = th[P_DELTA];
    double free_term = (v > 0.0) ? pow(v / v_targ, delta) : 0.0; /* R#24 */
    double a_raw;
    if (has_leader) {
        double s_opt = ora_optimal_spacing(a_max, th[P_APREF], th[P_SMIN], th[P_T], v, dv);
        double s_star = ora_softplus(s_opt);
        double ratio = s_star / dp;
        a_raw = a_max * (1.0 - free_term - ratio * ratio);
    } else {
        a_raw = a_max * (1.0 - free_term); /* R#8: exact free road */
    }
    double a_lb = fmax(-v / dt, a_min);
    return a_lb + ora_softplus(a_raw - a_lb);
}

/* Partial derivatives of a* with respect to the primitive inputs (v at fixed dv, dp, dv)
   and the six parameters -- SPEC's IdmGradient contract, derived
   by the chain rule from the formulas of ora_accel.
   out[0] = a*, out[1] = da/dv (dv held fixed), out[2] = da/d(dp), out[3] = da/d(dv),
   out[4..9] = da/dtheta_k.  dp_clamped => out[2] = 0 (R#7). */
void ora_accel_partials(const double th[NPAR], double v, double dp, double dv, int has_leader,
                        int dp_clamped, double dt, double a_min, double out[10])
{
    double a_max = th[P_AMAX], a_pref = th[P_APREF], T = th[P_T];
    double v_targ = th[P_VTARG], delta = th[P_DELTA];
    double x = v / v_targ;
    double w = (v > 0.0) ? pow(x, delta) : 0.0;
    double dw_dv = (v > 0.0) ? delta * w / v : 0.0;          /* d/dv x^delta */
    double dw_dvtarg = (v > 0.0) ? -delta * w / v_targ : 0.0; /* d/dv_targ x^delta */
    double dw_ddelta = (v > 0.0) ? w * log(x) : 0.0;          /* d/ddelta x^delta */

    double a_raw, da_dv, da_ddp = 0.0, da_ddv = 0.0;
    double da_dth[NPAR] = {0, 0, 0, 0, 0, 0};
    if (has_leader) {
        double sq = sqrt(a_max * a_pref);
        double c = 1.0 / (2.0 * sq);
        double s_opt = ora_optimal_spacing(a_max, a_pref, th[P_SMIN], T, v, dv);
        double s_star = ora_softplus(s_opt);
        double sig_s = ora_sigmoid(s_opt); /* d s_star / d s_opt */
        double r = s_star / dp;
        a_raw = a_max * (1.0 - w - r * r);
        /* d a_raw / d s* */
        double da_dsstar = -2.0 * a_max * r / dp;
        double da_dsopt = da_dsstar * sig_s;
        /* s_opt partials */
        double dsopt_dv = T + dv * c;
        double dsopt_ddv = v * c;
        double dc_damax = -c / (2.0 * a_max);
        double dc_dapref = -c / (2.0 * a_pref);
        da_dv = -a_max * dw_dv + da_dsopt * dsopt_dv;
        da_ddv = da_dsopt * dsopt_ddv;
        da_ddp = dp_clamped ? 0.0 : 2.0 * a_max * r * r / dp;
        da_dth[P_AMAX] = (1.0 - w - r * r) + da_dsopt * v * dv * dc_damax;
        da_dth[P_APREF] = da_dsopt * v * dv * dc_dapref;
        da_dth[P_SMIN] = da_dsopt;
        da_dth[P_T] = da_dsopt * v;
        da_dth[P_VTARG] = -a_max * dw_dvtarg;
        da_dth[P_DELTA] = -a_max * dw_ddelta;
    } else {
        a_raw = a_max * (1.0 - w);
        da_dv = -a_max * dw_dv;
        da_dth[P_AMAX] = 1.0 - w;
        da_dth[P_VTARG] = -a_max * dw_dvtarg;
        da_dth[P_DELTA] = -a_max * dw_ddelta;
    }
    double a_lb = fmax(-v / dt, a_min);
    double lb_active = (-v / dt > a_min) ? 1.0 : 0.0; /* R#5: tie -> a_min branch */
    double sig_a = ora_sigmoid(a_raw - a_lb);
    out[0] = a_lb + ora_softplus(a_raw - a_lb);
    out[1] = sig_a * da_dv + (1.0 - sig_a) * lb_active * (-1.0 / dt);
    out[2] = sig_a * da_ddp;
    out[3] = sig_a * da_ddv;
    for (int k = 0; k < NPAR; ++k) out[4 + k] = sig_a * da_dth[k];
}

/* ----------------------------------------------------------------- gather */

/* Sec. III-A gather for vehicle i from the snapshot (p, v).
   Returns has_leader; writes the (clamped, R#7) gap, the clamp flag and dv. */
static int gather(int64_t i, const int32_t* leader, const double* len, const double* p,
                  const double* v, double eps_gap, double* dp, int* clamped, double* dv)
{
    int32_t h = leader[i];
    if (h < 0) {
        *dp = INFINITY;
        *clamped = 0;
        *dv = 0.0;
        return 0;
    }
    double gap = p[h] - p[i] - len[h];
    *clamped = gap < eps_gap;
    *dp = *clamped ? eps_gap : gap;
    *dv = v[i] - v[h];
    return 1;
}

static void load_theta(const double* params, int64_t n_par, int64_t i, double th[NPAR])
{
    int64_t j = (n_par == 1) ? 0 : i;
    for (int k = 0; k < NPAR; ++k) th[k] = params[k * n_par + j];
}

/* ---------------------------------------------------------------- rollout */

/* K synchronous Euler steps (Eq. 3; Sec. III-B).
   params: SoA [6][n_par], n_par = n (per-vehicle) or 1 (shared).
   P, V: [(K+1)][n] outputs (row t = state at step t).  A (nullable): [K][n] a*.
   Returns 0, or 1 + t if a non-finite value appeared while computing step t. */
int ora_rollout(int64_t n, const int32_t* leader, const double* len, const double* p0,
                const double* v0, const double* params, int64_t n_par, int32_t K, double dt,
                double a_min, double eps_gap, double* P, double* V, double* A)
{
    memcpy(P, p0, sizeof(double) * (size_t)n);
    memcpy(V, v0, sizeof(double) * (size_t)n);
    for (int32_t t = 0; t < K; ++t) {
        const double* p = P + (int64_t)t * n;
        const double* v = V + (int64_t)t * n;
        double* pn = P + (int64_t)(t + 1) * n;
        double* vn = V + (int64_t)(t + 1) * n;
        int bad = 0;
        for (int64_t i = 0; i < n; ++i) {
            double th[NPAR], dp, dv;
            int clamped;
            load_theta(params, n_par, i, th);
            int hl = gather(i, leader, len, p, v, eps_gap, &dp, &clamped, &dv);
            double a = ora_accel(th, v[i], dp, dv, hl, dt, a_min);
            pn[i] = p[i] + dt * v[i];
            vn[i] = v[i] + dt * a;
            if (A) A[(int64_t)t * n + i] = a;
            if (!isfinite(pn[i]) || !isfinite(vn[i])) bad = 1;
        }
        if (bad) return 1 + t;
    }
    return 0;
}

/* ------------------------------------------------------------------- loss */

/* Eq. 4: L = sum over observed (t, i) of |obs - P| (kind 0, L1) or
   (obs - P)^2 (kind 1, L2 variant for smooth parity tests).  mask (nullable) [(K+1)][n]:
   nonzero = observed.  sign_override (nullable, L1 only): use this sign of (obs - P) instead
   of the computed one (GPU sign-mask protocol).  gP [(K+1)][n] = dL/dP, with
   sign(0) = 0 (R#11).  Returns L. */
double ora_loss(int kind, int64_t n, int32_t K, const double* P, const double* obs,
                const uint8_t* mask, const int8_t* sign_override, double* gP)
{
    double L = 0.0;
    int64_t m = (int64_t)(K + 1) * n;
    for (int64_t e = 0; e < m; ++e) {
        if (mask && !mask[e]) {
            gP[e] = 0.0;
            continue;
        }
        double r = obs[e] - P[e];
        if (kind == 0) {
            L += fabs(r);
            double s = sign_override ? (double)sign_override[e] : (r > 0) - (r < 0);
            gP[e] = -s;
        } else {
            L += r * r;
            gP[e] = -2.0 * r;
        }
    }
    return L;
}

/* --------------------------------------------------------------- backward */

/* Exact reverse-mode derivative of ora_rollout (position form), given dL/dP at every step.
   Adjoint of Eq. 3 step t (state x^t = (p^t, v^t), a_i = a*(v_i, dp_i, dv_i; theta_i)):
     lp^t = gP^t + lp^{t+1} + sum_i q_i da_i/dp^t         (q_i = dt lv_i^{t+1})
     lv^t = lv^{t+1} + dt lp^{t+1} + sum_i q_i da_i/dv^t
     g_theta_i += q_i da_i/dtheta_i
   with dp_i = p_h - p_i - len_h, dv_i = v_i - v_h (h = leader(i)), so vehicle i's
   acceleration also feeds its leader's adjoints.  Terminal lp^K = gP^K, lv^K = 0.
   Outputs: g_params [6][n_par] (accumulated over vehicles when shared),
   g_abs [6][n_par] (nullable) = sum |q da/dtheta| (condition number for parity tolerance),
   g_p0 = dL/dp(0) = lp^0, g_v0 = dL/dv(0) = lv^0 (nullable),
   g_p0_abs, g_v0_abs (nullable) = the sum of |every term added| into lp resp. lv over the
   sweep (|gP^t|, |dt lp^{t+1}|, |q da/dx|), the state analogue of g_abs: the scale below which
   a state gradient is a cancellation of larger terms (SURVEY.md 8(c) parity protocol; DESIGN.md
   section 7).  Returns 0 or 1+t on non-finite. */
int ora_backward(int64_t n, const int32_t* leader, const double* len, const double* params,
                 int64_t n_par, int32_t K, double dt, double a_min, double eps_gap, const double* P,
                 const double* V, const double* gP, double* g_params, double* g_abs, double* g_p0,
                 double* g_v0, double* g_p0_abs, double* g_v0_abs)
{
    double* lp = (double*)malloc(sizeof(double) * (size_t)n);
    double* lv = (double*)malloc(sizeof(double) * (size_t)n);
    double* lp_new = (double*)malloc(sizeof(double) * (size_t)n);
    double* lv_new = (double*)malloc(sizeof(double) * (size_t)n);
    /* running sums of |terms| added into lp, lv (condition scale of the state gradients) */
    double* pa = (double*)calloc((size_t)n, sizeof(double));
    double* va = (double*)calloc((size_t)n, sizeof(double));
    memset(g_params, 0, sizeof(double) * NPAR * (size_t)n_par);
    if (g_abs) memset(g_abs, 0, sizeof(double) * NPAR * (size_t)n_par);
    for (int64_t i = 0; i < n; ++i) {
        lp[i] = gP[(int64_t)K * n + i];
        lv[i] = 0.0;
        pa[i] = fabs(lp[i]);
    }
    int rc = 0;
    for (int32_t t = K - 1; t >= 0; --t) {
        const double* p = P + (int64_t)t * n;
        const double* v = V + (int64_t)t * n;
        for (int64_t i = 0; i < n; ++i) {
            lp_new[i] = gP[(int64_t)t * n + i] + lp[i];
            lv_new[i] = lv[i] + dt * lp[i];
            pa[i] += fabs(gP[(int64_t)t * n + i]);
            va[i] += fabs(dt * lp[i]);
        }
        for (int64_t i = 0; i < n; ++i) {
            double th[NPAR], dp, dv, d[10];
            int clamped;
            load_theta(params, n_par, i, th);
            int hl = gather(i, leader, len, p, v, eps_gap, &dp, &clamped, &dv);
            ora_accel_partials(th, v[i], dp, dv, hl, clamped, dt, a_min, d);
            double q = dt * lv[i];
            /* v_i enters directly and through dv = v_i - v_h */
            lv_new[i] += q * (d[1] + d[3]);
            va[i] += fabs(q * (d[1] + d[3]));
            if (hl) {
                int32_t h = leader[i];
                lv_new[h] += q * (-d[3]);
                lp_new[i] += q * (-d[2]);
                lp_new[h] += q * d[2];
                va[h] += fabs(q * d[3]);
                pa[i] += fabs(q * d[2]);
                pa[h] += fabs(q * d[2]);
            }
            int64_t j = (n_par == 1) ? 0 : i;
            for (int k = 0; k < NPAR; ++k) {
                double c = q * d[4 + k];
                g_params[k * n_par + j] += c;
                if (g_abs) g_abs[k * n_par + j] += fabs(c);
            }
        }
        double* tmp;
        tmp = lp; lp = lp_new; lp_new = tmp;
        tmp = lv; lv = lv_new; lv_new = tmp;
        for (int64_t i = 0; i < n; ++i)
            if (!isfinite(lp[i]) || !isfinite(lv[i])) rc = 1 + t;
        if (rc) break;
    }
    if (g_p0) memcpy(g_p0, lp, sizeof(double) * (size_t)n);
    if (g_v0) memcpy(g_v0, lv, sizeof(double) * (size_t)n);
    if (g_p0_abs) memcpy(g_p0_abs, pa, sizeof(double) * (size_t)n);
    if (g_v0_abs) memcpy(g_v0_abs, va, sizeof(double) * (size_t)n);
    free(lp); free(lv); free(lp_new); free(lv_new); free(pa); free(va);
    return rc;
}

/* ------------------------------------------------ forward mode (dual numbers) */
/* An independent derivative: the same formulas as ora_accel re-evaluated in dual-number
   arithmetic (value, tangent), so the tangent is produced mechanically by the chain rule of
   each elementary operation, not by the hand-derived partials above. */

typedef struct { double x, d; } dual;
static dual dc(double x) { dual r = {x, 0.0}; return r; }
static dual dadd(dual a, dual b) { dual r = {a.x + b.x, a.d + b.d}; return r; }
static dual dsub(dual a, dual b) { dual r = {a.x - b.x, a.d - b.d}; return r; }
static dual dmul(dual a, dual b) { dual r = {a.x * b.x, a.d * b.x + a.x * b.d}; return r; }
static dual ddiv(dual a, dual b)
{
    dual r = {a.x / b.x, (a.d * b.x - a.x * b.d) / (b.x * b.x)};
    return r;
}
static dual dsqrt(dual a) { double s = sqrt(a.x); dual r = {s, a.d / (2.0 * s)}; return r; }
static dual dexp(dual a) { double e = exp(a.x); dual r = {e, e * a.d}; return r; }
static dual dlog(dual a) { dual r = {log(a.x), a.d / a.x}; return r; }
static dual dlog1p(dual a) { dual r = {log1p(a.x), a.d / (1.0 + a.x)}; return r; }
static dual dneg(dual a) { dual r = {-a.x, -a.d}; return r; }
static dual dabs(dual a) { return a.x >= 0.0 ? a : dneg(a); }
static dual dmax0(dual a) { return a.x > 0.0 ? a : dc(0.0); }
/* x^y = exp(y log x) for x > 0; 0 (all derivatives 0) at x = 0 (R#24) */
static dual dpow(dual x, dual y)
{
    if (x.x <= 0.0) return dc(0.0);
    return dexp(dmul(y, dlog(x)));
}
static dual dsoftplus(dual a) { return dadd(dmax0(a), dlog1p(dexp(dneg(dabs(a))))); }

static dual dual_accel(const dual th[NPAR], dual v, dual dp, dual dv, int has_leader, double dt,
                       double a_min)
{
    dual a_max = th[P_AMAX];
    dual free_term = dpow(ddiv(v, th[P_VTARG]), th[P_DELTA]);
    dual a_raw;
    if (has_leader) {
        dual two_sq = dmul(dc(2.0), dsqrt(dmul(a_max, th[P_APREF])));
        dual s_opt = dadd(dadd(th[P_SMIN], dmul(v, th[P_T])), ddiv(dmul(v, dv), two_sq));
        dual ratio = ddiv(dsoftplus(s_opt), dp);
        a_raw = dmul(a_max, dsub(dsub(dc(1.0), free_term), dmul(ratio, ratio)));
    } else {
        a_raw = dmul(a_max, dsub(dc(1.0), free_term));
    }
    /* a_lb = max(-v/dt, a_min); tie -> a_min (R#5) */
    dual neg_v_dt = ddiv(dneg(v), dc(dt));
    dual a_lb = (neg_v_dt.x > a_min) ? neg_v_dt : dc(a_min);
    return dadd(a_lb, dsoftplus(dsub(a_raw, a_lb)));
}

/* Rollout of Eq. 3 in dual numbers.  Seeds: tangents of p0 [n], v0 [n] and params
   [6][n_par] (any may be NULL = 0).  Outputs P [(K+1)][n] values and dP [(K+1)][n] tangents.
   Returns 0 or 1 + t on non-finite. */
int ora_rollout_tangent(int64_t n, const int32_t* leader, const double* len, const double* p0,
                        const double* v0, const double* params, int64_t n_par, int32_t K,
                        double dt, double a_min, double eps_gap, const double* tp0,
                        const double* tv0, const double* tparams, double* P, double* dP)
{
    dual* p = (dual*)malloc(sizeof(dual) * (size_t)n);
    dual* v = (dual*)malloc(sizeof(dual) * (size_t)n);
    dual* pn = (dual*)malloc(sizeof(dual) * (size_t)n);
    dual* vn = (dual*)malloc(sizeof(dual) * (size_t)n);
    for (int64_t i = 0; i < n; ++i) {
        p[i].x = p0[i]; p[i].d = tp0 ? tp0[i] : 0.0;
        v[i].x = v0[i]; v[i].d = tv0 ? tv0[i] : 0.0;
        P[i] = p[i].x; dP[i] = p[i].d;
    }
    int rc = 0;
    for (int32_t t = 0; t < K && !rc; ++t) {
        for (int64_t i = 0; i < n; ++i) {
            dual th[NPAR];
            int64_t j = (n_par == 1) ? 0 : i;
            for (int k = 0; k < NPAR; ++k) {
                th[k].x = params[k * n_par + j];
                th[k].d = tparams ? tparams[k * n_par + j] : 0.0;
            }
            int32_t h = leader[i];
            dual dp = dc(INFINITY), dv = dc(0.0);
            int hl = h >= 0;
            if (hl) {
                dual lenh = dc(len[h]);
                dp = dsub(dsub(p[h], p[i]), lenh);
                if (dp.x < eps_gap) dp = dc(eps_gap); /* R#7: clamp, zero gradient */
                dv = dsub(v[i], v[h]);
            }
            dual a = dual_accel(th, v[i], dp, dv, hl, dt, a_min);
            pn[i] = dadd(p[i], dmul(dc(dt), v[i]));
            vn[i] = dadd(v[i], dmul(dc(dt), a));
        }
        dual* tmp;
        tmp = p; p = pn; pn = tmp;
        tmp = v; v = vn; vn = tmp;
        for (int64_t i = 0; i < n; ++i) {
            P[(int64_t)(t + 1) * n + i] = p[i].x;
            dP[(int64_t)(t + 1) * n + i] = p[i].d;
            if (!isfinite(p[i].x) || !isfinite(v[i].x) || !isfinite(p[i].d) || !isfinite(v[i].d))
                rc = 1 + t;
        }
    }
    free(p); free(v); free(pn); free(vn);
    return rc;
}

/* --------------------------------------------------------------- optimizer */

/* Linear learning-rate decay lr0 -> lr1 over iterations 0..total-1 (R#16). */
double ora_lr(int32_t it, int32_t total, double lr0, double lr1)
{
    if (total <= 1) return lr0;
    return lr0 + (lr1 - lr0) * (double)it / (double)(total - 1);
}

/* One Adam step (Kingma & Ba, cited at PAPER.md:267), bias-corrected, t = 1-based step
   count, over m scalars; entries with mask[e] == 0 (nullable) are left untouched. */
void ora_adam_step(int64_t m, double* x, const double* g, double* m1, double* m2, int32_t t,
                   double lr, double beta1, double beta2, double eps, const uint8_t* mask)
{
    double bc1 = 1.0 - pow(beta1, (double)t);
    double bc2 = 1.0 - pow(beta2, (double)t);
    for (int64_t e = 0; e < m; ++e) {
        if (mask && !mask[e]) continue;
        m1[e] = beta1 * m1[e] + (1.0 - beta1) * g[e];
        m2[e] = beta2 * m2[e] + (1.0 - beta2) * g[e] * g[e];
        double mhat = m1[e] / bc1;
        double vhat = m2[e] / bc2;
        x[e] -= lr * mhat / (sqrt(vhat) + eps);
    }
}

/* Box constraints of PAPER.md:208, matched positionally (R#15) to
   (a_max, a_pref, T_pref, s_min, v_targ): [5,10], [0.1,5], [0.1,5], [1,10], [20,60].
   Stored here in parameter order (a_max, a_pref, s_min, T_pref, v_targ); delta is unbounded. */
static const double BOX_LO[5] = {5.0, 0.1, 1.0, 0.1, 20.0};
static const double BOX_HI[5] = {10.0, 5.0, 10.0, 5.0, 60.0};

/* Clamp the five bounded parameters of SoA [6][n_par] into their boxes. */
void ora_project(int64_t n_par, double* params)
{
    for (int k = 0; k < 5; ++k)
        for (int64_t j = 0; j < n_par; ++j) {
            double* x = &params[k * n_par + j];
            if (*x < BOX_LO[k]) *x = BOX_LO[k];
            if (*x > BOX_HI[k]) *x = BOX_HI[k];
        }
}

/* ----------------------------------------------------- virtual-leader mode */
/* PAPER.md:208 ("We also optimize the lists of Delta p_k and Delta v_k for each simulation step
   k, initializing them to 10 and 0"; SPEC rollout_virtual_leader): each
   trajectory is fitted alone and its leader terms at step k are free variables dp[k][i],
   dv[k][i] (step-major [K][n]) instead of the gather of Sec. III-A.  dp < eps_gap is clamped
   with zero gradient (R#7). */
int ora_rollout_vl(int64_t n, const double* p0, const double* v0, const double* params,
                   int64_t n_par, int32_t K, double dt, double a_min, double eps_gap,
                   const double* dp, const double* dv, double* P, double* V)
{
    memcpy(P, p0, sizeof(double) * (size_t)n);
    memcpy(V, v0, sizeof(double) * (size_t)n);
    for (int32_t t = 0; t < K; ++t) {
        int bad = 0;
        for (int64_t i = 0; i < n; ++i) {
            double th[NPAR];
            load_theta(params, n_par, i, th);
            double gap = dp[(int64_t)t * n + i];
            double dpu = gap < eps_gap ? eps_gap : gap;
            double p = P[(int64_t)t * n + i], v = V[(int64_t)t * n + i];
            double a = ora_accel(th, v, dpu, dv[(int64_t)t * n + i], 1, dt, a_min);
            P[(int64_t)(t + 1) * n + i] = p + dt * v;
            V[(int64_t)(t + 1) * n + i] = v + dt * a;
            if (!isfinite(P[(int64_t)(t + 1) * n + i]) || !isfinite(V[(int64_t)(t + 1) * n + i]))
                bad = 1;
        }
        if (bad) return 1 + t;
    }
    return 0;
}

/* Reverse mode of ora_rollout_vl: lp^t = gP^t + lp^{t+1}; lv^t = lv^{t+1} + dt lp^{t+1} +
   q da/dv (dv is a free variable here, so v enters only directly); g_dp[t] = q da/d(dp),
   g_dv[t] = q da/d(dv), g_theta += q da/dtheta, q = dt lv^{t+1}.  Outputs as ora_backward plus
   g_dp, g_dv [K][n]. */
int ora_backward_vl(int64_t n, const double* params, int64_t n_par, int32_t K, double dt,
                    double a_min, double eps_gap, const double* dp, const double* dv,
                    const double* P, const double* V, const double* gP, double* g_params,
                    double* g_abs, double* g_dp, double* g_dv, double* g_p0, double* g_v0,
                    double* g_p0_abs, double* g_v0_abs)
{
    (void)P;
    memset(g_params, 0, sizeof(double) * NPAR * (size_t)n_par);
    if (g_abs) memset(g_abs, 0, sizeof(double) * NPAR * (size_t)n_par);
    int rc = 0;
    for (int64_t i = 0; i < n; ++i) {
        double lp = gP[(int64_t)K * n + i], lv = 0.0;
        double pa = fabs(lp), va = 0.0; /* sums of |terms added| (as ora_backward) */
        double th[NPAR];
        load_theta(params, n_par, i, th);
        int64_t j = (n_par == 1) ? 0 : i;
        for (int32_t t = K - 1; t >= 0; --t) {
            double gap = dp[(int64_t)t * n + i];
            int clamped = gap < eps_gap;
            double d[10];
            ora_accel_partials(th, V[(int64_t)t * n + i], clamped ? eps_gap : gap,
                               dv[(int64_t)t * n + i], 1, clamped, dt, a_min, d);
            double q = dt * lv;
            double lp_new = gP[(int64_t)t * n + i] + lp;
            double lv_new = lv + dt * lp + q * d[1];
            pa += fabs(gP[(int64_t)t * n + i]);
            va += fabs(dt * lp) + fabs(q * d[1]);
            g_dp[(int64_t)t * n + i] = q * d[2];
            g_dv[(int64_t)t * n + i] = q * d[3];
            for (int k = 0; k < NPAR; ++k) {
                double c = q * d[4 + k];
                g_params[k * n_par + j] += c;
                if (g_abs) g_abs[k * n_par + j] += fabs(c);
            }
            lp = lp_new;
            lv = lv_new;
        }
        if (!isfinite(lp) || !isfinite(lv)) rc = 1;
        if (g_p0) g_p0[i] = lp;
        if (g_v0) g_v0[i] = lv;
        if (g_p0_abs) g_p0_abs[i] = pa;
        if (g_v0_abs) g_v0_abs[i] = va;
    }
    return rc;
}

/* Forward mode (dual numbers) of ora_rollout_vl, independent of the hand adjoint: seeds for
   p0, v0 [n], params [6][n_par], dp, dv [K][n] (each nullable).  Outputs P, dP [(K+1)][n]. */
int ora_rollout_vl_tangent(int64_t n, const double* p0, const double* v0, const double* params,
                           int64_t n_par, int32_t K, double dt, double a_min, double eps_gap,
                           const double* dp, const double* dv, const double* tp0,
                           const double* tv0, const double* tparams, const double* tdp,
                           const double* tdv, double* P, double* dP)
{
    int rc = 0;
    for (int64_t i = 0; i < n; ++i) {
        dual th[NPAR];
        int64_t j = (n_par == 1) ? 0 : i;
        for (int k = 0; k < NPAR; ++k) {
            th[k].x = params[k * n_par + j];
            th[k].d = tparams ? tparams[k * n_par + j] : 0.0;
        }
        dual p = {p0[i], tp0 ? tp0[i] : 0.0}, v = {v0[i], tv0 ? tv0[i] : 0.0};
        P[i] = p.x;
        dP[i] = p.d;
        for (int32_t t = 0; t < K; ++t) {
            int64_t e = (int64_t)t * n + i;
            dual gap = {dp[e], tdp ? tdp[e] : 0.0};
            if (gap.x < eps_gap) gap = dc(eps_gap); /* R#7: clamp, zero gradient */
            dual ddv = {dv[e], tdv ? tdv[e] : 0.0};
            dual a = dual_accel(th, v, gap, ddv, 1, dt, a_min);
            dual pn = dadd(p, dmul(dc(dt), v));
            dual vn = dadd(v, dmul(dc(dt), a));
            p = pn;
            v = vn;
            P[(int64_t)(t + 1) * n + i] = p.x;
            dP[(int64_t)(t + 1) * n + i] = p.d;
            if (!isfinite(p.x) || !isfinite(v.x)) rc = 1 + t;
        }
    }
    return rc;
}

/* Adam over unconstrained variables (the virtual-leader lists, PAPER.md:208 gives them no
   box): ora_adam_step without projection -- provided for symmetry of the fit loop. */
