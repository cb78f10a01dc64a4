// idm_device.cuh -- per-vehicle IDM step math for sm_100a (forward step and its adjoint).
//
// Internal state is the GAP form of Eq. 3: each vehicle
// carries s_i = p_{h(i)} - p_i - length_{h(i)} (its gap Delta p), its speed v_i
// and its displacement D_i = p_i - p_i(0).  Euler (Eq. 3) in this form is
//     s' = s + dt (v_h - v),   v' = v + dt a*,   D' = D + dt v,
// mathematically identical to the paper's position update and far better conditioned in fp32
// (no km-scale cancellation in the gap).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace idm {

constexpr int kThreads = 256;             // CTA size
constexpr int kVpt = 2;                   // vehicles per thread (ILP)
constexpr int kCap = kThreads * kVpt;     // lane-tile capacity (vehicles per CTA)
constexpr int kMaxCkpt = 48;              // max checkpoint interval k (smem history depth:
                                          // 48 x 513 x 8 B = 197 KB of the 227 KB per CTA)

struct Consts {
    float dt, inv_dt, a_min, eps;
};

// Forward constants of one vehicle (hoisted out of the time loop).
struct VehP {
    float a_max, s_min, T, inv_vtarg, delta, c;  // c = 1 / (2 sqrt(a_max a_pref))  (Eq. 1)
};

__device__ __forceinline__ float ex2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ float lg2(float x) {
    float y;
    asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ float rcp(float x) {
    float y;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.6931471805599453f;

// softplus(x) = log(1 + e^x) = max(x, 0) + log(1 + e^{-|x|})  (Sec. III-C);
// returns e = e^{-|x|} for the sigmoid.
__device__ __forceinline__ float softplus_e(float x, float& e) {
    e = ex2(__fmul_rn(-fabsf(x), kLog2e));
    return __fadd_rn(fmaxf(x, 0.f), __fmul_rn(lg2(__fadd_rn(1.f, e)), kLn2));
}

// (v / v_targ)^delta for x = v / v_targ >= 0 (delta = 4 is two squarings).
__device__ __forceinline__ float pow_delta(float x, float delta) {
    if (delta == 4.f) {
        float x2 = __fmul_rn(x, x);
        return __fmul_rn(x2, x2);
    }
    return x > 0.f ? ex2(__fmul_rn(delta, lg2(x))) : 0.f;
}

// One synchronous IDM + Euler step of one vehicle (Eqs. 1-3 with the Sec. III-C bounds).
// vl is the leader's speed v_{h(i)}(t) (ignored when !lead: exact free road, R#8).
// Written with explicit _rn intrinsics so the forward kernel and the backward recompute
// produce bitwise identical states (no compiler-chosen FMA contraction).
__device__ __forceinline__ void fwd_step(float& s, float& v, float vl, bool lead, const VehP& p,
                                         const Consts& k) {
    float x = __fmul_rn(v, p.inv_vtarg);
    float w = pow_delta(x, p.delta);
    float dv = __fsub_rn(v, vl);                                   // Delta v = v_i - v_h
    float s_opt = __fmaf_rn(v, __fmaf_rn(dv, p.c, p.T), p.s_min);  // Eq. 1
    float e;
    float s_star = softplus_e(s_opt, e);                           // s*_opt
    float dp = fmaxf(s, k.eps);                                    // R#7 clamp
    float r = __fmul_rn(s_star, rcp(dp));
    float inter = lead ? __fmul_rn(r, r) : 0.f;
    float a_raw = __fmul_rn(p.a_max, __fsub_rn(__fsub_rn(1.f, w), inter));  // Eq. 2
    float vda = __fmaf_rn(k.dt, k.a_min, v);                       // v + dt a_min
    // a_lb = max(-v/dt, a_min); -v/dt wins iff v + dt a_min < 0
    float a_lb = vda < 0.f ? __fmul_rn(-v, k.inv_dt) : k.a_min;
    float sp = softplus_e(__fsub_rn(a_raw, a_lb), e);              // a* = a_lb + sp (:149)
    // v' = v + dt a* = max(0, v + dt a_min) + dt sp  (exact identity; >= 0 in floats, :152)
    float vn = __fmaf_rn(k.dt, sp, fmaxf(vda, 0.f));
    if (lead) s = __fmaf_rn(k.dt, __fsub_rn(vl, v), s);            // gap form of Eq. 3
    v = vn;
}

// Accumulators of q * d a*/d theta, factored so per-vehicle constants are applied once at the
// end (q = dt * lambda_v^{t+1}, qa = q sigma_a, qB = qa * d a_raw/d s_opt):
//   S1 = sum qa (1 - w - r^2)   S2 = sum qB v dv   S3 = sum qB   S4 = sum qB v
//   S5 = sum qa w               S6 = sum qa w ln x
struct GradAcc {
    float S1, S2, S3, S4, S5, S6;
};

// Reverse step of one vehicle at state (s, v) with leader speed vl: consumes the adjoints
// lambda^{t+1} = (ls, lv, lD), returns F_out = dL contribution this vehicle sends to its
// LEADER's speed adjoint, and updates ls/lv (without the follower's F_in, added by the caller)
// and the gradient accumulators.  Derivation: DESIGN.md "Adjoint (gap form)".
__device__ __forceinline__ float bwd_step(float s, float v, float vl, bool lead, const VehP& p,
                                          const Consts& k, float& ls, float& lv, float lD,
                                          GradAcc& g) {
    float x = v * p.inv_vtarg;
    float w, xm1;  // x^delta, x^(delta-1)
    float lnx = x > 0.f ? lg2(x) * kLn2 : 0.f;
    if (p.delta == 4.f) {
        float x2 = x * x;
        xm1 = x2 * x;
        w = x2 * x2;
    } else {
        w = x > 0.f ? ex2(p.delta * lnx * kLog2e) : 0.f;
        xm1 = x > 0.f ? w * rcp(x) : 0.f;
    }
    float dv = v - vl;
    float c1 = fmaf(dv, p.c, p.T);
    float s_opt = fmaf(v, c1, p.s_min);
    float es = ex2(-fabsf(s_opt) * kLog2e);
    float s_star = fmaxf(s_opt, 0.f) + lg2(1.f + es) * kLn2;
    float rs = rcp(1.f + es);
    float sig_s = s_opt >= 0.f ? rs : es * rs;
    float dp = fmaxf(s, k.eps);
    float idp = rcp(dp);
    float r = s_star * idp;
    float r2 = lead ? r * r : 0.f;
    float a_raw = p.a_max * (1.f - w - r2);
    float vda = fmaf(k.dt, k.a_min, v);
    bool lb_act = vda < 0.f;
    float a_lb = lb_act ? -v * k.inv_dt : k.a_min;
    float z = a_raw - a_lb;
    float ea = ex2(-fabsf(z) * kLog2e);
    float ra = rcp(1.f + ea);
    float sig_a = z >= 0.f ? ra : ea * ra;
    float one_m_sig_a = z >= 0.f ? ea * ra : ra;

    float q = k.dt * lv;
    float qa = q * sig_a;
    float As = -2.f * p.a_max * r * idp;           // d a_raw / d s*
    float qB = lead ? qa * As * sig_s : 0.f;       // q d a*/d s_opt
    // q d a*/d v (leader speed held fixed; includes the a_lb branch, R#5)
    float dadv = qa * (-p.a_max * p.delta * xm1 * p.inv_vtarg) + qB * fmaf(v, p.c, c1);
    if (lb_act) dadv = fmaf(-q * one_m_sig_a, k.inv_dt, dadv);
    float F_out = lead ? fmaf(k.dt, ls, qB * (-v * p.c)) : 0.f;  // to the leader's lambda_v
    float ds = (lead && s >= k.eps) ? -qa * As * r : 0.f;         // q d a*/d s
    g.S1 = fmaf(qa, 1.f - w - r2, g.S1);
    g.S2 = fmaf(qB * v, dv, g.S2);
    g.S3 += qB;
    g.S4 = fmaf(qB, v, g.S4);
    g.S5 = fmaf(qa, w, g.S5);
    g.S6 = fmaf(qa * w, lnx, g.S6);
    float lv_new = lv + dadv + k.dt * lD - (lead ? k.dt * ls : 0.f);
    ls = lead ? ls + ds : 0.f;
    lv = lv_new;
    return F_out;
}

}  // namespace idm
