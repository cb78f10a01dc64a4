// idm_device.cuh -- per-vehicle IDM step math for sm_100a (forward step and its adjoint).
//
// Internal state is the GAP form of Eq. 3: each vehicle carries
// s_i = p_{h(i)} - p_i - length_{h(i)} (its gap Delta p), its speed v_i and
// its displacement D_i = p_i - p_i(0).  Euler (Eq. 3) in this form is
//     s' = s + dt (v_h - v),   v' = v + dt a*,   D' = D + dt v,
// mathematically identical to the paper's position update and far better conditioned in
// fp32 (no km-scale cancellation in the gap).
//
// The softplus arguments are carried in base-2 units (x2 = x log2 e) with the log2(e) / ln 2
// factors folded into per-vehicle constants, so each softplus is ex2 + lg2 + 3 FP ops.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace idm {

constexpr int kCap = 512;      // lane-tile capacity (vehicles per CTA)

constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.6931471805599453f;
constexpr float kLn2Sq = 0.4804530139182014f;

struct Consts {
    float dt, inv_dt, a_min, eps;
    float dt_ln2;     // dt ln 2
    float a_min2;     // a_min log2 e
    float ninv_dt2;   // -log2(e) / dt
};

// Forward constants of one vehicle (hoisted out of the time loop), base-2 scaled:
//   s_opt log2e = sm2 + v (T2 + dv c2)          (Eq. 1)
//   a_raw log2e = am2 (1 - w) - amln2 qr^2      (Eq. 2, qr = s*_opt log2e / dp)
struct VehP {
    float sm2, T2, c2, ivt, am2, amln2, delta;
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

__device__ __forceinline__ VehP make_vehp(float a_max, float a_pref, float s_min, float T,
                                          float v_targ, float delta) {
    VehP p;
    float c = 0.5f / sqrtf(a_max * a_pref);  // 1 / (2 sqrt(a_max a_pref))  (Eq. 1)
    p.sm2 = s_min * kLog2e;
    p.T2 = T * kLog2e;
    p.c2 = c * kLog2e;
    p.ivt = 1.f / v_targ;
    p.am2 = a_max * kLog2e;
    p.amln2 = a_max * kLn2;
    p.delta = delta;
    return p;
}

// Everything one step computes from (s, v, v_leader) before the state update; shared by the
// forward update and the adjoint so both see the same values.
struct Core {
    float x, x2, w, dv, c12, s_opt2, es, ones, ss2, idp, qr, inter2, t1, vda, z2, ea, onea, lx;
    bool lb_act;
};

// Eqs. 1-2 with the Sec. III-C bounds, exact free road
// without a leader (R#8), gap clamped at eps (R#7).  Explicit _rn intrinsics: the forward
// kernel and the backward recompute produce bitwise identical states.
template <bool D4>
__device__ __forceinline__ void core_dv(float s, float v, float dv, bool lead, const VehP& p,
                                        const Consts& k, Core& c);

template <bool D4>
__device__ __forceinline__ void core(float s, float v, float vl, bool lead, const VehP& p,
                                     const Consts& k, Core& c) {
    core_dv<D4>(s, v, __fsub_rn(v, vl), lead, p, k, c);  // Delta v = v_i - v_h
}

// The step core given the approach rate dv directly (virtual-leader mode, where
// (Delta p_k, Delta v_k) are free variables; the lane path passes dv = v - v_h).
template <bool D4>
__device__ __forceinline__ void core_dv(float s, float v, float dv, bool lead, const VehP& p,
                                        const Consts& k, Core& c) {
    c.x = __fmul_rn(v, p.ivt);
    c.x2 = __fmul_rn(c.x, c.x);
    if (D4) {
        c.w = __fmul_rn(c.x2, c.x2);  // (v / v_targ)^4
        c.lx = 0.f;
    } else {
        c.lx = c.x > 0.f ? lg2(c.x) : 0.f;
        c.w = c.x > 0.f ? ex2(__fmul_rn(p.delta, c.lx)) : 0.f;
    }
    c.dv = dv;
    c.c12 = __fmaf_rn(c.dv, p.c2, p.T2);
    c.s_opt2 = __fmaf_rn(v, c.c12, p.sm2);                     // s_opt log2 e
    c.es = ex2(-fabsf(c.s_opt2));
    c.ones = __fadd_rn(1.f, c.es);
    c.ss2 = __fadd_rn(fmaxf(c.s_opt2, 0.f), lg2(c.ones));      // softplus(s_opt) log2 e
    c.idp = rcp(fmaxf(s, k.eps));                              // 1 / Delta p
    c.qr = __fmul_rn(c.ss2, c.idp);                            // (s*/Delta p) log2 e
    c.inter2 = lead ? __fmul_rn(c.qr, c.qr) : 0.f;
    c.t1 = __fsub_rn(1.f, c.w);
    const float a_raw2 = __fmaf_rn(-p.amln2, c.inter2, __fmul_rn(p.am2, c.t1));
    c.vda = __fmaf_rn(k.dt, k.a_min, v);                       // v + dt a_min
    c.lb_act = c.vda < 0.f;                                    // a_lb = -v/dt branch
    const float a_lb2 = c.lb_act ? __fmul_rn(v, k.ninv_dt2) : k.a_min2;
    c.z2 = __fsub_rn(a_raw2, a_lb2);                           // (a - a_lb) log2 e
    c.ea = ex2(-fabsf(c.z2));
    c.onea = __fadd_rn(1.f, c.ea);
}

// State update of one vehicle from its step core (Eq. 3).  v' = v + dt a* computed as
// max(0, v + dt a_min) + dt softplus(a - a_lb): exact identity, >= 0 in floats.
__device__ __forceinline__ void advance(const Core& c, float& s, float& v, bool lead,
                                        const Consts& k) {
    const float sp2 = __fadd_rn(fmaxf(c.z2, 0.f), lg2(c.onea));  // softplus(a - a_lb) log2 e
    const float vn = __fmaf_rn(k.dt_ln2, sp2, fmaxf(c.vda, 0.f));
    if (lead) s = __fmaf_rn(-k.dt, c.dv, s);                       // s + dt (v_h - v)
    v = vn;
}

// One synchronous IDM + Euler step of one vehicle (Eqs. 1-3, Sec. III-C).
template <bool D4>
__device__ __forceinline__ void fwd_step(float& s, float& v, float vl, bool lead, const VehP& p,
                                         const Consts& k) {
    Core c;
    core<D4>(s, v, vl, lead, p, k, c);
    advance(c, s, v, lead, k);
}

// Backward-only per-vehicle constants.
struct VehB {
    float nam2ln2;  // -2 a_max ln2          (d a_raw / d s* = nam2ln2 qr idp)
    float ndamivt;  // -delta a_max / v_targ (d a_raw / d v, free term, times x^(delta-1))
    float nc;       // -c                    (d s_opt / d v_h)
};

__device__ __forceinline__ VehB make_vehb(float a_max, float a_pref, float v_targ, float delta) {
    VehB b;
    b.nam2ln2 = -2.f * a_max * kLn2;
    b.ndamivt = -delta * a_max / v_targ;
    b.nc = -0.5f / sqrtf(a_max * a_pref);
    return b;
}

// Accumulators of q * d a*/d theta, factored so per-vehicle constants are applied once at the
// end (q = dt lambda_v^{t+1}, qa = q sigma_a, qB = q d a*/d s_opt):
//   S1 = sum qa (1 - w - r^2)   S2 = sum qB v dv   S3 = sum qB   S4 = sum qB v
//   S5 = sum qa w               S6 = sum qa w log2 x
struct GradAcc {
    float S1, S2, S3, S4, S5, S6;
};

// Per vehicle-step record the backward recompute stores in shared memory (24 B), the local
// Jacobian of one step (derivation: DESIGN.md "Adjoint (gap form)"):
//   R1 = (sigma_a, beta = d a*/d s_opt, J_v = d a*/d v |_{v_h}, J_s = d a*/d s)
//   R2 = (1 - w - r^2, w log2 x)          with w = (v/v_targ)^delta, r = s*/dp
// sigma_a = d a*/d a_raw, d s*/d s_opt = sigmoid(s_opt) (:148); beta = 0 without
// a leader (R#8) and J_s = 0 while the gap is clamped (R#7).
template <bool D4>
__device__ __forceinline__ void jac_record(const Core& c, float s, float v, bool lead,
                                           const VehP& p, const VehB& b, const Consts& k,
                                           float4& R1, float2& R2) {
    const float rs = rcp(c.ones);
    const float sig_s = c.s_opt2 >= 0.f ? rs : c.es * rs;       // d s*/d s_opt
    const float ra = rcp(c.onea);
    const float eara = c.ea * ra;
    const bool zpos = c.z2 >= 0.f;
    const float sig_a = zpos ? ra : eara;                        // d a*/d a_raw
    const float omsa = zpos ? eara : ra;                         // d a*/d a_lb
    const float As = b.nam2ln2 * c.qr * c.idp;                  // d a_raw/d s*
    const float beta = lead ? sig_a * As * sig_s : 0.f;          // d a*/d s_opt
    const float xm1 = D4 ? c.x2 * c.x : (c.x > 0.f ? c.w * rcp(c.x) : 0.f);  // x^(delta-1)
    // d a*/d v at fixed leader speed: free term + s_opt term (T + (dv + v) c) + a_lb branch (R#5)
    float Jv = fmaf(beta * kLn2, fmaf(v, p.c2, c.c12), sig_a * b.ndamivt * xm1);
    if (c.lb_act) Jv = fmaf(-omsa, k.inv_dt, Jv);
    const float Js = (lead && s >= k.eps) ? -sig_a * As * c.qr * kLn2 : 0.f;
    const float lx = D4 ? (c.x > 0.f ? lg2(c.x) : 0.f) : c.lx;
    R1 = make_float4(sig_a, beta, Jv, Js);
    R2 = make_float2(fmaf(-kLn2Sq, c.inter2, c.t1), c.w * lx);
}

// Reverse step from the stored record: consumes lambda^{t+1} = (ls, lv, lD), returns F_out
// (this vehicle's term for its LEADER's lambda_v), updates ls, lv (the follower's F_in is added
// by the caller) and the gradient accumulators.  ls = 0 and beta = 0 for a lane head, so no
// leader predicates are needed.
template <bool D4>
__device__ __forceinline__ float bwd_from_record(float4 R1, float2 R2, float v, float vl,
                                                 const VehP& p, const VehB& b, const Consts& k,
                                                 float& ls, float& lv, float lD, GradAcc& g) {
    const float q = k.dt * lv;
    const float qa = q * R1.x;
    const float qb = q * R1.y;
    const float dtls = k.dt * ls;
    const float qbv = qb * v;
    const float F_out = fmaf(qbv, b.nc, dtls);                   // q d a*/d v_h + dt lambda_s
    lv = fmaf(k.dt, lD, fmaf(q, R1.z, lv)) - dtls;
    ls = fmaf(q, R1.w, ls);
    float w;
    if (D4) {
        const float x = v * p.ivt;
        const float x2 = x * x;
        w = x2 * x2;
    } else {
        const float x = v * p.ivt;
        w = x > 0.f ? ex2(p.delta * lg2(x)) : 0.f;
    }
    g.S1 = fmaf(qa, R2.x, g.S1);
    g.S2 = fmaf(qbv, v - vl, g.S2);
    g.S3 += qb;
    g.S4 += qbv;
    g.S5 = fmaf(qa, w, g.S5);
    g.S6 = fmaf(qa, R2.y, g.S6);
    return F_out;
}

// Virtual-leader reverse step: at state v with free leader terms (dp, dv) the
// local Jacobian is d a*/d v |_{dv} (dv is a leaf, so v enters only directly), d a*/d dp and
// d a*/d dv = beta v c.  Consumes lambda^{t+1} = (lv, lD); writes q d a*/d dp and q d a*/d dv
// (the leaf gradients of step t) and updates lv and the parameter accumulators.
template <bool D4>
__device__ __forceinline__ void bwd_vl(const Core& c, float dp, float v, const VehP& p,
                                       const VehB& b, const Consts& k, float& lv, float lD,
                                       GradAcc& g, float& gdp, float& gdv) {
    const float rs = rcp(c.ones);
    const float sig_s = c.s_opt2 >= 0.f ? rs : c.es * rs;
    const float ra = rcp(c.onea);
    const float eara = c.ea * ra;
    const bool zpos = c.z2 >= 0.f;
    const float sig_a = zpos ? ra : eara;
    const float omsa = zpos ? eara : ra;
    const float As = b.nam2ln2 * c.qr * c.idp;                  // d a_raw/d s*
    const float beta = sig_a * As * sig_s;                      // d a*/d s_opt
    const float xm1 = D4 ? c.x2 * c.x : (c.x > 0.f ? c.w * rcp(c.x) : 0.f);
    // d a*/d v at fixed dv: free term + s_opt term (T + dv c) + a_lb branch (R#5)
    float Jv = fmaf(beta * kLn2, c.c12, sig_a * b.ndamivt * xm1);
    if (c.lb_act) Jv = fmaf(-omsa, k.inv_dt, Jv);
    const float Js = dp >= k.eps ? -sig_a * As * c.qr * kLn2 : 0.f;  // R#7
    const float q = k.dt * lv;
    const float qa = q * sig_a;
    const float qb = q * beta;
    gdp = q * Js;
    gdv = -qb * v * b.nc;                                       // d s_opt/d dv = v c
    lv = fmaf(k.dt, lD, fmaf(q, Jv, lv));
    const float lx = D4 ? (c.x > 0.f ? lg2(c.x) : 0.f) : c.lx;
    g.S1 = fmaf(qa, fmaf(-kLn2Sq, c.inter2, c.t1), g.S1);
    const float qbv = qb * v;
    g.S2 = fmaf(qbv, c.dv, g.S2);
    g.S3 += qb;
    g.S4 += qbv;
    const float qaw = qa * c.w;
    g.S5 += qaw;
    g.S6 = fmaf(qaw, lx, g.S6);
}

}  // namespace idm
