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
//
// Every function is a template over the lane type T: T = float is one vehicle, T = float2 is
// TWO vehicles whose FP32 arithmetic issues as packed f32x2 instructions (FFMA2 / FMUL2 /
// FADD2, sm_100): one issue slot for two vehicles' multiply-adds.  The same template with the
// same operation order serves both widths and every rounding is explicit (_rn), so a vehicle
// gets bit-identical results whichever width computes it (FFMA2 = two FFMA.RN).
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
    float dt_amin;    // dt a_min (fp32 product)
    float dt2;        // dt^2 (fp32 product): scale of the lane adjoint's lambda_D
};

// ------------------------------------------------------------------ lane arithmetic
struct bool2 {
    bool x, y;
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
__device__ __forceinline__ float rsqrt_a(float x) {
    float y;
    asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ float2 ex2(float2 x) { return make_float2(ex2(x.x), ex2(x.y)); }
__device__ __forceinline__ float2 lg2(float2 x) { return make_float2(lg2(x.x), lg2(x.y)); }
__device__ __forceinline__ float2 rcp(float2 x) { return make_float2(rcp(x.x), rcp(x.y)); }

__device__ __forceinline__ float2 f2(float a) { return make_float2(a, a); }

__device__ __forceinline__ float vadd(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ float2 vadd(float2 a, float2 b) { return __fadd2_rn(a, b); }
__device__ __forceinline__ float2 vadd(float2 a, float b) { return __fadd2_rn(a, f2(b)); }
__device__ __forceinline__ float vsub(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ float2 vsub(float2 a, float2 b) {
    return __fadd2_rn(a, make_float2(-b.x, -b.y));
}
__device__ __forceinline__ float2 vsub(float a, float2 b) {
    return __fadd2_rn(make_float2(-b.x, -b.y), f2(a));
}
__device__ __forceinline__ float vmul(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ float2 vmul(float2 a, float2 b) { return __fmul2_rn(a, b); }
__device__ __forceinline__ float2 vmul(float2 a, float b) { return __fmul2_rn(a, f2(b)); }
__device__ __forceinline__ float vfma(float a, float b, float c) { return __fmaf_rn(a, b, c); }
__device__ __forceinline__ float2 vfma(float2 a, float2 b, float2 c) { return __ffma2_rn(a, b, c); }
__device__ __forceinline__ float2 vfma(float2 a, float b, float2 c) {
    return __ffma2_rn(a, f2(b), c);
}
__device__ __forceinline__ float vneg(float a) { return -a; }
__device__ __forceinline__ float2 vneg(float2 a) { return make_float2(-a.x, -a.y); }
__device__ __forceinline__ float vnabs(float a) { return -fabsf(a); }
__device__ __forceinline__ float2 vnabs(float2 a) { return make_float2(-fabsf(a.x), -fabsf(a.y)); }
__device__ __forceinline__ float vabs(float a) { return fabsf(a); }
__device__ __forceinline__ float2 vabs(float2 a) { return make_float2(fabsf(a.x), fabsf(a.y)); }
// -sign(a) with sign(0) = 0: one LOP3 copies the flipped sign bit onto 1, one select zeroes 0
__device__ __forceinline__ float vnsign(float a) { return a != 0.f ? copysignf(1.f, -a) : 0.f; }
__device__ __forceinline__ float2 vnsign(float2 a) { return make_float2(vnsign(a.x), vnsign(a.y)); }
__device__ __forceinline__ float vmax(float a, float b) { return fmaxf(a, b); }
__device__ __forceinline__ float2 vmax(float2 a, float b) {
    return make_float2(fmaxf(a.x, b), fmaxf(a.y, b));
}
__device__ __forceinline__ float2 vmax(float2 a, float2 b) {
    return make_float2(fmaxf(a.x, b.x), fmaxf(a.y, b.y));
}
__device__ __forceinline__ bool vge(float a, float b) { return a >= b; }
__device__ __forceinline__ bool2 vge(float2 a, float b) { return bool2{a.x >= b, a.y >= b}; }
__device__ __forceinline__ bool vgt(float a, float b) { return a > b; }
__device__ __forceinline__ bool2 vgt(float2 a, float b) { return bool2{a.x > b, a.y > b}; }
__device__ __forceinline__ float vsel(bool m, float a, float b) { return m ? a : b; }
__device__ __forceinline__ float2 vsel(bool2 m, float2 a, float2 b) {
    return make_float2(m.x ? a.x : b.x, m.y ? a.y : b.y);
}
template <class T> __device__ __forceinline__ T splat(float a);
template <> __device__ __forceinline__ float splat<float>(float a) { return a; }
template <> __device__ __forceinline__ float2 splat<float2>(float a) { return f2(a); }

// 0.5 + sign(z) |h| (z >= 0 keeps h's value bit for bit; one LOP3 per lane): with h = r - 0.5
// and r = 1 / (1 + 2^-|z|) in [0.5, 1] (Sterbenz: exact), this is sigmoid(z) and 0.5 - ... is
// 1 - sigmoid(z), branch-free.
__device__ __forceinline__ float vcopysign(float h, float z) { return copysignf(h, z); }
__device__ __forceinline__ float2 vcopysign(float2 h, float2 z) {
    return make_float2(copysignf(h.x, z.x), copysignf(h.y, z.y));
}

template <class T> struct MaskOf { using type = bool; };
template <> struct MaskOf<float2> { using type = bool2; };
template <class T> using Mask = typename MaskOf<T>::type;

// ------------------------------------------------------------------ per-vehicle constants
// Forward constants of one vehicle (hoisted out of the time loop), base-2 scaled:
//   s_opt log2e = sm2 + v (T2 + dv c2)          (Eq. 1)
//   a_raw log2e = am2 (1 - w) - amln2 qr^2      (Eq. 2, qr = s*_opt log2e / dp)
template <class T>
struct VehPT {
    T sm2, T2, c2, ivt, am2, amln2, delta;
};
using VehP = VehPT<float>;

__device__ __forceinline__ VehP make_vehp(float a_max, float a_pref, float s_min, float T,
                                          float v_targ, float delta) {
    VehP p;
    // per-vehicle reciprocals with the MUFU (a few ulp; every path shares these constants)
    const float c = __fmul_rn(0.5f, rsqrt_a(__fmul_rn(a_max, a_pref)));  // 1/(2 sqrt(a b)), Eq. 1
    p.sm2 = s_min * kLog2e;
    p.T2 = T * kLog2e;
    p.c2 = c * kLog2e;
    p.ivt = rcp(v_targ);
    p.am2 = a_max * kLog2e;
    p.amln2 = a_max * kLn2;
    p.delta = delta;
    return p;
}

__device__ __forceinline__ VehPT<float2> pack(const VehP& a, const VehP& b) {
    return VehPT<float2>{make_float2(a.sm2, b.sm2),     make_float2(a.T2, b.T2),
                         make_float2(a.c2, b.c2),       make_float2(a.ivt, b.ivt),
                         make_float2(a.am2, b.am2),     make_float2(a.amln2, b.amln2),
                         make_float2(a.delta, b.delta)};
}

// Everything one step computes from (s, v, v_leader) before the state update; shared by the
// forward update and the adjoint so both see the same values.
template <class T>
struct CoreT {
    T x, x2, w, dv, c12, s_opt2, es, ones, ss2, idp, qr, inter2, t1, r1, vda, z2, ea, onea, lx,
        vlb2;
};
using Core = CoreT<float>;

// Eqs. 1-2 with the Sec. III-C bounds, exact free road
// without a leader (R#8), gap clamped at eps (R#7), given the approach rate dv = v_i - v_h
// directly (the virtual-leader mode, passes its free variable).
// A vehicle without a leader (lane head, or an empty slot of a tile) carries the gap s = +inf:
// 1/Delta p = rcp(inf) = 0 makes the interaction term and every derivative through it vanish
// exactly, and s + dt (v_h - v) stays +inf.
// Explicit _rn intrinsics: every kernel that evaluates a step on the same state (the lane,
// on-chip-fit and virtual-leader forwards and backwards) gets the same bits.
template <bool D4, class T>
__device__ __forceinline__ void core_dv(T s, T v, T dv, const VehPT<T>& p, const Consts& k,
                                        CoreT<T>& c) {
    c.x = vmul(v, p.ivt);
    c.x2 = vmul(c.x, c.x);
    if (D4) {
        c.w = vmul(c.x2, c.x2);  // (v / v_targ)^4
        c.lx = splat<T>(0.f);
    } else {
        const Mask<T> xp = vgt(c.x, 0.f);
        c.lx = vsel(xp, lg2(c.x), splat<T>(0.f));
        c.w = vsel(xp, ex2(vmul(p.delta, c.lx)), splat<T>(0.f));
    }
    c.dv = dv;
    c.c12 = vfma(c.dv, p.c2, p.T2);
    c.s_opt2 = vfma(v, c.c12, p.sm2);                          // s_opt log2 e
    c.es = ex2(vnabs(c.s_opt2));
    c.ones = vadd(c.es, 1.f);
    c.idp = rcp(vmax(s, k.eps));                               // 1 / Delta p (0: no leader)
    c.ss2 = vadd(vmax(c.s_opt2, 0.f), lg2(c.ones));            // softplus(s_opt) log2 e
    c.qr = vmul(c.ss2, c.idp);                                 // (s*/Delta p) log2 e
    c.inter2 = vmul(c.qr, c.qr);
    c.t1 = vsub(1.f, c.w);
    c.r1 = vfma(c.inter2, -kLn2Sq, c.t1);                      // 1 - w - r^2 (backward only)
    c.vda = vadd(v, k.dt_amin);                                // v + dt a_min
    c.vlb2 = vmul(v, k.ninv_dt2);                              // (-v / dt) log2 e
    const T a_lb2 = vmax(c.vlb2, k.a_min2);                    // a_lb = max(-v/dt, a_min)
    // a_raw from (1 - w) and r^2 directly, not as a_max r1: r1 is off the forward's serial
    // chain (it feeds only the backward's dL/da_max), so the step's latency is one op shorter
    // (step 23)
    const T a_raw2 = vfma(vneg(p.amln2), c.inter2, vmul(p.am2, c.t1));
    c.z2 = vsub(a_raw2, a_lb2);                                // (a - a_lb) log2 e
    c.ea = ex2(vnabs(c.z2));
    c.onea = vadd(c.ea, 1.f);
}

template <bool D4, class T>
__device__ __forceinline__ void core(T s, T v, T vl, const VehPT<T>& p, const Consts& k,
                                     CoreT<T>& c) {
    core_dv<D4>(s, v, vsub(v, vl), p, k, c);  // Delta v = v_i - v_h
}

// State update of one vehicle from its step core (Eq. 3).  v' = v + dt a* computed as
// max(0, v + dt a_min) + dt softplus(a - a_lb): exact identity, >= 0 in floats.
// The gap moves by dt (v_h - v); a lane head's gap is never read (leadf = 0).
template <class T>
__device__ __forceinline__ void advance(const CoreT<T>& c, T& s, T& v, const Consts& k) {
    const T sp2 = vadd(vmax(c.z2, 0.f), lg2(c.onea));          // softplus(a - a_lb) log2 e
    const T vn = vfma(sp2, k.dt_ln2, vmax(c.vda, 0.f));
    s = vfma(c.dv, -k.dt, s);                                  // s + dt (v_h - v)
    v = vn;
}

// One synchronous IDM + Euler step (Eqs. 1-3, Sec. III-C).
template <bool D4, class T>
__device__ __forceinline__ void fwd_step(T& s, T& v, T vl, const VehPT<T>& p, const Consts& k) {
    CoreT<T> c;
    core<D4>(s, v, vl, p, k, c);
    advance(c, s, v, k);
}

// Eq. 4 terms of a vehicle (pair), branch-free: observed iff finite (NaN =
// missing; absent vehicles are fed NaN).  Returns dL/dP; adds the loss terms to acc.
template <int KIND, class T>
__device__ __forceinline__ T loss_term(T o, T P, T& acc) {
    const T r = vsub(o, P);
    const T rm = vsel(vge(vnabs(o), -3.4e38f), r, splat<T>(0.f));  // 0 where unobserved
    if (KIND == 0) {  // L1: |r|, dL/dP = -sign(r), sign(0) = 0 (R#11)
        acc = vadd(acc, vabs(rm));
        return vnsign(rm);
    }
    acc = vfma(rm, rm, acc);  // L2: r^2, dL/dP = -2 r
    return vmul(rm, -2.f);
}

// Backward-only per-vehicle constants.
template <class T>
struct VehBT {
    T nam2ln2;  // -2 a_max ln2          (d a_raw / d s* = nam2ln2 qr idp)
    T ndamivt;  // -delta a_max / v_targ (d a_raw / d v, free term, times x^(delta-1))
    T nc;       // -c                    (d s_opt / d v_h)
};
using VehB = VehBT<float>;

__device__ __forceinline__ VehB make_vehb(float a_max, float a_pref, float v_targ, float delta) {
    VehB b;
    b.nam2ln2 = -2.f * a_max * kLn2;
    b.ndamivt = __fmul_rn(__fmul_rn(-delta, a_max), rcp(v_targ));
    b.nc = __fmul_rn(-0.5f, rsqrt_a(__fmul_rn(a_max, a_pref)));
    return b;
}

// Backward constants of the LANE adjoint, scaled: the reverse
// sweep carries u = dt lambda_v (= q), m = -dt lambda_s and e = dt^2 lambda_D, so the per-step
// factors dt and ln 2 live in these constants instead of in multiplies:
//   Kb = -2 a_max ln2^2 dt    (d a_raw/d s* = nam2ln2 qr idp, times ln2 dt)
//   ndvt = -delta a_max dt / v_targ
//   ncl = -c / ln2            (d s_opt/d v_h over ln2)
template <class T>
struct VehAT {
    T Kb, ndvt, ncl;
};
using VehA = VehAT<float>;

__device__ __forceinline__ VehA make_veha(float a_max, float a_pref, float v_targ, float delta,
                                          const Consts& k) {
    VehA b;
    b.Kb = __fmul_rn(__fmul_rn(-2.f * a_max, kLn2Sq), k.dt);
    b.ndvt = __fmul_rn(__fmul_rn(__fmul_rn(-delta, a_max), rcp(v_targ)), k.dt);
    b.ncl = __fmul_rn(-0.5f * kLog2e, rsqrt_a(__fmul_rn(a_max, a_pref)));
    return b;
}

__device__ __forceinline__ VehAT<float2> pack(const VehA& a, const VehA& b) {
    return VehAT<float2>{make_float2(a.Kb, b.Kb), make_float2(a.ndvt, b.ndvt),
                         make_float2(a.ncl, b.ncl)};
}

// dL/d(a_max, a_pref, s_min, T_pref, v_targ, delta) of one vehicle from its factored
// accumulators (GradAcc) and raw parameters r; shared by every backward so they agree bitwise:
//   c = 1/(2 sqrt(a b)),  ds_opt/da = -c/(2a) v dv,  ds_opt/db = -c/(2b) v dv,
//   dw/dv_targ = -delta w / v_targ,  dw/ddelta = w ln x
__device__ __forceinline__ void param_grads(const float r[6], const float S[6], float gr[6]) {
    const float c = __fmul_rn(0.5f, rsqrt_a(__fmul_rn(r[0], r[1])));
    gr[0] = __fmaf_rn(-__fmul_rn(c, __fmul_rn(0.5f, rcp(r[0]))), S[1], S[0]);       // a_max
    gr[1] = __fmul_rn(-__fmul_rn(c, __fmul_rn(0.5f, rcp(r[1]))), S[1]);             // a_pref
    gr[2] = S[2];                                                                    // s_min
    gr[3] = S[3];                                                                    // T_pref
    gr[4] = __fmul_rn(__fmul_rn(__fmul_rn(r[0], r[5]), rcp(r[4])), S[4]);            // v_targ
    gr[5] = __fmul_rn(__fmul_rn(-r[0], kLn2), S[5]);                                  // delta
}

__device__ __forceinline__ VehBT<float2> pack(const VehB& a, const VehB& b) {
    return VehBT<float2>{make_float2(a.nam2ln2, b.nam2ln2), make_float2(a.ndamivt, b.ndamivt),
                         make_float2(a.nc, b.nc)};
}

// Accumulators of q * d a*/d theta, factored so per-vehicle constants are applied once at the
// end (q = dt lambda_v^{t+1}, qa = q sigma_a, qB = q d a*/d s_opt):
//   S1 = sum qa (1 - w - r^2)   S2 = sum qB v dv   S3 = sum qB   S4 = sum qB v
//   S5 = sum qa w               S6 = sum qa w log2 x
template <class T>
struct GradAccT {
    T S1, S2, S3, S4, S5, S6;
};
using GradAcc = GradAccT<float>;

// Local Jacobian of one vehicle-step of the LANE adjoint (derivation: DESIGN.md "Adjoint (gap
// form)" and "Adjoint scaling"): sigma_a = d a*/d a_raw; beta = (d a*/d s_opt) ln2 dt
// with d s*/d s_opt = sigmoid(s_opt) (:148); J_v = dt d a*/d v |_{v_h}; J_s = -dt^2 (d a*/d s)
// ln 2 / ln 2 = sAs qr (see jac_record); r1 = 1 - w - r^2, r2 = w log2 x with w = (v/v_targ)^delta,
// r = s*/dp.  beta = J_s = 0 without a leader (idp = 0, R#8) and J_s = 0 while the gap is clamped
// (R#7).
template <class T>
struct RecT {
    T sig_a, beta, Jv, Js, r1, r2;  // Jv: 1 + dt d a*/d v (see jac_record)
    T w, dv;  // (v/v_targ)^delta and v - v_h, reused by the reverse step
};

//   GD = false: dL/d delta is not wanted (delta frozen at 4 on an optimizer path): r2 = 0, and the
//   delta = 4 step skips the log2 x it would need.
template <bool D4, bool GD = true, class T>
__device__ __forceinline__ RecT<T> jac_record(const CoreT<T>& c, T s, T v, const VehPT<T>& p,
                                              const VehAT<T>& b, const Consts& k) {
    // 1/ones and 1/onea from ONE reciprocal (both in [1, 2], product in [1, 4])
    const T rp = rcp(vmul(c.ones, c.onea));
    const T hs = vcopysign(vfma(c.onea, rp, splat<T>(-0.5f)), c.s_opt2);
    const T sig_s = vadd(hs, 0.5f);                                  // d s*/d s_opt
    const T ha = vcopysign(vfma(c.ones, rp, splat<T>(-0.5f)), c.z2);
    const T sig_a = vadd(ha, 0.5f);                                  // d a*/d a_raw
    const T As = vmul(vmul(b.Kb, c.qr), c.idp);                     // (d a_raw/d s*) ln2 dt
    const T sAs = vmul(sig_a, As);
    RecT<T> R;
    R.w = c.w;
    R.dv = c.dv;
    R.sig_a = sig_a;
    R.beta = vmul(sAs, sig_s);                                       // (d a*/d s_opt) ln2 dt
    T xm1;                                                           // x^(delta-1)
    if (D4) xm1 = vmul(c.x2, c.x);
    else xm1 = vsel(vgt(c.x, 0.f), vmul(c.w, rcp(c.x)), splat<T>(0.f));
    // 1 + dt d a*/d v at fixed leader speed: free term + s_opt term (T + (dv + v) c; c2 = c
    // log2 e meets beta's ln 2) + a_lb branch (R#5: dt (1 - sigma_a)(-1/dt)).  The 1 of the
    // adjoint's lambda_v^{t+1} term rides in the FMA of the free term, and on the a_lb = -v/dt
    // branch 1 - (1 - sigma_a) = sigma_a replaces it (a select instead of two adds)
    const Mask<T> lb_act = vgt(c.vlb2, k.a_min2);                    // a_lb = -v/dt branch
    R.Jv = vfma(R.beta, vfma(v, p.c2, c.c12),
                vfma(vmul(sig_a, b.ndvt), xm1, vsel(lb_act, sig_a, splat<T>(1.f))));
    // d a*/d Delta p = sig_a (d a_raw/d s*)(-qr ln2) (log2 units): -dt^2 times it is sAs qr
    R.Js = vsel(vge(s, k.eps), vmul(sAs, c.qr), splat<T>(0.f));
    // log2 x (x = 0: w = 0 makes w log2 x = 0 with log2 of the smallest normal)
    R.r1 = c.r1;
    if (GD) {
        const T lx = D4 ? lg2(vmax(c.x, 1.17549435e-38f)) : c.lx;
        R.r2 = vmul(c.w, lx);
    } else {
        R.r2 = splat<T>(0.f);
    }
    return R;
}

// Reverse step of the lane adjoint from the stored record, in the scaled variables
//   u = dt lambda_v (= q of the paper's recursion),  m = -dt lambda_s,  e = dt^2 lambda_D:
//   lambda_v^t = lambda_v + q J_v + dt lambda_D - dt lambda_s   ->  u' = u (1 + Jv) + (e - dt^2 lambda_s)
//   lambda_s^t = lambda_s + q J_s                              ->  m' = m + u Js
// Consumes (u, m, e) of step t + 1; returns dt F_out (this vehicle's term for its LEADER's u:
// dt (q d a*/d v_h + dt lambda_s)); updates u, m (the follower's term is added by the caller) and
// the accumulators (S2, S3, S4 scaled by ln2 dt: unscale_acc).  m = 0 and beta = 0 for a lane
// head, so no leader predicates are needed (vl only has to be finite there).
template <bool D4, bool GD = true, class T>
__device__ __forceinline__ T bwd_from_record(const RecT<T>& R, T v, T vl, const VehPT<T>& p,
                                             const VehAT<T>& b, const Consts& k, T& m, T& u,
                                             T e, GradAccT<T>& g) {
    const T qa = vmul(u, R.sig_a);
    const T qb = vmul(u, R.beta);
    const T qbv = vmul(qb, v);
    const T ndm = vmul(m, -k.dt);                                // dt^2 lambda_s
    const T F_out = vfma(qbv, b.ncl, ndm);
    m = vfma(u, R.Js, m);
    u = vfma(u, R.Jv, vsub(e, ndm));  // R.Jv holds 1 + dt d a*/d v
    g.S1 = vfma(qa, R.r1, g.S1);
    g.S2 = vfma(qbv, R.dv, g.S2);
    g.S3 = vadd(g.S3, qb);
    g.S4 = vadd(g.S4, qbv);
    g.S5 = vfma(qa, R.w, g.S5);
    if (GD) g.S6 = vfma(qa, R.r2, g.S6);
    return F_out;
}

// Undo the lane adjoint's scaling at the end of a rollout: S2, S3, S4 carry a factor ln2 dt
// (bwd_from_record), the initial-state gradients come from u = dt lambda_v, m = -dt lambda_s,
// e = dt^2 lambda_D (m_f: the follower's m, 0 without one):
//   dL/dv0 = lambda_v,  dL/dp0 = lambda_D - lambda_s + lambda_s(follower)   (gap form)
template <class T>
__device__ __forceinline__ void unscale_acc(GradAccT<T>& g, const Consts& k) {
    const float us = __fmul_rn(kLog2e, k.inv_dt);  // 1 / (ln2 dt)
    g.S2 = vmul(g.S2, us);
    g.S3 = vmul(g.S3, us);
    g.S4 = vmul(g.S4, us);
}
template <class T>
__device__ __forceinline__ T grad_v0(T u, const Consts& k) { return vmul(u, k.inv_dt); }
template <class T>
__device__ __forceinline__ T grad_p0(T e, T m, T m_f, const Consts& k) {
    return vmul(vadd(vmul(e, k.inv_dt), vsub(m, m_f)), k.inv_dt);
}

// Virtual-leader reverse step: at state v with free leader terms (dp, dv) the
// local Jacobian is d a*/d v |_{dv} (dv is a leaf, so v enters only directly), d a*/d dp and
// d a*/d dv = beta v c.  Consumes lambda^{t+1} = (lv, lD); writes q d a*/d dp and q d a*/d dv
// (the leaf gradients of step t) and updates lv and the parameter accumulators.
template <bool D4, class T>
__device__ __forceinline__ void bwd_vl(const CoreT<T>& c, T dp, T v, const VehPT<T>& p,
                                       const VehBT<T>& b, const Consts& k, T& lv, T lD,
                                       GradAccT<T>& g, T& gdp, T& gdv) {
    const T rp = rcp(vmul(c.ones, c.onea));
    const T hs = vcopysign(vfma(c.onea, rp, splat<T>(-0.5f)), c.s_opt2);
    const T sig_s = vadd(hs, 0.5f);
    const T ha = vcopysign(vfma(c.ones, rp, splat<T>(-0.5f)), c.z2);
    const T sig_a = vadd(ha, 0.5f);
    const T omsa = vsub(0.5f, ha);
    const T As = vmul(vmul(b.nam2ln2, c.qr), c.idp);            // d a_raw/d s*
    const T sAs = vmul(sig_a, As);
    const T beta = vmul(sAs, sig_s);                            // d a*/d s_opt
    T xm1;
    if (D4) xm1 = vmul(c.x2, c.x);
    else xm1 = vsel(vgt(c.x, 0.f), vmul(c.w, rcp(c.x)), splat<T>(0.f));
    // d a*/d v at fixed dv: free term + s_opt term (T + dv c) + a_lb branch (R#5)
    const T Jv0 = vfma(vmul(beta, kLn2), c.c12, vmul(vmul(sig_a, b.ndamivt), xm1));
    const T Jv = vsel(vgt(c.vlb2, k.a_min2), vfma(omsa, -k.inv_dt, Jv0), Jv0);
    const T Js = vsel(vge(dp, k.eps), vmul(vmul(sAs, c.qr), -kLn2), splat<T>(0.f));  // R#7
    const T q = vmul(lv, k.dt);
    const T qa = vmul(q, sig_a);
    const T qb = vmul(q, beta);
    gdp = vmul(q, Js);
    const T qbv = vmul(qb, v);
    gdv = vmul(vneg(qbv), b.nc);                                // d s_opt/d dv = v c
    lv = vfma(lD, k.dt, vfma(q, Jv, lv));
    const T lx = D4 ? lg2(vmax(c.x, 1.17549435e-38f)) : c.lx;
    g.S1 = vfma(qa, c.r1, g.S1);
    g.S2 = vfma(qbv, c.dv, g.S2);
    g.S3 = vadd(g.S3, qb);
    g.S4 = vadd(g.S4, qbv);
    const T qaw = vmul(qa, c.w);
    g.S5 = vadd(g.S5, qaw);
    g.S6 = vfma(qaw, lx, g.S6);
}

}  // namespace idm
