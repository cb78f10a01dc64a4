// idm_kernels.cu -- sm_100a kernels of the differentiable IDM hot path (arXiv 2412.16750).
//
//   NK0 validate_kernel   input checks (finite, v >= 0, params > 0)            once per init
//   NK1 fwd_kernel        K fused steps per lane tile, state in registers       Eqs. 1-3, III-C
//   NK2 loss_kernel       Eq. 4 L1/L2 + dL/dP, fixed-order fp64 partials
//   NK3 bwd_kernel        checkpoint recompute + reverse sweep per lane tile    adjoint of NK1
//   NK4 reduce_kernel     fixed-order sum of per-block fp64 partials (loss / shared grads)
//   NK5 adam_kernel       Adam + linear lr + box clamp
//
// A lane tile is a run of WHOLE lanes of at most kCap = 512 vehicles (lanes are independent, so
// no tile ever needs another tile's data).  A CTA of kT = 256 threads owns one tile; local
// vehicle id = j * kT + threadIdx.x (j < kVpt = 2), so every global access of a warp is 32
// consecutive floats and the leader of local vehicle id is id + 1, exchanged through shared
// memory (one barrier per step).  Checkpoint segments are KS steps (compile-time, unrolled);
// step-major rows (observations, dL/dP) are prefetched a segment ahead into registers.
#include <cstdint>
#include <type_traits>
#include <cuda_runtime.h>

#include "idm_device.cuh"
#include "idm_internal.h"

namespace idm {

// ------------------------------------------------------------------------------ NK0
__global__ void validate_kernel(ValidateArgs a) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (; i < a.n; i += stride) {
        float p = a.pos0[i], v = a.vel0[i], l = a.length[i];
        bool ok = isfinite(p) && isfinite(v) && isfinite(l) && v >= 0.f && l >= 0.f;
        if (!ok) atomicMin(a.status, (unsigned long long)(kBadInput) << 32 | (uint64_t)i);
    }
    int64_t m = 6 * a.n_par;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < m; e += stride) {
        float x = a.params[e];
        bool ok = isfinite(x) && x > 0.f;  // every IDM parameter is positive
        if (!ok) atomicMin(a.status, (unsigned long long)(kBadParam) << 32 | (uint64_t)e);
        if (e >= 5 * a.n_par && x != 4.f) atomicOr(a.delta_not4, 1u);
    }
}

__device__ __forceinline__ void report_nonfinite(unsigned long long* status, int step,
                                                 int64_t veh) {
    atomicMin(status, (unsigned long long)(unsigned)step << 32 | (uint64_t)(uint32_t)veh);
}

struct RawP {
    float a_max, a_pref, s_min, T, v_targ, delta;
};

__device__ __forceinline__ RawP load_raw(const float* __restrict__ prm, int64_t n_par,
                                         int64_t i) {
    const int64_t j = n_par == 1 ? 0 : i;
    RawP r;
    r.a_max = prm[j];
    r.a_pref = prm[n_par + j];
    r.s_min = prm[2 * n_par + j];
    r.T = prm[3 * n_par + j];
    r.v_targ = prm[4 * n_par + j];
    r.delta = prm[5 * n_par + j];
    return r;
}

__device__ __forceinline__ RawP dummy_raw() { return RawP{1.f, 1.f, 1.f, 1.f, 1.f, 4.f}; }

constexpr int kVpt = 2;          // vehicles per thread
constexpr int kT = kCap / kVpt;   // 256 threads per CTA

// Eq. 4 term of one observation, branch-free: observed iff finite (NaN =
// missing).  Returns dL/dP; adds the loss term to acc.
template <int KIND>
__device__ __forceinline__ float loss_term(float o, float P, bool valid, float& acc) {
    const float r = o - P;
    const bool ok = valid && fabsf(o) <= 3.4e38f;
    if (KIND == 0) {  // L1: |r|, dL/dP = -sign(r), sign(0) = 0 (R#11)
        acc += ok ? fabsf(r) : 0.f;
        const float sg = r > 0.f ? -1.f : (r < 0.f ? 1.f : 0.f);
        return ok ? sg : 0.f;
    }
    acc = ok ? fmaf(r, r, acc) : acc;  // L2: r^2, dL/dP = -2 r
    return ok ? -2.f * r : 0.f;
}

// fixed-order CTA reduction of one double per thread -> out[blockIdx.x] (deterministic)
__device__ __forceinline__ void block_sum_to(double x, double* out) {
    __shared__ double red[kT / 32];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = x;
    __syncthreads();
    if (threadIdx.x == 0) {
        double y = 0.0;
        for (int w = 0; w < kT / 32; ++w) y += red[w];
        out[blockIdx.x] = y;
    }
}

// ------------------------------------------------------------------------------ NK1
// One CTA = one lane tile.  All `steps` steps run in one launch, in checkpoint segments of KS
// steps (compile-time, fully unrolled; the K mod KS tail runs as one predicated segment); per
// step one __syncthreads separates the speed publication from the leader read
// (double-buffered exchange).  LOSS = 0: record P (idm_forward).  LOSS = 1 (L1) / 2 (L2):
// fused Eq. 4 for idm_fit_step -- the observation rows of the next segment are prefetched into
// registers while the current one runs; each step evaluates Eq. 4 against the fresh positions
// and writes dL/dP instead of P.
// CK = checkpoint interval (the backward's segment length); the forward's own prefetch
// segment is KS = max(4, CK) steps, so CK | KS and checkpoints fall at static positions.
template <bool D4, bool KAHAN, bool RECV, int LOSS, int CK>
__global__ void __launch_bounds__(kT, (CK > 4 ? 2 : (LOSS ? 3 : 4))) fwd_kernel(FwdArgs a) {
    constexpr int KS = CK > 4 ? CK : 4;
    __shared__ float xv[2][kCap + 1];
    const int tid = threadIdx.x;
    const int64_t base = a.tile_start[blockIdx.x];
    const int n_loc = (int)(a.tile_start[blockIdx.x + 1] - base);
    const Consts k = a.k;
    const int64_t N = a.n;
    const int steps = a.steps;
    const int nfull = steps / KS, tail = steps - nfull * KS;

    float s[kVpt], v[kVpt], D[kVpt], cmp[kVpt], p0[kVpt];
    bool lead[kVpt], valid[kVpt];
    VehP P[kVpt];
#pragma unroll
    for (int j = 0; j < kVpt; ++j) {
        const int id = j * kT + tid;
        const int64_t i = base + id;
        valid[j] = id < n_loc;
        D[j] = 0.f;
        cmp[j] = 0.f;
        RawP r = dummy_raw();
        if (valid[j]) {
            p0[j] = a.pos0[i];
            v[j] = a.vel0[i];
            lead[j] = a.lead[i] != 0;
            s[j] = lead[j] ? (a.pos0[i + 1] - p0[j]) - a.length[i + 1] : 0.f;
            r = load_raw(a.params, a.n_par, i);
            if (D4 && r.delta != 4.f)
                atomicMin(a.status, (unsigned long long)kBadDelta << 32 | (uint64_t)i);
        } else {
            p0[j] = 0.f; v[j] = 0.f; s[j] = 0.f; lead[j] = false;
        }
        P[j] = make_vehp(r.a_max, r.a_pref, r.s_min, r.T, r.v_targ, r.delta);
    }
    if (tid == 0) { xv[0][kCap] = 0.f; xv[1][kCap] = 0.f; }

    // out: P row (LOSS = 0) or dL/dP row (LOSS) of the current step
    float* orow = (LOSS ? a.grad_traj : a.traj) + base + tid;
    float* vrow = RECV ? a.vel_traj + base + tid : nullptr;
    float* cks = a.ckpt_s + base + tid;
    float* ckv = a.ckpt_v + base + tid;
    const float* obs = LOSS ? a.obs + base + tid : nullptr;
    float onx[KS][kVpt];  // LOSS: observation rows of the next segment (registers)
    float lseg = 0.f;     // loss of this thread's vehicles in this segment (fp32)
    double lacc = 0.0;    // and across segments (fp64)
    // prefetch the observation rows 1 .. KS (predicated for a short rollout)
    auto prefetch = [&](int row0, int nrows) {
        const float* o = obs + (int64_t)row0 * N;
#pragma unroll
        for (int tt = 0; tt < KS; ++tt, o += N)
#pragma unroll
            for (int j = 0; j < kVpt; ++j)
                onx[tt][j] = (valid[j] && tt < nrows) ? __ldcs(o + j * kT) : 0.f;
    };
    if (LOSS) prefetch(1, min(KS, steps));
#pragma unroll
    for (int j = 0; j < kVpt; ++j) {
        if (!valid[j]) continue;
        __stcs(orow + j * kT, LOSS ? loss_term<LOSS - 1>(obs[j * kT], p0[j], true, lseg) : p0[j]);
        if (RECV) vrow[j * kT] = v[j];
        cks[j * kT] = s[j];
        ckv[j * kT] = v[j];
    }
    int par = 0;
    // one synchronous step of the whole tile; o = this step's observations (LOSS)
    auto step = [&](const float (&o)[kVpt]) {
#pragma unroll
        for (int j = 0; j < kVpt; ++j) xv[par][j * kT + tid] = v[j];
        __syncthreads();
        float vl[kVpt];
#pragma unroll
        for (int j = 0; j < kVpt; ++j) vl[j] = xv[par][j * kT + tid + 1];
        par ^= 1;
#pragma unroll
        for (int j = 0; j < kVpt; ++j) {
            const float vlj = lead[j] ? vl[j] : v[j];
            if (KAHAN) {  // compensated displacement for long horizons (C3)
                const float y = __fmaf_rn(k.dt, v[j], -cmp[j]);
                const float tt2 = __fadd_rn(D[j], y);
                cmp[j] = __fsub_rn(__fsub_rn(tt2, D[j]), y);
                D[j] = tt2;
            } else {
                D[j] = __fmaf_rn(k.dt, v[j], D[j]);
            }
            fwd_step<D4>(s[j], v[j], vlj, lead[j], P[j], k);
        }
        orow += N;
        if (RECV) vrow += N;
#pragma unroll
        for (int j = 0; j < kVpt; ++j) {
            const float Pv = __fadd_rn(p0[j], D[j]);
            const float out = LOSS ? loss_term<LOSS - 1>(o[j], Pv, valid[j], lseg) : Pv;
            if (valid[j]) {
                __stcs(orow + j * kT, out);
                if (RECV) vrow[j * kT] = v[j];
            }
        }
    };
    auto checkpoint = [&](int t0) {  // (gap, speed) at step t0 > 0 + finiteness check
        cks += N;
        ckv += N;
#pragma unroll
        for (int j = 0; j < kVpt; ++j) {
            if (!valid[j]) continue;
            cks[j * kT] = s[j];
            ckv[j * kT] = v[j];
            if (!(isfinite(s[j]) && isfinite(v[j]) && isfinite(D[j])))
                report_nonfinite(a.status, t0, base + j * kT + tid);
        }
    };
    for (int seg = 0; seg < nfull; ++seg) {
        const int t0 = seg * KS;
        float ocur[KS][kVpt];
        if (LOSS) {
#pragma unroll
            for (int tt = 0; tt < KS; ++tt)
#pragma unroll
                for (int j = 0; j < kVpt; ++j) ocur[tt][j] = onx[tt][j];
            const int nxt = (seg + 1) * KS;  // the next segment observes rows nxt+1 ..
            if (nxt < steps) prefetch(nxt + 1, min(KS, steps - nxt));
        }
#pragma unroll
        for (int tt = 0; tt < KS; ++tt) {
            if (tt % CK == 0 && (tt > 0 || seg > 0)) checkpoint(t0 + tt);
            step(ocur[tt]);
        }
        if (LOSS) {
            lacc += (double)lseg;
            lseg = 0.f;
        }
    }
    if (tail > 0) {
#pragma unroll
        for (int tt = 0; tt < KS; ++tt) {
            if (tt < tail) {  // CTA-uniform predicate
                if (tt % CK == 0 && (tt > 0 || nfull > 0)) checkpoint(nfull * KS + tt);
                step(onx[tt]);
            }
        }
    }
#pragma unroll
    for (int j = 0; j < kVpt; ++j) {
        if (!valid[j]) continue;
        const int64_t i = base + j * kT + tid;
        if (!(isfinite(s[j]) && isfinite(v[j]) && isfinite(D[j])))
            report_nonfinite(a.status, steps, i);
        if (a.state_out) {
            a.state_out[i] = __fadd_rn(p0[j], D[j]);
            a.state_out[N + i] = v[j];
        }
    }
    if (LOSS) block_sum_to(lacc + (double)lseg, a.loss_partials);
}

// ------------------------------------------------------------------------------ NK3
// Per CTA (lane tile), segments of KS steps (compile-time, unrolled) from last to first:
//   recompute: reload the (gap, speed) checkpoint (prefetched one segment ahead) and re-run the
//              segment bit-identically; per step store the speed (leader reads) and the 24-byte
//              local-Jacobian record in shared memory; the segment's dL/dP rows are loaded into
//              registers meanwhile;
//   reverse:   sweep the segment backwards from the stored records; the follower -> leader
//              adjoint term F passes through shared memory (local id -> id + 1).
// Gradient accumulators stay in registers for the whole rollout; ADAM: per-vehicle Adam in the
// epilogue (idm_fit_step).
template <int KS>
constexpr size_t bwd_smem_of() {
    return (size_t)KS * (kCap * (sizeof(float4) + sizeof(float2)) + (kCap + 1) * sizeof(float));
}

template <bool D4, bool SHARED, bool ADAM, int KS>
#ifndef IDM_BWD_MINB
#define IDM_BWD_MINB 3  // CTAs per SM the backward is register-budgeted for (80 registers)
#endif
__global__ void __launch_bounds__(kT, (KS <= 4 ? IDM_BWD_MINB : 1)) bwd_kernel(BwdArgs a) {
    constexpr int HS = kCap + 1;
    extern __shared__ __align__(16) float4 smem4[];
    float4* hR1 = smem4;                                                  // [KS][kCap]
    float2* hR2 = reinterpret_cast<float2*>(hR1 + KS * kCap);             // [KS][kCap]
    float* hv = reinterpret_cast<float*>(hR2 + KS * kCap);                // [KS][kCap + 1]
    __shared__ float fx[2][kCap + 1];
    const int tid = threadIdx.x;
    const int64_t base = a.tile_start[blockIdx.x];
    const int n_loc = (int)(a.tile_start[blockIdx.x + 1] - base);
    const Consts k = a.k;
    const int64_t N = a.n;
    const int steps = a.steps;

    float ls[kVpt], lv[kVpt], lD[kVpt], s[kVpt], v[kVpt], cs[kVpt], cv[kVpt];
    bool lead[kVpt], valid[kVpt];
    VehP P[kVpt];
    VehB B[kVpt];
    GradAcc G[kVpt];
    const int nseg = (steps + KS - 1) / KS;
#pragma unroll
    for (int j = 0; j < kVpt; ++j) {
        const int id = j * kT + tid;
        const int64_t i = base + id;
        valid[j] = id < n_loc;
        ls[j] = 0.f;
        lv[j] = 0.f;
        G[j] = GradAcc{0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
        RawP r = dummy_raw();
        lead[j] = false;
        lD[j] = 0.f;
        cs[j] = 0.f;
        cv[j] = 0.f;
        if (valid[j]) {
            lead[j] = a.lead[i] != 0;
            r = load_raw(a.params, a.n_par, i);
            if (D4 && r.delta != 4.f)
                atomicMin(a.status, (unsigned long long)kBadDelta << 32 | (uint64_t)i);
            lD[j] = a.grad_traj[(int64_t)steps * N + i];   // lambda_D^K = dL/dP(K)
            cs[j] = a.ckpt_s[(int64_t)(nseg - 1) * N + i];  // checkpoint of the last segment
            cv[j] = a.ckpt_v[(int64_t)(nseg - 1) * N + i];
        }
        P[j] = make_vehp(r.a_max, r.a_pref, r.s_min, r.T, r.v_targ, r.delta);
        B[j] = make_vehb(r.a_max, r.a_pref, r.v_targ, r.delta);
    }
    if (tid == 0) { fx[0][0] = 0.f; fx[1][0] = 0.f; }  // never written again (slots id+1 >= 1)

    int par = 0;
    // one checkpoint segment [t0, t0 + len); FULL (len == KS) drops every step predicate
    auto run_segment = [&](const int seg, const int len, auto FULL) {
        constexpr bool kFull = decltype(FULL)::value;
        const int t0 = seg * KS;
        // ---- this segment's dL/dP rows into registers (consumed by the reverse sweep)
        float gr_[KS][kVpt];
        {
            const float* g = a.grad_traj + (int64_t)t0 * N + base + tid;
#pragma unroll
            for (int tt = 0; tt < KS; ++tt, g += N)
#pragma unroll
                for (int j = 0; j < kVpt; ++j)
                    gr_[tt][j] = (valid[j] && (kFull || tt < len)) ? __ldcs(g + j * kT) : 0.f;
        }
        // ---- recompute the segment from its checkpoint; prefetch the next one
#pragma unroll
        for (int j = 0; j < kVpt; ++j) {
            s[j] = cs[j];
            v[j] = cv[j];
        }
        if (seg > 0) {
            const int64_t off = (int64_t)(seg - 1) * N + base + tid;
#pragma unroll
            for (int j = 0; j < kVpt; ++j) {
                if (valid[j]) {
                    cs[j] = a.ckpt_s[off + j * kT];
                    cv[j] = a.ckpt_v[off + j * kT];
                }
            }
        }
#pragma unroll
        for (int tt = 0; tt < KS; ++tt) {
            if (kFull || tt < len) {  // CTA-uniform
                float* hvr = hv + tt * HS + tid;
#pragma unroll
                for (int j = 0; j < kVpt; ++j) hvr[j * kT] = v[j];
                __syncthreads();
#pragma unroll
                for (int j = 0; j < kVpt; ++j) {
                    const float vl = lead[j] ? hvr[j * kT + 1] : v[j];
                    Core c;
                    core<D4>(s[j], v[j], vl, lead[j], P[j], k, c);
                    float4 R1;
                    float2 R2;
                    jac_record<D4>(c, s[j], v[j], lead[j], P[j], B[j], k, R1, R2);
                    hR1[tt * kCap + j * kT + tid] = R1;
                    hR2[tt * kCap + j * kT + tid] = R2;
                    if (tt + 1 < (kFull ? KS : len)) advance(c, s[j], v[j], lead[j], k);
                }
            }
        }
        // ---- reverse sweep, t = t0 + len - 1 ... t0 (reads only this thread's records and
        //      the speed rows, all written before the last recompute barrier)
#pragma unroll
        for (int tt = KS - 1; tt >= 0; --tt) {
            if (kFull || tt < len) {  // CTA-uniform
                const float* hvr = hv + tt * HS + tid;
                float F[kVpt];
#pragma unroll
                for (int j = 0; j < kVpt; ++j) {
                    const float vj = hvr[j * kT];
                    const float vl = lead[j] ? hvr[j * kT + 1] : vj;
                    F[j] = bwd_from_record<D4>(hR1[tt * kCap + j * kT + tid],
                                               hR2[tt * kCap + j * kT + tid], vj, vl, P[j], B[j],
                                               k, ls[j], lv[j], lD[j], G[j]);
                }
#pragma unroll
                for (int j = 0; j < kVpt; ++j) fx[par][j * kT + tid + 1] = F[j];
                __syncthreads();
#pragma unroll
                for (int j = 0; j < kVpt; ++j) {
                    lv[j] += fx[par][j * kT + tid];  // F from the follower (id - 1)
                    lD[j] += gr_[tt][j];             // lambda_D^t = g^t + lambda_D^{t+1}
                }
                par ^= 1;
            }
        }
    };
    const int tail = steps - (nseg - 1) * KS;  // length of the last segment (1..KS)
    int seg = nseg - 1;
    if (tail < KS) run_segment(seg--, tail, std::false_type{});
    for (; seg >= 0; --seg) run_segment(seg, KS, std::true_type{});
    // dL/dp0_i = lambda_D - lambda_s_i + lambda_s_{follower}; dL/dv0 = lambda_v
#pragma unroll
    for (int j = 0; j < kVpt; ++j) fx[par][j * kT + tid + 1] = lead[j] ? ls[j] : 0.f;
    __syncthreads();
    float gp0[kVpt];
#pragma unroll
    for (int j = 0; j < kVpt; ++j)
        gp0[j] = lD[j] - (lead[j] ? ls[j] : 0.f) + fx[par][j * kT + tid];

    // parameter gradients from the factored accumulators
    float gr[kVpt][6];
#pragma unroll
    for (int j = 0; j < kVpt; ++j) {
#pragma unroll
        for (int q = 0; q < 6; ++q) gr[j][q] = 0.f;
        if (!valid[j]) continue;
        const int64_t i = base + j * kT + tid;
        const RawP r = load_raw(a.params, a.n_par, i);
        const float c = 0.5f / sqrtf(r.a_max * r.a_pref);
        gr[j][0] = G[j].S1 - c * (0.5f / r.a_max) * G[j].S2;             // a_max
        gr[j][1] = -c * (0.5f / r.a_pref) * G[j].S2;                      // a_pref
        gr[j][2] = G[j].S3;                                               // s_min
        gr[j][3] = G[j].S4;                                               // T_pref
        gr[j][4] = r.a_max * r.delta / r.v_targ * G[j].S5;               // v_targ
        gr[j][5] = -r.a_max * kLn2 * G[j].S6;                             // delta
        if (a.grad_state0) {
            a.grad_state0[i] = gp0[j];
            a.grad_state0[N + i] = lv[j];
        }
        if (!(isfinite(lv[j]) && isfinite(gp0[j]))) report_nonfinite(a.status, 0, i);
    }
    if (!SHARED) {
#pragma unroll
        for (int j = 0; j < kVpt; ++j) {
            if (!valid[j]) continue;
            const int64_t i = base + j * kT + tid;
#pragma unroll
            for (int q = 0; q < 6; ++q) {
                a.grad_params[q * N + i] = gr[j][q];
                // fused iteration: Adam on this vehicle's parameters right here (idm_fit_step)
                if (ADAM && ((a.adam.opt_mask >> q) & 1u)) adam_update(a.adam, q, q * N + i, gr[j][q]);
            }
        }
    } else {
        // fixed-order block reduction in fp64 -> partial[tile][6]
        __shared__ double red[kT / 32][6];
        double acc[6];
#pragma unroll
        for (int q = 0; q < 6; ++q) {
            double x = 0.0;
#pragma unroll
            for (int j = 0; j < kVpt; ++j) x += (double)gr[j][q];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
            acc[q] = x;
        }
        if ((tid & 31) == 0)
#pragma unroll
            for (int q = 0; q < 6; ++q) red[tid >> 5][q] = acc[q];
        __syncthreads();
        if (tid < 6) {
            double x = 0.0;
            for (int w = 0; w < kT / 32; ++w) x += red[w][tid];
            a.shared_partials[(int64_t)blockIdx.x * 6 + tid] = x;
        }
    }
}

// ------------------------------------------------------------------------------ NK2
// Eq. 4 over the flat [(steps+1) * N] arrays.  Fixed grid + fixed per-thread element order +
// fixed tree => bitwise deterministic partial sums.
template <bool VEC>
__global__ void __launch_bounds__(256) loss_kernel(LossArgs a) {
    double acc = 0.0;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const bool l1 = a.kind == 0;
    if (VEC) {
        const int64_t n4 = a.n_elem >> 2;
        const float4* P4 = reinterpret_cast<const float4*>(a.traj);
        const float4* O4 = reinterpret_cast<const float4*>(a.obs);
        float4* G4 = reinterpret_cast<float4*>(a.grad);
        const uchar4* M4 = reinterpret_cast<const uchar4*>(a.mask);
        for (int64_t e = t0; e < n4; e += stride) {
            float4 p = __ldcs(P4 + e), o = __ldcs(O4 + e);
            uchar4 m = a.mask ? __ldcs(M4 + e) : make_uchar4(1, 1, 1, 1);
            // an observation is used iff its mask is set and it is finite (NaN = missing)
            m.x = m.x && fabsf(o.x) <= 3.4e38f;
            m.y = m.y && fabsf(o.y) <= 3.4e38f;
            m.z = m.z && fabsf(o.z) <= 3.4e38f;
            m.w = m.w && fabsf(o.w) <= 3.4e38f;
            float r0 = o.x - p.x, r1 = o.y - p.y, r2 = o.z - p.z, r3 = o.w - p.w;
            float4 g;
            if (l1) {
                g.x = m.x ? -copysignf(r0 != 0.f, r0) : 0.f;
                g.y = m.y ? -copysignf(r1 != 0.f, r1) : 0.f;
                g.z = m.z ? -copysignf(r2 != 0.f, r2) : 0.f;
                g.w = m.w ? -copysignf(r3 != 0.f, r3) : 0.f;
                acc += (m.x ? (double)fabsf(r0) : 0.0) + (m.y ? (double)fabsf(r1) : 0.0) +
                       (m.z ? (double)fabsf(r2) : 0.0) + (m.w ? (double)fabsf(r3) : 0.0);
            } else {
                g.x = m.x ? -2.f * r0 : 0.f;
                g.y = m.y ? -2.f * r1 : 0.f;
                g.z = m.z ? -2.f * r2 : 0.f;
                g.w = m.w ? -2.f * r3 : 0.f;
                acc += (m.x ? (double)r0 * r0 : 0.0) + (m.y ? (double)r1 * r1 : 0.0) +
                       (m.z ? (double)r2 * r2 : 0.0) + (m.w ? (double)r3 * r3 : 0.0);
            }
            __stcs(G4 + e, g);
        }
        // tail (n_elem % 4) handled by the first threads
        for (int64_t e = (n4 << 2) + t0; e < a.n_elem; e += stride) {
            bool m = (a.mask ? a.mask[e] != 0 : true) && fabsf(a.obs[e]) <= 3.4e38f;
            float r = a.obs[e] - a.traj[e];
            float g = l1 ? -copysignf(r != 0.f, r) : -2.f * r;
            a.grad[e] = m ? g : 0.f;
            if (m) acc += l1 ? (double)fabsf(r) : (double)r * r;
        }
    } else {
        for (int64_t e = t0; e < a.n_elem; e += stride) {
            bool m = (a.mask ? a.mask[e] != 0 : true) && fabsf(a.obs[e]) <= 3.4e38f;
            float r = a.obs[e] - a.traj[e];
            float g = l1 ? -copysignf(r != 0.f, r) : -2.f * r;
            a.grad[e] = m ? g : 0.f;
            if (m) acc += l1 ? (double)fabsf(r) : (double)r * r;
        }
    }
    // block reduction (fixed tree)
    __shared__ double red[8];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        double x = 0.0;
        for (int w = 0; w < 8; ++w) x += red[w];
        a.partials[blockIdx.x] = x;
    }
}

// ------------------------------------------------------------------------------ NK4
// Sums `n` rows of `width` fp64 partials in fixed order; out_f (nullable) gets a float copy.
__global__ void reduce_kernel(const double* __restrict__ partials, int64_t n, int width,
                              double* __restrict__ out, float* __restrict__ out_f) {
    __shared__ double red[256];
    for (int c = 0; c < width; ++c) {
        double x = 0.0;
        for (int64_t r = threadIdx.x; r < n; r += blockDim.x) x += partials[r * width + c];
        red[threadIdx.x] = x;
        __syncthreads();
        for (int s = blockDim.x / 2; s > 0; s >>= 1) {
            if (threadIdx.x < s) red[threadIdx.x] += red[threadIdx.x + s];
            __syncthreads();
        }
        if (threadIdx.x == 0) {
            if (out) out[c] = red[0];
            if (out_f) out_f[c] = (float)red[0];
        }
        __syncthreads();
    }
}

// ------------------------------------------------------------------------------ NK5
__global__ void __launch_bounds__(256) adam_kernel(AdamArgs a) {
    const int64_t m = 6 * a.n_par;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < m;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int q = (int)(e / a.n_par);
        if ((a.opt_mask >> q) & 1u) adam_update(a, q, e, a.grad[e]);
    }
}

// ------------------------------------------------------------------------------ launchers
cudaError_t launch_validate(const ValidateArgs& a, cudaStream_t st) {
    validate_kernel<<<148 * 4, 256, 0, st>>>(a);
    return cudaGetLastError();
}

bool ckpt_supported(int k) { return k == 2 || k == 4 || k == 8; }

size_t bwd_smem_bytes(int ckpt_every) {
    return ckpt_every == 2 ? bwd_smem_of<2>() : ckpt_every == 8 ? bwd_smem_of<8>()
                                                                : bwd_smem_of<4>();
}

template <bool D4, bool KH, int KS>
static void launch_fwd_k(const FwdArgs& a, int ntiles, const FwdVariant& var, cudaStream_t st) {
    dim3 g(ntiles), b(kT);
    if (var.loss == 1) fwd_kernel<D4, KH, false, 1, KS><<<g, b, 0, st>>>(a);
    else if (var.loss == 2) fwd_kernel<D4, KH, false, 2, KS><<<g, b, 0, st>>>(a);
    else if (var.rec_v) fwd_kernel<D4, KH, true, 0, KS><<<g, b, 0, st>>>(a);
    else fwd_kernel<D4, KH, false, 0, KS><<<g, b, 0, st>>>(a);
}

template <bool D4, bool KH>
static void launch_fwd_dk(const FwdArgs& a, int ntiles, const FwdVariant& var, cudaStream_t st) {
    switch (a.ckpt_every) {
        case 2: launch_fwd_k<D4, KH, 2>(a, ntiles, var, st); break;
        case 8: launch_fwd_k<D4, KH, 8>(a, ntiles, var, st); break;
        default: launch_fwd_k<D4, KH, 4>(a, ntiles, var, st); break;
    }
}

cudaError_t launch_fwd(const FwdArgs& a, int ntiles, const FwdVariant& var, cudaStream_t st) {
    if (!ckpt_supported(a.ckpt_every)) return cudaErrorInvalidValue;
    if (var.delta4) {
        if (var.kahan) launch_fwd_dk<true, true>(a, ntiles, var, st);
        else launch_fwd_dk<true, false>(a, ntiles, var, st);
    } else {
        if (var.kahan) launch_fwd_dk<false, true>(a, ntiles, var, st);
        else launch_fwd_dk<false, false>(a, ntiles, var, st);
    }
    return cudaGetLastError();
}

template <int KS>
static cudaError_t configure_k() {
    cudaError_t e = cudaSuccess;
    const int mb = (int)bwd_smem_of<KS>();
#define IDM_CFG(D4, SH, AD)                                                                 \
    if (e == cudaSuccess)                                                                  \
        e = cudaFuncSetAttribute(bwd_kernel<D4, SH, AD, KS>,                               \
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, mb);
    IDM_CFG(true, true, false) IDM_CFG(true, false, false) IDM_CFG(false, true, false)
    IDM_CFG(false, false, false) IDM_CFG(true, false, true) IDM_CFG(false, false, true)
#undef IDM_CFG
    return e;
}

cudaError_t kernels_configure(int ckpt_every) {
    switch (ckpt_every) {
        case 2: return configure_k<2>();
        case 4: return configure_k<4>();
        case 8: return configure_k<8>();
        default: return cudaErrorInvalidValue;
    }
}

template <int KS>
static void launch_bwd_k(const BwdArgs& a, int ntiles, bool delta4, bool shared, bool adam,
                         cudaStream_t st) {
    const size_t smem = bwd_smem_of<KS>();
    dim3 g(ntiles), b(kT);
    if (delta4) {
        if (shared) bwd_kernel<true, true, false, KS><<<g, b, smem, st>>>(a);
        else if (adam) bwd_kernel<true, false, true, KS><<<g, b, smem, st>>>(a);
        else bwd_kernel<true, false, false, KS><<<g, b, smem, st>>>(a);
    } else {
        if (shared) bwd_kernel<false, true, false, KS><<<g, b, smem, st>>>(a);
        else if (adam) bwd_kernel<false, false, true, KS><<<g, b, smem, st>>>(a);
        else bwd_kernel<false, false, false, KS><<<g, b, smem, st>>>(a);
    }
}

cudaError_t launch_bwd(const BwdArgs& a, int ntiles, bool delta4, bool shared, bool adam,
                       cudaStream_t st) {
    switch (a.ckpt_every) {
        case 2: launch_bwd_k<2>(a, ntiles, delta4, shared, adam, st); break;
        case 4: launch_bwd_k<4>(a, ntiles, delta4, shared, adam, st); break;
        case 8: launch_bwd_k<8>(a, ntiles, delta4, shared, adam, st); break;
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

cudaError_t launch_loss(const LossArgs& a, int nblocks, cudaStream_t st) {
    bool vec = ((uintptr_t)a.traj % 16 == 0) && ((uintptr_t)a.obs % 16 == 0) &&
               ((uintptr_t)a.grad % 16 == 0) && (a.mask == nullptr || (uintptr_t)a.mask % 4 == 0);
    if (vec)
        loss_kernel<true><<<nblocks, 256, 0, st>>>(a);
    else
        loss_kernel<false><<<nblocks, 256, 0, st>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_reduce(const double* partials, int64_t n, int width, double* out,
                          float* out_f, cudaStream_t st) {
    reduce_kernel<<<1, 256, 0, st>>>(partials, n, width, out, out_f);
    return cudaGetLastError();
}

cudaError_t launch_adam(const AdamArgs& a, cudaStream_t st) {
    int64_t m = 6 * a.n_par;
    int64_t blocks = (m + 255) / 256;
    if (blocks > 148 * 16) blocks = 148 * 16;
    adam_kernel<<<(int)blocks, 256, 0, st>>>(a);
    return cudaGetLastError();
}

}  // namespace idm
