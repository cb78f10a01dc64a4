// idm_vl.cu -- virtual-leader mode.
//
// The paper fits each trajectory on its own: the leader terms of vehicle i at step k are free
// variables (Delta p_k, Delta v_k), initialised to 10 and 0 and optimised with Adam alongside
// the five IDM parameters.  Every vehicle is independent, so a CTA is 256 threads, thread t
// owning the adjacent vehicles 2t, 2t + 1 as one float2 pair (packed f32x2 arithmetic, as the
// lane kernels), with no exchange and no barrier; the per-step leaf rows are loaded a segment
// at a time into registers.  The mode is HBM-bound (per vehicle-step: dp, dv in the forward;
// dp, dv, dL/dP in and the two leaf gradients out in the backward; Adam over 2 N K leaves).
//
//   vl_fwd_kernel    K steps per vehicle from (p0, v0); records P (or fused Eq. 4: dL/dP)
//   vl_bwd_kernel    per segment: recompute speeds from the checkpoint, reverse sweep writing
//                    dL/d(dp_k), dL/d(dv_k); parameter gradients (+ Adam epilogue when fused)
//   adam_free_kernel Adam over the unconstrained leaf lists (PAPER.md:208 gives them no box)
#include <climits>
#include <cstdint>
#include <cuda_runtime.h>

#include "idm_device.cuh"
#include "idm_internal.h"

namespace idm {

namespace {
constexpr int kVT = 256;  // threads per CTA
constexpr int kVV = 2;    // vehicles per thread (one adjacent pair)
constexpr int kVB = kVT * kVV;

__device__ __forceinline__ void vl_block_sum(double x, double* out) {
    __shared__ double red[kVT / 32];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = x;
    __syncthreads();
    if (threadIdx.x == 0) {
        double y = 0.0;
        for (int w = 0; w < kVT / 32; ++w) y += red[w];
        out[blockIdx.x] = y;
    }
}

__device__ __forceinline__ void vl_params(const float* prm, int64_t n_par, int64_t i, float* r) {
    const int64_t j = n_par == 1 ? 0 : i;
#pragma unroll
    for (int q = 0; q < 6; ++q) r[q] = prm[q * n_par + j];
}

// predicated pair access at p (vehicles i0, i0 + 1)
__device__ __forceinline__ float2 ld_pair(const float* p, bool on0, bool on1, float dflt) {
    return make_float2(ld_cs_if(p, on0, dflt), ld_cs_if(p + 1, on1, dflt));
}
__device__ __forceinline__ void st_pair(float* p, bool on0, bool on1, float2 x) {
    st_cs_if(p, on0, x.x);
    st_cs_if(p + 1, on1, x.y);
}
}  // namespace

// ------------------------------------------------------------------------------ forward
template <bool D4, int LOSS, int KS>
__global__ void __launch_bounds__(kVT) vl_fwd_kernel(VlArgs a) {
    const int tid = threadIdx.x;
    const int64_t N = a.n;
    const int steps = a.steps;
    const int64_t i0 = (int64_t)blockIdx.x * kVB + 2 * tid;
    const bool val0 = i0 < N, val1 = i0 + 1 < N;
    const float qnan = __int_as_float(0x7fc00000);
    float pj[2] = {0.f, 0.f}, vj[2] = {0.f, 0.f};
    VehP Pj[2];
#pragma unroll
    for (int j = 0; j < 2; ++j) {
        const int64_t i = i0 + j;
        float r[6] = {1.f, 1.f, 1.f, 1.f, 1.f, 4.f};
        if (i < N) {
            pj[j] = a.pos0[i];
            vj[j] = a.vel0[i];
            vl_params(a.params, a.n_par, i, r);
            if (D4 && r[5] != 4.f)
                atomicMin(a.status, (unsigned long long)kBadDelta << 32 | (uint64_t)i);
        }
        Pj[j] = make_vehp(r[0], r[1], r[2], r[3], r[4], r[5]);
    }
    const VehPT<float2> P = pack(Pj[0], Pj[1]);
    const float2 p0 = make_float2(pj[0], pj[1]);
    float2 v = make_float2(vj[0], vj[1]), D = f2(0.f);
    const Consts k = a.k;
    // LOSS = 3: only the history for a backward that derives Eq. 4 itself -- speed and
    // displacement checkpoints, no per-step row
    constexpr bool ROWS = LOSS != 3;
    constexpr bool OBSV = LOSS == 1 || LOSS == 2;
    float* orow = ROWS ? (LOSS ? a.grad_traj : a.traj) + i0 : nullptr;
    float* vrow = (!LOSS && a.vel_traj) ? a.vel_traj + i0 : nullptr;
    float* ckv = a.ckpt_v + i0;
    float* ckd = LOSS == 3 ? a.ckpt_d + i0 : nullptr;
    const float* dpr = a.vl_dp + i0;
    const float* dvr = a.vl_dv + i0;
    const float* obs = OBSV ? a.obs + i0 : nullptr;
    float2 lseg = f2(0.f);
    double lacc = 0.0;
    if (ROWS)
        st_pair(orow, val0, val1,
                OBSV ? loss_term<(LOSS == 2 ? 1 : 0)>(ld_pair(obs, val0, val1, qnan), p0, lseg)
                     : p0);
    if (vrow) st_pair(vrow, val0, val1, v);
    st_pair(ckv, val0, val1, v);
    if (LOSS == 3) st_pair(ckd, val0, val1, D);
    int bad0 = INT_MAX, bad1 = INT_MAX;  // first non-finite checkpoint (reported at the end)
    const int nseg = (steps + KS - 1) / KS;
    for (int seg = 0; seg < nseg; ++seg) {
        const int t0 = seg * KS;
        const int len = min(KS, steps - t0);
        if (seg > 0) {
            ckv += N;
            st_pair(ckv, val0, val1, v);
            if (LOSS == 3) {
                ckd += N;
                st_pair(ckd, val0, val1, D);
            }
            bad0 = (!(isfinite(v.x) && isfinite(D.x)) && bad0 == INT_MAX) ? t0 : bad0;
            bad1 = (!(isfinite(v.y) && isfinite(D.y)) && bad1 == INT_MAX) ? t0 : bad1;
        }
        // this segment's leaf rows (and observation rows) into registers
        float2 dp[KS], dv[KS], ob[OBSV ? KS : 1];
#pragma unroll
        for (int tt = 0; tt < KS; ++tt) {
            const bool on = tt < len;
            const int64_t off = (int64_t)(t0 + (on ? tt : 0)) * N;
            dp[tt] = ld_pair(dpr + off, on && val0, on && val1, 10.f);
            dv[tt] = ld_pair(dvr + off, on && val0, on && val1, 0.f);
            if (OBSV) ob[tt] = ld_pair(obs + off + N, on && val0, on && val1, qnan);
        }
#pragma unroll
        for (int tt = 0; tt < KS; ++tt) {
            if (tt < len) {
                if (ROWS) orow += N;
                if (vrow) vrow += N;
                D = vfma(v, k.dt, D);
                CoreT<float2> c;
                core_dv<D4>(dp[tt], v, dv[tt], P, k, c);
                float2 sdummy = f2(0.f);
                advance(c, sdummy, v, k);
                const float2 Pv = vadd(p0, D);
                if (ROWS)
                    st_pair(orow, val0, val1,
                            OBSV ? loss_term<(LOSS == 2 ? 1 : 0)>(ob[tt], Pv, lseg) : Pv);
                if (vrow) st_pair(vrow, val0, val1, v);
            }
        }
        if (OBSV) {
            lacc += (double)lseg.x + (double)lseg.y;
            lseg = f2(0.f);
        }
    }
    bad0 = (!(isfinite(v.x) && isfinite(D.x)) && bad0 == INT_MAX) ? steps : bad0;
    bad1 = (!(isfinite(v.y) && isfinite(D.y)) && bad1 == INT_MAX) ? steps : bad1;
    const float2 Pend = vadd(p0, D);
    const int badj[2] = {bad0, bad1};
    const float pend[2] = {Pend.x, Pend.y}, vend[2] = {v.x, v.y};
#pragma unroll
    for (int j = 0; j < 2; ++j) {
        const int64_t i = i0 + j;
        if (i >= N) continue;
        if (badj[j] != INT_MAX)
            atomicMin(a.status,
                      (unsigned long long)(unsigned)badj[j] << 32 | (uint64_t)(uint32_t)i);
        if (a.state_out) {
            a.state_out[i] = pend[j];
            a.state_out[N + i] = vend[j];
        }
    }
    if (OBSV) vl_block_sum(lacc + (double)lseg.x + (double)lseg.y, a.loss_partials);
}

// ------------------------------------------------------------------------------ backward
// OK = -1: dL/dP rows from grad_traj; 0 / 1 (fused iteration after the history-only forward):
// the Eq. 4 terms (L1 / L2) and dL/dP from obs and the positions rebuilt from the displacement
// checkpoints (the forward's own recurrence, bitwise), the loss per block to loss_partials
template <bool D4, bool ADAM, int KS, int OK>
__global__ void __launch_bounds__(kVT, 2) vl_bwd_kernel(VlArgs a) {
    const int tid = threadIdx.x;
    const int64_t N = a.n;
    const int steps = a.steps;
    const int64_t i0 = (int64_t)blockIdx.x * kVB + 2 * tid;
    const bool val0 = i0 < N, val1 = i0 + 1 < N;
    const Consts k = a.k;
    const int64_t KN = (int64_t)a.max_steps * N;  // leaf plane stride
    const float qnan = __int_as_float(0x7fc00000);
    float ldj[2] = {0.f, 0.f}, pj[2] = {0.f, 0.f};
    VehP Pj[2];
    VehB Bj[2];
#pragma unroll
    for (int j = 0; j < 2; ++j) {
        const int64_t i = i0 + j;
        float r[6] = {1.f, 1.f, 1.f, 1.f, 1.f, 4.f};
        if (i < N) {
            vl_params(a.params, a.n_par, i, r);
            if (OK < 0) ldj[j] = a.grad_traj[(int64_t)steps * N + i];  // lambda_P^K = dL/dP(K)
            else pj[j] = a.pos0[i];
        }
        Pj[j] = make_vehp(r[0], r[1], r[2], r[3], r[4], r[5]);
        Bj[j] = make_vehb(r[0], r[1], r[4], r[5]);
    }
    const VehPT<float2> P = pack(Pj[0], Pj[1]);
    const VehBT<float2> B = pack(Bj[0], Bj[1]);
    float2 lv = f2(0.f), lD = make_float2(ldj[0], ldj[1]);
    const float2 p0 = make_float2(pj[0], pj[1]);
    double lacc = 0.0;
    GradAccT<float2> G = {f2(0.f), f2(0.f), f2(0.f), f2(0.f), f2(0.f), f2(0.f)};
    const int nseg = (steps + KS - 1) / KS;
    for (int seg = nseg - 1; seg >= 0; --seg) {
        const int t0 = seg * KS;
        const int len = min(KS, steps - t0);
        float2 dp[KS], dv[KS], gr[KS], vt[KS];
        // ADAM (fused iteration): the leaves' Adam moments of this segment, updated in place
        float2 am[ADAM ? KS : 1][2], av[ADAM ? KS : 1][2];
#pragma unroll
        for (int tt = 0; tt < KS; ++tt) {
            const bool on = tt < len;
            const bool o0 = on && val0, o1 = on && val1;
            const int64_t off = (int64_t)(t0 + (on ? tt : 0)) * N + i0;
            dp[tt] = ld_pair(a.vl_dp + off, o0, o1, 10.f);
            dv[tt] = ld_pair(a.vl_dv + off, o0, o1, 0.f);
            if (OK < 0) gr[tt] = ld_pair(a.grad_traj + off, o0, o1, 0.f);
            else gr[tt] = ld_pair(a.obs + off, o0, o1, qnan);  // absent vehicles: missing
            if (ADAM) {
#pragma unroll
                for (int pl = 0; pl < 2; ++pl) {
                    am[tt][pl] = ld_pair(a.vl_adam_m + pl * KN + off, o0, o1, 0.f);
                    av[tt][pl] = ld_pair(a.vl_adam_v + pl * KN + off, o0, o1, 0.f);
                }
            }
        }
        // recompute the segment's speeds from its checkpoint (bit-identical to the forward)
        vt[0] = ld_pair(a.ckpt_v + (int64_t)seg * N + i0, val0, val1, 0.f);
#pragma unroll
        for (int tt = 0; tt + 1 < KS; ++tt) {
            if (tt + 1 < len) {
                CoreT<float2> c;
                core_dv<D4>(dp[tt], vt[tt], dv[tt], P, k, c);
                float2 sdummy = f2(0.f), vn = vt[tt];
                advance(c, sdummy, vn, k);
                vt[tt + 1] = vn;
            }
        }
        if (OK >= 0) {  // positions by the forward's recurrence, then Eq. 4 and dL/dP
            float2 D = ld_pair(a.ckpt_d + (int64_t)seg * N + i0, val0, val1, 0.f);
            float2 lsum = f2(0.f);
#pragma unroll
            for (int tt = 0; tt < KS; ++tt) {
                if (tt < len) {
                    gr[tt] = loss_term<(OK > 0 ? 1 : 0)>(gr[tt], vadd(p0, D), lsum);
                    D = vfma(vt[tt], k.dt, D);
                }
            }
            if (seg == nseg - 1)  // lambda_P^K = dL/dP(K), the rollout's last row
                lD = loss_term<(OK > 0 ? 1 : 0)>(
                    ld_pair(a.obs + (int64_t)steps * N + i0, val0, val1, qnan), vadd(p0, D),
                    lsum);
            lacc += (double)lsum.x + (double)lsum.y;
        }
        // reverse sweep
#pragma unroll
        for (int tt = KS - 1; tt >= 0; --tt) {
            if (tt < len) {
                const int64_t off = (int64_t)(t0 + tt) * N + i0;
                CoreT<float2> c;
                core_dv<D4>(dp[tt], vt[tt], dv[tt], P, k, c);
                float2 gdp, gdv;
                bwd_vl<D4>(c, dp[tt], vt[tt], P, B, k, lv, lD, G, gdp, gdv);
                lD = vadd(lD, gr[tt]);  // lambda_P^t = g^t + lambda_P^{t+1}
                if (ADAM) {  // Adam on the two leaves of step t, in place (no box)
                    const float gg[2][2] = {{gdp.x, gdp.y}, {gdv.x, gdv.y}};
                    const float x0[2][2] = {{dp[tt].x, dp[tt].y}, {dv[tt].x, dv[tt].y}};
                    float* xs[2] = {const_cast<float*>(a.vl_dp), const_cast<float*>(a.vl_dv)};
#pragma unroll
                    for (int pl = 0; pl < 2; ++pl) {
                        float mm[2] = {am[tt][pl].x, am[tt][pl].y};
                        float vv[2] = {av[tt][pl].x, av[tt][pl].y};
                        float xn[2];
#pragma unroll
                        for (int j = 0; j < 2; ++j)
                            xn[j] = leaf_adam(x0[pl][j], gg[pl][j], mm[j], vv[j],
                                              a.adam.step_size, a.adam.sqrt_bc2, a.adam.beta1,
                                              a.adam.beta2, a.adam.eps);
                        st_pair(a.vl_adam_m + pl * KN + off, val0, val1, make_float2(mm[0], mm[1]));
                        st_pair(a.vl_adam_v + pl * KN + off, val0, val1, make_float2(vv[0], vv[1]));
                        st_pair(xs[pl] + off, val0, val1, make_float2(xn[0], xn[1]));
                    }
                } else {
                    st_pair(a.vl_grad + off, val0, val1, gdp);
                    st_pair(a.vl_grad + KN + off, val0, val1, gdv);
                }
            }
        }
    }
    const float Sj[6][2] = {{G.S1.x, G.S1.y}, {G.S2.x, G.S2.y}, {G.S3.x, G.S3.y},
                            {G.S4.x, G.S4.y}, {G.S5.x, G.S5.y}, {G.S6.x, G.S6.y}};
    const float lvj[2] = {lv.x, lv.y}, lDj[2] = {lD.x, lD.y};
#pragma unroll
    for (int j = 0; j < 2; ++j) {
        const int64_t i = i0 + j;
        if (i >= N) continue;
        float r[6];
        vl_params(a.params, a.n_par, i, r);
        const float Sv[6] = {Sj[0][j], Sj[1][j], Sj[2][j], Sj[3][j], Sj[4][j], Sj[5][j]};
        float gr6[6];
        param_grads(r, Sv, gr6);
        if (ADAM && !((a.adam.opt_mask >> 5) & 1u)) gr6[5] = 0.f;  // delta frozen: not reported
        if (a.grad_state0) {
            a.grad_state0[i] = lDj[j];  // dL/dp0: position enters every later P
            a.grad_state0[N + i] = lvj[j];
        }
        if (!(isfinite(lvj[j]) && isfinite(lDj[j])))
            atomicMin(a.status, (unsigned long long)0 << 32 | (uint64_t)(uint32_t)i);
        int bq = -1;  // first optimised parameter with a non-finite gradient
#pragma unroll
        for (int q = 0; q < 6; ++q) {
            a.grad_params[q * N + i] = gr6[q];
            if (ADAM && ((a.adam.opt_mask >> q) & 1u)) {
                if (bq < 0 && !isfinite(gr6[q])) bq = q;
                adam_update(a.adam, q, q * N + i, gr6[q]);
            }
        }
        if (ADAM && bq >= 0) report_bad_grad(a.status, bq * N + i);
    }
    if (OK >= 0) vl_block_sum(lacc, a.loss_partials);  // this block's Eq. 4 loss
}

// Adam over unconstrained leaves (same update as adam_update, no box).
__global__ void __launch_bounds__(256) adam_free_kernel(float* x, const float* g, float* m,
                                                         float* v, int64_t n, float step_size,
                                                         float sqrt_bc2, float b1, float b2,
                                                         float eps) {
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n;
         e += (int64_t)gridDim.x * blockDim.x) {
        float mm = m[e], vv = v[e];
        x[e] = leaf_adam(x[e], g[e], mm, vv, step_size, sqrt_bc2, b1, b2, eps);
        m[e] = mm;
        v[e] = vv;
    }
}

// ------------------------------------------------------------------------------ launchers
int64_t vl_blocks(int64_t n) { return (n + kVB - 1) / kVB; }

template <bool D4>
static void vl_fwd_d(const VlArgs& a, int loss, cudaStream_t st) {
    dim3 g((unsigned)vl_blocks(a.n)), b(kVT);
    if (loss == 1) vl_fwd_kernel<D4, 1, 4><<<g, b, 0, st>>>(a);
    else if (loss == 2) vl_fwd_kernel<D4, 2, 4><<<g, b, 0, st>>>(a);
    else if (loss == 3) vl_fwd_kernel<D4, 3, 4><<<g, b, 0, st>>>(a);
    else vl_fwd_kernel<D4, 0, 4><<<g, b, 0, st>>>(a);
}

cudaError_t launch_vl_fwd(const VlArgs& a, bool delta4, int loss, cudaStream_t st) {
    if (a.ckpt_every != 4) return cudaErrorInvalidValue;
    if (delta4) vl_fwd_d<true>(a, loss, st);
    else vl_fwd_d<false>(a, loss, st);
    return cudaGetLastError();
}

template <bool D4>
static void vl_bwd_d(const VlArgs& a, bool adam, int obs_kind, cudaStream_t st) {
    dim3 g((unsigned)vl_blocks(a.n)), b(kVT);
    if (!adam) vl_bwd_kernel<D4, false, 4, -1><<<g, b, 0, st>>>(a);
    else if (obs_kind == 0) vl_bwd_kernel<D4, true, 4, 0><<<g, b, 0, st>>>(a);
    else if (obs_kind == 1) vl_bwd_kernel<D4, true, 4, 1><<<g, b, 0, st>>>(a);
    else vl_bwd_kernel<D4, true, 4, -1><<<g, b, 0, st>>>(a);
}

cudaError_t launch_vl_bwd(const VlArgs& a, bool delta4, bool adam, cudaStream_t st,
                          int obs_kind) {
    if (a.ckpt_every != 4) return cudaErrorInvalidValue;
    if (obs_kind >= 0 && !adam) return cudaErrorInvalidValue;  // the fused iteration only
    if (delta4) vl_bwd_d<true>(a, adam, obs_kind, st);
    else vl_bwd_d<false>(a, adam, obs_kind, st);
    return cudaGetLastError();
}

cudaError_t launch_adam_free(float* x, const float* g, float* m, float* v, int64_t n,
                             const AdamArgs& hp, cudaStream_t st) {
    int64_t blocks = (n + 255) / 256;
    if (blocks > 148 * 16) blocks = 148 * 16;
    adam_free_kernel<<<(int)blocks, 256, 0, st>>>(x, g, m, v, n, hp.step_size, hp.sqrt_bc2,
                                                  hp.beta1, hp.beta2, hp.eps);
    return cudaGetLastError();
}

}  // namespace idm
