// idm_vl.cu -- virtual-leader mode.
//
// The paper fits each trajectory on its own: the leader terms of vehicle i at step k are free
// variables (Delta p_k, Delta v_k), initialised to 10 and 0 and optimised with Adam alongside
// the five IDM parameters.  Every vehicle is independent, so a CTA is 256 threads x 2 vehicles
// with no exchange and no barrier; the per-step leaf rows are prefetched a segment ahead into
// registers.  The mode is HBM-bound (per vehicle-step: dp, dv in the forward; dp, dv, dL/dP in
// and the two leaf gradients out in the backward; Adam over 2 N K leaves).
//
//   vl_fwd_kernel    K steps per vehicle from (p0, v0); records P (or fused Eq. 4: dL/dP)
//   vl_bwd_kernel    per segment: recompute speeds from the checkpoint, reverse sweep writing
//                    dL/d(dp_k), dL/d(dv_k); parameter gradients (+ Adam epilogue when fused)
//   adam_free_kernel Adam over the unconstrained leaf lists (PAPER.md:208 gives them no box)
#include <cstdint>
#include <cuda_runtime.h>

#include "idm_device.cuh"
#include "idm_internal.h"

namespace idm {

namespace {
constexpr int kVT = 256;  // threads per CTA
constexpr int kVV = 2;    // vehicles per thread
constexpr int kVB = kVT * kVV;

__device__ __forceinline__ float vl_loss_term(int kind, float o, float P, bool valid,
                                              float& acc) {
    const float r = o - P;
    const bool ok = valid && fabsf(o) <= 3.4e38f;
    if (kind == 0) {
        acc += ok ? fabsf(r) : 0.f;
        const float sg = r > 0.f ? -1.f : (r < 0.f ? 1.f : 0.f);
        return ok ? sg : 0.f;
    }
    acc = ok ? fmaf(r, r, acc) : acc;
    return ok ? -2.f * r : 0.f;
}

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
}  // namespace

// ------------------------------------------------------------------------------ forward
template <bool D4, int LOSS, int KS>
__global__ void __launch_bounds__(kVT) vl_fwd_kernel(VlArgs a) {
    const int tid = threadIdx.x;
    const int64_t N = a.n;
    const int steps = a.steps;
    const int64_t base = (int64_t)blockIdx.x * kVB + tid;
    float v[kVV], D[kVV], p0[kVV];
    bool valid[kVV];
    VehP P[kVV];
#pragma unroll
    for (int j = 0; j < kVV; ++j) {
        const int64_t i = base + j * kVT;
        valid[j] = i < N;
        float r[6] = {1.f, 1.f, 1.f, 1.f, 1.f, 4.f};
        p0[j] = 0.f;
        v[j] = 0.f;
        if (valid[j]) {
            p0[j] = a.pos0[i];
            v[j] = a.vel0[i];
            vl_params(a.params, a.n_par, i, r);
            if (D4 && r[5] != 4.f)
                atomicMin(a.status, (unsigned long long)kBadDelta << 32 | (uint64_t)i);
        }
        D[j] = 0.f;
        P[j] = make_vehp(r[0], r[1], r[2], r[3], r[4], r[5]);
    }
    const Consts k = a.k;
    float* orow = (LOSS ? a.grad_traj : a.traj) + base;
    float* vrow = (!LOSS && a.vel_traj) ? a.vel_traj + base : nullptr;
    float* ckv = a.ckpt_v + base;
    const float* dpr = a.vl_dp + base;
    const float* dvr = a.vl_dv + base;
    const float* obs = LOSS ? a.obs + base : nullptr;
    float lseg = 0.f;
    double lacc = 0.0;
#pragma unroll
    for (int j = 0; j < kVV; ++j) {
        if (!valid[j]) continue;
        __stcs(orow + j * kVT,
               LOSS ? vl_loss_term(LOSS - 1, obs[j * kVT], p0[j], true, lseg) : p0[j]);
        if (vrow) vrow[j * kVT] = v[j];
        ckv[j * kVT] = v[j];
    }
    const int nseg = (steps + KS - 1) / KS;
    for (int seg = 0; seg < nseg; ++seg) {
        const int t0 = seg * KS;
        const int len = min(KS, steps - t0);
        if (seg > 0) {
            ckv += N;
#pragma unroll
            for (int j = 0; j < kVV; ++j) {
                if (!valid[j]) continue;
                ckv[j * kVT] = v[j];
                if (!(isfinite(v[j]) && isfinite(D[j])))
                    atomicMin(a.status, (unsigned long long)(unsigned)t0 << 32 |
                                            (uint64_t)(uint32_t)(base + j * kVT));
            }
        }
        // this segment's leaf rows (and observation rows) into registers
        float dp[KS][kVV], dv[KS][kVV], ob[LOSS ? KS : 1][kVV];
#pragma unroll
        for (int tt = 0; tt < KS; ++tt)
#pragma unroll
            for (int j = 0; j < kVV; ++j) {
                const bool ok = valid[j] && tt < len;
                const int64_t off = (int64_t)(t0 + tt) * N + j * kVT;
                dp[tt][j] = ok ? __ldcs(dpr + off) : 10.f;
                dv[tt][j] = ok ? __ldcs(dvr + off) : 0.f;
                if (LOSS) ob[tt][j] = ok ? __ldcs(obs + off + N) : 0.f;
            }
#pragma unroll
        for (int tt = 0; tt < KS; ++tt) {
            if (tt < len) {
                orow += N;
                if (vrow) vrow += N;
#pragma unroll
                for (int j = 0; j < kVV; ++j) {
                    D[j] = __fmaf_rn(k.dt, v[j], D[j]);
                    Core c;
                    core_dv<D4>(dp[tt][j], v[j], dv[tt][j], 1.f, P[j], k, c);
                    float sdummy = 0.f;
                    advance(c, sdummy, v[j], k);
                    const float Pv = __fadd_rn(p0[j], D[j]);
                    const float out =
                        LOSS ? vl_loss_term(LOSS - 1, ob[tt][j], Pv, valid[j], lseg) : Pv;
                    if (valid[j]) {
                        __stcs(orow + j * kVT, out);
                        if (vrow) vrow[j * kVT] = v[j];
                    }
                }
            }
        }
        if (LOSS) {
            lacc += (double)lseg;
            lseg = 0.f;
        }
    }
#pragma unroll
    for (int j = 0; j < kVV; ++j) {
        if (!valid[j]) continue;
        const int64_t i = base + j * kVT;
        if (!(isfinite(v[j]) && isfinite(D[j])))
            atomicMin(a.status, (unsigned long long)(unsigned)steps << 32 | (uint64_t)(uint32_t)i);
        if (a.state_out) {
            a.state_out[i] = __fadd_rn(p0[j], D[j]);
            a.state_out[N + i] = v[j];
        }
    }
    if (LOSS) vl_block_sum(lacc + (double)lseg, a.loss_partials);
}

// ------------------------------------------------------------------------------ backward
template <bool D4, bool ADAM, int KS>
__global__ void __launch_bounds__(kVT, 2) vl_bwd_kernel(VlArgs a) {
    const int tid = threadIdx.x;
    const int64_t N = a.n;
    const int steps = a.steps;
    const int64_t base = (int64_t)blockIdx.x * kVB + tid;
    const Consts k = a.k;
    const int64_t KN = (int64_t)a.max_steps * N;  // leaf plane stride
    float lv[kVV], lD[kVV];
    bool valid[kVV];
    VehP P[kVV];
    VehB B[kVV];
    GradAcc G[kVV];
#pragma unroll
    for (int j = 0; j < kVV; ++j) {
        const int64_t i = base + j * kVT;
        valid[j] = i < N;
        float r[6] = {1.f, 1.f, 1.f, 1.f, 1.f, 4.f};
        lv[j] = 0.f;
        lD[j] = 0.f;
        if (valid[j]) {
            vl_params(a.params, a.n_par, i, r);
            lD[j] = a.grad_traj[(int64_t)steps * N + i];  // lambda_P^K = dL/dP(K)
        }
        P[j] = make_vehp(r[0], r[1], r[2], r[3], r[4], r[5]);
        B[j] = make_vehb(r[0], r[1], r[4], r[5]);
        G[j] = GradAcc{0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    }
    const int nseg = (steps + KS - 1) / KS;
    for (int seg = nseg - 1; seg >= 0; --seg) {
        const int t0 = seg * KS;
        const int len = min(KS, steps - t0);
        float dp[KS][kVV], dv[KS][kVV], gr[KS][kVV], vt[KS][kVV];
        // ADAM (fused iteration): the leaves' Adam moments of this segment, updated in place
        float am[ADAM ? KS : 1][kVV][2], av[ADAM ? KS : 1][kVV][2];
#pragma unroll
        for (int tt = 0; tt < KS; ++tt)
#pragma unroll
            for (int j = 0; j < kVV; ++j) {
                const bool ok = valid[j] && tt < len;
                const int64_t off = (int64_t)(t0 + tt) * N + base + j * kVT;
                dp[tt][j] = ok ? __ldcs(a.vl_dp + off) : 10.f;
                dv[tt][j] = ok ? __ldcs(a.vl_dv + off) : 0.f;
                gr[tt][j] = ok ? __ldcs(a.grad_traj + off) : 0.f;
                if (ADAM) {
#pragma unroll
                    for (int pl = 0; pl < 2; ++pl) {
                        am[tt][j][pl] = ok ? __ldcs(a.vl_adam_m + pl * KN + off) : 0.f;
                        av[tt][j][pl] = ok ? __ldcs(a.vl_adam_v + pl * KN + off) : 0.f;
                    }
                }
            }
        // recompute the segment's speeds from its checkpoint (bit-identical to the forward)
#pragma unroll
        for (int j = 0; j < kVV; ++j)
            vt[0][j] = valid[j] ? a.ckpt_v[(int64_t)seg * N + base + j * kVT] : 0.f;
#pragma unroll
        for (int tt = 0; tt + 1 < KS; ++tt) {
            if (tt + 1 < len) {
#pragma unroll
                for (int j = 0; j < kVV; ++j) {
                    Core c;
                    core_dv<D4>(dp[tt][j], vt[tt][j], dv[tt][j], 1.f, P[j], k, c);
                    float sdummy = 0.f, vn = vt[tt][j];
                    advance(c, sdummy, vn, k);
                    vt[tt + 1][j] = vn;
                }
            }
        }
        // reverse sweep
#pragma unroll
        for (int tt = KS - 1; tt >= 0; --tt) {
            if (tt < len) {
                const int64_t off = (int64_t)(t0 + tt) * N + base;
#pragma unroll
                for (int j = 0; j < kVV; ++j) {
                    Core c;
                    core_dv<D4>(dp[tt][j], vt[tt][j], dv[tt][j], 1.f, P[j], k, c);
                    float gdp, gdv;
                    bwd_vl<D4>(c, dp[tt][j], vt[tt][j], P[j], B[j], k, lv[j], lD[j], G[j], gdp,
                               gdv);
                    lD[j] += gr[tt][j];  // lambda_P^t = g^t + lambda_P^{t+1}
                    if (valid[j]) {
                        if (ADAM) {  // Adam on the two leaves of step t, in place (no box)
                            const float gg[2] = {gdp, gdv};
                            float* xs[2] = {const_cast<float*>(a.vl_dp), const_cast<float*>(a.vl_dv)};
                            const float x0[2] = {dp[tt][j], dv[tt][j]};
#pragma unroll
                            for (int pl = 0; pl < 2; ++pl) {
                                float mm = am[tt][j][pl], vv = av[tt][j][pl];
                                const float xn = leaf_adam(x0[pl], gg[pl], mm, vv,
                                                           a.adam.step_size, a.adam.sqrt_bc2,
                                                           a.adam.beta1, a.adam.beta2, a.adam.eps);
                                __stcs(a.vl_adam_m + pl * KN + off + j * kVT, mm);
                                __stcs(a.vl_adam_v + pl * KN + off + j * kVT, vv);
                                __stcs(xs[pl] + off + j * kVT, xn);
                            }
                        } else {
                            __stcs(a.vl_grad + off + j * kVT, gdp);
                            __stcs(a.vl_grad + KN + off + j * kVT, gdv);
                        }
                    }
                }
            }
        }
    }
#pragma unroll
    for (int j = 0; j < kVV; ++j) {
        if (!valid[j]) continue;
        const int64_t i = base + j * kVT;
        float r[6];
        vl_params(a.params, a.n_par, i, r);
        const float c = 0.5f / sqrtf(r[0] * r[1]);
        float gr6[6];
        gr6[0] = G[j].S1 - c * (0.5f / r[0]) * G[j].S2;
        gr6[1] = -c * (0.5f / r[1]) * G[j].S2;
        gr6[2] = G[j].S3;
        gr6[3] = G[j].S4;
        gr6[4] = r[0] * r[5] / r[4] * G[j].S5;
        gr6[5] = -r[0] * kLn2 * G[j].S6;
        if (a.grad_state0) {
            a.grad_state0[i] = lD[j];  // dL/dp0: position enters every later P
            a.grad_state0[N + i] = lv[j];
        }
        if (!(isfinite(lv[j]) && isfinite(lD[j])))
            atomicMin(a.status, (unsigned long long)0 << 32 | (uint64_t)(uint32_t)i);
#pragma unroll
        for (int q = 0; q < 6; ++q) {
            a.grad_params[q * N + i] = gr6[q];
            if (ADAM && ((a.adam.opt_mask >> q) & 1u)) adam_update(a.adam, q, q * N + i, gr6[q]);
        }
    }
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
    else vl_fwd_kernel<D4, 0, 4><<<g, b, 0, st>>>(a);
}

cudaError_t launch_vl_fwd(const VlArgs& a, bool delta4, int loss, cudaStream_t st) {
    if (a.ckpt_every != 4) return cudaErrorInvalidValue;
    if (delta4) vl_fwd_d<true>(a, loss, st);
    else vl_fwd_d<false>(a, loss, st);
    return cudaGetLastError();
}

cudaError_t launch_vl_bwd(const VlArgs& a, bool delta4, bool adam, cudaStream_t st) {
    if (a.ckpt_every != 4) return cudaErrorInvalidValue;
    dim3 g((unsigned)vl_blocks(a.n)), b(kVT);
    if (delta4) {
        if (adam) vl_bwd_kernel<true, true, 4><<<g, b, 0, st>>>(a);
        else vl_bwd_kernel<true, false, 4><<<g, b, 0, st>>>(a);
    } else {
        if (adam) vl_bwd_kernel<false, true, 4><<<g, b, 0, st>>>(a);
        else vl_bwd_kernel<false, false, 4><<<g, b, 0, st>>>(a);
    }
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
