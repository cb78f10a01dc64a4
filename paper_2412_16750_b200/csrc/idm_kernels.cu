// idm_kernels.cu -- sm_100a kernels of the differentiable IDM hot path (arXiv 2412.16750).
//
//   NK0 validate_kernel   input checks (finite, v >= 0, params > 0)            once per init
//   NK1 fwd_kernel        K fused steps per lane tile, state in registers       Eqs. 1-3, III-C
//   NK2 loss_kernel       Eq. 4 L1/L2 + dL/dP, fixed-order fp64 partials
//   NK3 bwd_kernel        checkpoint recompute + reverse sweep per lane tile    adjoint of NK1
//   NK4 reduce_kernel     fixed-order sum of per-block fp64 partials (loss / shared grads)
//   NK5 adam_kernel       Adam + linear lr + box clamp
//
// A lane tile is a run of WHOLE lanes of at most kCap vehicles (lanes are independent, so no
// tile ever needs another tile's data).  Local vehicle id = j * kThreads + threadIdx.x
// (j < kVpt): every global access of a warp is 32 consecutive floats, and the leader of local
// vehicle id is id + 1, exchanged through shared memory (one barrier per step).
#include <cstdint>
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
    }
}

__device__ __forceinline__ void report_nonfinite(unsigned long long* status, int step,
                                                 int64_t veh) {
    atomicMin(status, (unsigned long long)(unsigned)step << 32 | (uint64_t)(uint32_t)veh);
}

__device__ __forceinline__ VehP load_params(const float* __restrict__ prm, int64_t n_par,
                                            int64_t i) {
    int64_t j = n_par == 1 ? 0 : i;
    float a_max = prm[j], a_pref = prm[n_par + j];
    VehP p;
    p.a_max = a_max;
    p.s_min = prm[2 * n_par + j];
    p.T = prm[3 * n_par + j];
    p.inv_vtarg = 1.f / prm[4 * n_par + j];
    p.delta = prm[5 * n_par + j];
    p.c = 0.5f / sqrtf(a_max * a_pref);
    return p;
}

__device__ __forceinline__ VehP dummy_params() {
    VehP p;
    p.a_max = 1.f; p.s_min = 1.f; p.T = 1.f; p.inv_vtarg = 1.f; p.delta = 4.f; p.c = 0.5f;
    return p;
}

// ------------------------------------------------------------------------------ NK1
// One CTA = one lane tile.  All `steps` steps run in one launch; per step one __syncthreads
// separates the speed publication from the leader read (double-buffered exchange).
template <bool KAHAN>
__global__ void __launch_bounds__(kThreads) fwd_kernel(FwdArgs a) {
    __shared__ float xv[2][kCap + 1];
    const int tid = threadIdx.x;
    const int64_t base = a.tile_start[blockIdx.x];
    const int n_loc = (int)(a.tile_start[blockIdx.x + 1] - base);
    const Consts k = a.k;

    float s[kVpt], v[kVpt], D[kVpt], cmp[kVpt], p0[kVpt];
    bool lead[kVpt], valid[kVpt];
    VehP P[kVpt];
#pragma unroll
    for (int j = 0; j < kVpt; ++j) {
        int id = j * kThreads + tid;
        int64_t i = base + id;
        valid[j] = id < n_loc;
        D[j] = 0.f;
        cmp[j] = 0.f;
        if (valid[j]) {
            p0[j] = a.pos0[i];
            v[j] = a.vel0[i];
            lead[j] = a.lead[i] != 0;
            s[j] = lead[j] ? (a.pos0[i + 1] - p0[j]) - a.length[i + 1] : 0.f;
            P[j] = load_params(a.params, a.n_par, i);
        } else {
            p0[j] = 0.f; v[j] = 0.f; s[j] = 0.f; lead[j] = false;
            P[j] = dummy_params();
        }
    }
    if (tid == 0) { xv[0][kCap] = 0.f; xv[1][kCap] = 0.f; }

    const int64_t N = a.n;
    float* traj = a.traj;
    float* vtraj = a.vel_traj;
    // row 0 (P(0) = p(0)) and checkpoint 0
#pragma unroll
    for (int j = 0; j < kVpt; ++j) {
        if (!valid[j]) continue;
        int64_t i = base + j * kThreads + tid;
        if (traj) traj[i] = p0[j];
        if (vtraj) vtraj[i] = v[j];
        a.ckpt_s[i] = s[j];
        a.ckpt_v[i] = v[j];
    }
    int next_ck = a.ckpt_every;
    int ck = 1;
    for (int t = 0; t < a.steps; ++t) {
        const int par = t & 1;
#pragma unroll
        for (int j = 0; j < kVpt; ++j) xv[par][j * kThreads + tid] = v[j];
        __syncthreads();
#pragma unroll
        for (int j = 0; j < kVpt; ++j) {
            float vl = xv[par][j * kThreads + tid + 1];
            vl = lead[j] ? vl : v[j];
            if (KAHAN) {  // compensated displacement for long horizons (C3)
                float y = __fmaf_rn(k.dt, v[j], -cmp[j]);
                float tt = __fadd_rn(D[j], y);
                cmp[j] = __fsub_rn(__fsub_rn(tt, D[j]), y);
                D[j] = tt;
            } else {
                D[j] = __fmaf_rn(k.dt, v[j], D[j]);
            }
            fwd_step(s[j], v[j], vl, lead[j], P[j], k);
        }
        const int t1 = t + 1;
        if (traj) {
            float* row = traj + (int64_t)t1 * N + base + tid;
#pragma unroll
            for (int j = 0; j < kVpt; ++j)
                if (valid[j]) row[j * kThreads] = __fadd_rn(p0[j], D[j]);
        }
        if (vtraj) {
            float* row = vtraj + (int64_t)t1 * N + base + tid;
#pragma unroll
            for (int j = 0; j < kVpt; ++j)
                if (valid[j]) row[j * kThreads] = v[j];
        }
        if (t1 == next_ck || t1 == a.steps) {
            if (t1 == next_ck && t1 < a.steps) {
                int64_t off = (int64_t)ck * N + base + tid;
#pragma unroll
                for (int j = 0; j < kVpt; ++j) {
                    if (!valid[j]) continue;
                    a.ckpt_s[off + j * kThreads] = s[j];
                    a.ckpt_v[off + j * kThreads] = v[j];
                }
                ++ck;
                next_ck += a.ckpt_every;
            }
#pragma unroll
            for (int j = 0; j < kVpt; ++j)
                if (valid[j] && !(isfinite(s[j]) && isfinite(v[j]) && isfinite(D[j])))
                    report_nonfinite(a.status, t1, base + j * kThreads + tid);
        }
    }
    if (a.state_out) {
#pragma unroll
        for (int j = 0; j < kVpt; ++j) {
            if (!valid[j]) continue;
            int64_t i = base + j * kThreads + tid;
            a.state_out[i] = __fadd_rn(p0[j], D[j]);
            a.state_out[N + i] = v[j];
        }
    }
}

// ------------------------------------------------------------------------------ NK3
// Per CTA (lane tile), segments of ckpt_every steps from last to first:
//   recompute: reload the (gap, speed) checkpoint, re-run the segment's steps bit-identically,
//              storing the state at every step in shared memory (hist);
//   reverse:   sweep the segment backwards; the follower -> leader adjoint term F is passed
//              through shared memory (local id -> id + 1, one barrier per step).
// Per-vehicle gradient accumulators stay in registers for the whole rollout.
template <bool SHARED>
__global__ void __launch_bounds__(kThreads) bwd_kernel(BwdArgs a) {
    extern __shared__ float2 hist[];  // [ckpt_every][kCap + 1]
    __shared__ float fx[2][kCap + 1];
    const int tid = threadIdx.x;
    const int64_t base = a.tile_start[blockIdx.x];
    const int n_loc = (int)(a.tile_start[blockIdx.x + 1] - base);
    const Consts k = a.k;
    const int64_t N = a.n;
    const int HS = kCap + 1;

    float ls[kVpt], lv[kVpt], lD[kVpt], s[kVpt], v[kVpt];
    bool lead[kVpt], valid[kVpt];
    VehP P[kVpt];
    GradAcc G[kVpt];
#pragma unroll
    for (int j = 0; j < kVpt; ++j) {
        int id = j * kThreads + tid;
        int64_t i = base + id;
        valid[j] = id < n_loc;
        ls[j] = 0.f;
        lv[j] = 0.f;
        G[j] = GradAcc{0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
        if (valid[j]) {
            lead[j] = a.lead[i] != 0;
            P[j] = load_params(a.params, a.n_par, i);
            lD[j] = a.grad_traj[(int64_t)a.steps * N + i];  // lambda_D^K = dL/dP(K)
        } else {
            lead[j] = false;
            P[j] = dummy_params();
            lD[j] = 0.f;
        }
    }
    if (tid == 0) { fx[0][0] = 0.f; fx[1][0] = 0.f; }
    // (fx[.][0] is never written again: slot id+1 >= 1.)

    const int kseg = a.ckpt_every;
    const int nseg = (a.steps + kseg - 1) / kseg;
    int par = 0;
    for (int seg = nseg - 1; seg >= 0; --seg) {
        const int t0 = seg * kseg;
        const int len = min(kseg, a.steps - t0);
        // ---- recompute the segment from its checkpoint
#pragma unroll
        for (int j = 0; j < kVpt; ++j) {
            int64_t off = (int64_t)seg * N + base + j * kThreads + tid;
            s[j] = valid[j] ? a.ckpt_s[off] : 0.f;
            v[j] = valid[j] ? a.ckpt_v[off] : 0.f;
        }
        for (int tt = 0; tt < len; ++tt) {
            float2* h = hist + tt * HS;
#pragma unroll
            for (int j = 0; j < kVpt; ++j) h[j * kThreads + tid] = make_float2(s[j], v[j]);
            __syncthreads();
            if (tt + 1 < len) {
#pragma unroll
                for (int j = 0; j < kVpt; ++j) {
                    float vl = h[j * kThreads + tid + 1].y;
                    vl = lead[j] ? vl : v[j];
                    fwd_step(s[j], v[j], vl, lead[j], P[j], k);
                }
            }
        }
        // ---- reverse sweep
        for (int tt = len - 1; tt >= 0; --tt) {
            const int t = t0 + tt;
            const float2* h = hist + tt * HS;
            float gt[kVpt];
#pragma unroll
            for (int j = 0; j < kVpt; ++j)
                gt[j] = valid[j] ? a.grad_traj[(int64_t)t * N + base + j * kThreads + tid] : 0.f;
            float F[kVpt];
#pragma unroll
            for (int j = 0; j < kVpt; ++j) {
                int id = j * kThreads + tid;
                float2 sv = h[id];
                float vl = lead[j] ? h[id + 1].y : sv.y;
                F[j] = bwd_step(sv.x, sv.y, vl, lead[j], P[j], k, ls[j], lv[j], lD[j], G[j]);
            }
#pragma unroll
            for (int j = 0; j < kVpt; ++j) fx[par][j * kThreads + tid + 1] = F[j];
            __syncthreads();
#pragma unroll
            for (int j = 0; j < kVpt; ++j) {
                lv[j] += fx[par][j * kThreads + tid];  // F from the follower (id - 1)
                lD[j] += gt[j];                        // lambda_D^t = g^t + lambda_D^{t+1}
            }
            par ^= 1;
        }
    }
    // dL/dp0_i = lambda_D - lambda_s_i + lambda_s_{follower}; dL/dv0 = lambda_v
#pragma unroll
    for (int j = 0; j < kVpt; ++j) fx[par][j * kThreads + tid + 1] = lead[j] ? ls[j] : 0.f;
    __syncthreads();
    float gp0[kVpt];
#pragma unroll
    for (int j = 0; j < kVpt; ++j)
        gp0[j] = lD[j] - (lead[j] ? ls[j] : 0.f) + fx[par][j * kThreads + tid];

    // parameter gradients from the factored accumulators
    float gr[kVpt][6];
#pragma unroll
    for (int j = 0; j < kVpt; ++j) {
        if (!valid[j]) {
#pragma unroll
            for (int q = 0; q < 6; ++q) gr[j][q] = 0.f;
            continue;
        }
        int64_t i = base + j * kThreads + tid;
        int64_t jj = a.n_par == 1 ? 0 : i;
        float a_max = a.params[jj], a_pref = a.params[a.n_par + jj];
        float c = P[j].c;
        gr[j][0] = G[j].S1 - c * (0.5f / a_max) * G[j].S2;              // a_max
        gr[j][1] = -c * (0.5f / a_pref) * G[j].S2;                       // a_pref
        gr[j][2] = G[j].S3;                                              // s_min
        gr[j][3] = G[j].S4;                                              // T_pref
        gr[j][4] = a_max * P[j].delta * P[j].inv_vtarg * G[j].S5;       // v_targ
        gr[j][5] = -a_max * G[j].S6;                                     // delta
        if (a.grad_state0) {
            a.grad_state0[i] = gp0[j];
            a.grad_state0[N + i] = lv[j];
        }
    }
    if (!SHARED) {
#pragma unroll
        for (int j = 0; j < kVpt; ++j) {
            if (!valid[j]) continue;
            int64_t i = base + j * kThreads + tid;
#pragma unroll
            for (int q = 0; q < 6; ++q) a.grad_params[q * N + i] = gr[j][q];
        }
        for (int j = 0; j < kVpt; ++j)
            if (valid[j] && !(isfinite(lv[j]) && isfinite(gp0[j])))
                report_nonfinite(a.status, 0, base + j * kThreads + tid);
    } else {
        // fixed-order block reduction in fp64 -> partial[tile][6]
        __shared__ double red[kThreads / 32][6];
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
            for (int w = 0; w < kThreads / 32; ++w) x += red[w][tid];
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
            float r0 = o.x - p.x, r1 = o.y - p.y, r2 = o.z - p.z, r3 = o.w - p.w;
            float4 g;
            float part;
            if (l1) {
                g.x = m.x ? -copysignf(r0 != 0.f, r0) : 0.f;
                g.y = m.y ? -copysignf(r1 != 0.f, r1) : 0.f;
                g.z = m.z ? -copysignf(r2 != 0.f, r2) : 0.f;
                g.w = m.w ? -copysignf(r3 != 0.f, r3) : 0.f;
                part = (m.x ? fabsf(r0) : 0.f) + (m.y ? fabsf(r1) : 0.f) +
                       (m.z ? fabsf(r2) : 0.f) + (m.w ? fabsf(r3) : 0.f);
            } else {
                g.x = m.x ? -2.f * r0 : 0.f;
                g.y = m.y ? -2.f * r1 : 0.f;
                g.z = m.z ? -2.f * r2 : 0.f;
                g.w = m.w ? -2.f * r3 : 0.f;
                part = (m.x ? r0 * r0 : 0.f) + (m.y ? r1 * r1 : 0.f) +
                       (m.z ? r2 * r2 : 0.f) + (m.w ? r3 * r3 : 0.f);
            }
            __stcs(G4 + e, g);
            acc += (double)part;
        }
        // tail (n_elem % 4) handled by the first threads
        for (int64_t e = (n4 << 2) + t0; e < a.n_elem; e += stride) {
            bool m = a.mask ? a.mask[e] != 0 : true;
            float r = a.obs[e] - a.traj[e];
            float g = l1 ? -copysignf(r != 0.f, r) : -2.f * r;
            a.grad[e] = m ? g : 0.f;
            if (m) acc += l1 ? (double)fabsf(r) : (double)r * r;
        }
    } else {
        for (int64_t e = t0; e < a.n_elem; e += stride) {
            bool m = a.mask ? a.mask[e] != 0 : true;
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
        int q = (int)(e / a.n_par);
        if (!((a.opt_mask >> q) & 1u)) continue;
        float g = a.grad[e];
        float m1 = a.m[e] * a.beta1 + (1.f - a.beta1) * g;
        float m2 = a.v[e] * a.beta2 + (1.f - a.beta2) * g * g;
        a.m[e] = m1;
        a.v[e] = m2;
        float denom = sqrtf(m2) / a.sqrt_bc2 + a.eps;
        float x = a.x[e] - a.step_size * (m1 / denom);
        if (q < 5) x = fminf(fmaxf(x, a.lo[q]), a.hi[q]);
        a.x[e] = x;
    }
}

// ------------------------------------------------------------------------------ launchers
cudaError_t launch_validate(const ValidateArgs& a, cudaStream_t st) {
    validate_kernel<<<148 * 4, 256, 0, st>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_fwd(const FwdArgs& a, int ntiles, bool kahan, cudaStream_t st) {
    if (kahan)
        fwd_kernel<true><<<ntiles, kThreads, 0, st>>>(a);
    else
        fwd_kernel<false><<<ntiles, kThreads, 0, st>>>(a);
    return cudaGetLastError();
}

size_t bwd_smem_bytes(int ckpt_every) { return (size_t)ckpt_every * (kCap + 1) * sizeof(float2); }

cudaError_t bwd_configure(int ckpt_every) {
    size_t mx = bwd_smem_bytes(ckpt_every);
    cudaError_t e = cudaFuncSetAttribute(bwd_kernel<false>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)mx);
    if (e != cudaSuccess) return e;
    return cudaFuncSetAttribute(bwd_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)mx);
}

cudaError_t launch_bwd(const BwdArgs& a, int ntiles, bool shared, cudaStream_t st) {
    size_t smem = bwd_smem_bytes(a.ckpt_every);
    if (shared)
        bwd_kernel<true><<<ntiles, kThreads, smem, st>>>(a);
    else
        bwd_kernel<false><<<ntiles, kThreads, smem, st>>>(a);
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
