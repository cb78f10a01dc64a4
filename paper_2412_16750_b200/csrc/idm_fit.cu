// idm_fit.cu -- whole fits in one launch for short horizons.
//
// Waymo-shaped prediction fits the IDM parameters of every agent on a
// 1-second history (10 steps of 0.1 s) before rolling out.  With K <= kFitMaxSteps the whole
// state history, the observations and the Adam moments of a 512-vehicle lane tile fit on chip,
// so fit_kernel runs `iters` complete iterations (forward + Eq. 4 + reverse sweep + Adam) in
// one launch with no HBM traffic between iterations.  Arithmetic is the same device code as
// fwd_kernel<LOSS> / bwd_kernel<ADAM> (core, jac_record, bwd_from_record, loss term, Adam), in
// the same order, so the parameters come out bit-identical to `iters` idm_fit_step calls.
#include <cstdint>
#include <cuda_runtime.h>

#include "idm_device.cuh"
#include "idm_internal.h"

namespace idm {

constexpr int kFT = kCap;  // one vehicle per thread, 512 threads per CTA

template <int KM, bool D4, int KIND>
__global__ void __launch_bounds__(kFT, 1) fit_kernel(FitArgs a) {
    __shared__ float hv[KM][kCap + 1];  // speeds per step (leader reads)
    __shared__ float fx[2][kCap + 1];   // follower -> leader adjoint term
    __shared__ double red[kFT / 32];
    const int tid = threadIdx.x;
    const int64_t base = a.tile_start[blockIdx.x];
    const int n_loc = (int)(a.tile_start[blockIdx.x + 1] - base);
    const int64_t N = a.n;
    const int K = a.steps;
    const Consts k = a.k;
    const bool valid = tid < n_loc;
    const int64_t i = base + tid;

    float p0 = 0.f, v0 = 0.f, s0 = 0.f, leadf = 0.f;
    float x[6] = {1.f, 1.f, 1.f, 1.f, 1.f, 4.f}, m1[6], m2[6];
    float ob[KM + 1];
    if (valid) {
        p0 = a.pos0[i];
        v0 = a.vel0[i];
        const bool lead = a.lead[i] != 0;
        leadf = lead ? 1.f : 0.f;
        s0 = lead ? (a.pos0[i + 1] - p0) - a.length[i + 1] : 0.f;
#pragma unroll
        for (int q = 0; q < 6; ++q) {
            x[q] = a.params[q * N + i];
            m1[q] = a.adam_m[q * N + i];
            m2[q] = a.adam_v[q * N + i];
        }
    } else {
#pragma unroll
        for (int q = 0; q < 6; ++q) { m1[q] = 0.f; m2[q] = 0.f; }
    }
#pragma unroll
    for (int t = 0; t <= KM; ++t)  // absent vehicles observe NaN (= missing)
        ob[t] = (valid && t <= K) ? a.obs[(int64_t)t * N + i] : __int_as_float(0x7fc00000);
    if (tid == 0) {
        fx[0][0] = 0.f;
        fx[1][0] = 0.f;
    }
    if (tid < KM) hv[tid][kCap] = 0.f;  // leader-read sentinel of the last thread
    if (D4 && valid && x[5] != 4.f)
        atomicMin(a.status, (unsigned long long)kBadDelta << 32 | (uint64_t)i);

    float st[KM], vt[KM], g[KM + 1];
    float lsum = 0.f;
    int par = 0;
    for (int it = 0; it < a.iters; ++it) {
        const VehP P = make_vehp(x[0], x[1], x[2], x[3], x[4], x[5]);
        const VehB B = make_vehb(x[0], x[1], x[4], x[5]);
        // ---- forward + Eq. 4 (as fwd_kernel<LOSS>)
        float s = s0, v = v0, D = 0.f;
        lsum = 0.f;
        g[0] = loss_term<KIND>(ob[0], p0, lsum);
#pragma unroll
        for (int t = 0; t < KM; ++t) {
            if (t < K) {
                st[t] = s;
                vt[t] = v;
                hv[t][tid] = v;
                __syncthreads();
                const float vl = hv[t][tid + 1];
                D = vfma(v, k.dt, D);
                fwd_step<D4>(s, v, vl, leadf, P, k);
                g[t + 1] = loss_term<KIND>(ob[t + 1], vadd(p0, D), lsum);
            }
        }
        // ---- reverse sweep (as bwd_kernel: local Jacobian of each step, then the update)
        float ls = 0.f, lv = 0.f, lD = 0.f;
        GradAcc G = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int t = KM; t >= 0; --t)
            if (t == K) lD = g[t];  // lambda_D^K = dL/dP(K)
#pragma unroll
        for (int t = KM - 1; t >= 0; --t) {
            if (t < K) {
                const float vl = hv[t][tid + 1];
                Core c;
                core<D4>(st[t], vt[t], vl, leadf, P, k, c);
                const RecT<float> R = jac_record<D4>(c, st[t], vt[t], P, B, k);
                const float F = bwd_from_record<D4>(R, vt[t], vl, P, B, k, ls, lv, lD, G);
                fx[par][tid + 1] = F;
                __syncthreads();
                lv = vadd(lv, fx[par][tid]);
                lD = vadd(lD, g[t]);
                par ^= 1;
            }
        }
        // ---- gradients (as bwd_kernel's epilogue) + Adam (as adam_update)
        const float c = 0.5f / sqrtf(x[0] * x[1]);
        float gr[6];
        gr[0] = G.S1 - c * (0.5f / x[0]) * G.S2;
        gr[1] = -c * (0.5f / x[1]) * G.S2;
        gr[2] = G.S3;
        gr[3] = G.S4;
        gr[4] = x[0] * x[5] / x[4] * G.S5;
        gr[5] = -x[0] * kLn2 * G.S6;
        const float step_size = a.adam_table[2 * it], sqrt_bc2 = a.adam_table[2 * it + 1];
#pragma unroll
        for (int q = 0; q < 6; ++q) {
            if (!((a.opt_mask >> q) & 1u)) continue;
            float xn = leaf_adam(x[q], gr[q], m1[q], m2[q], step_size, sqrt_bc2, a.beta1,
                                 a.beta2, a.eps);
            if (q < 5) xn = fminf(fmaxf(xn, a.lo[q]), a.hi[q]);
            x[q] = xn;
        }
        if (it + 1 == a.iters && valid) {
#pragma unroll
            for (int q = 0; q < 6; ++q) a.grad_params[q * N + i] = gr[q];
            if (a.grad_state0) fx[par][tid + 1] = vmul(ls, leadf);
        }
        if (it + 1 == a.iters) {
            __syncthreads();
            if (a.grad_state0 && valid) {
                a.grad_state0[i] = vadd(vsub(lD, vmul(ls, leadf)), fx[par][tid]);
                a.grad_state0[N + i] = lv;
            }
        }
    }
    if (valid) {
#pragma unroll
        for (int q = 0; q < 6; ++q) {
            a.params[q * N + i] = x[q];
            a.adam_m[q * N + i] = m1[q];
            a.adam_v[q * N + i] = m2[q];
        }
    }
    // loss of the last iteration: fixed-order CTA sum -> partials[tile]
    double y = (double)lsum;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) y += __shfl_xor_sync(0xffffffffu, y, o);
    if ((tid & 31) == 0) red[tid >> 5] = y;
    __syncthreads();
    if (tid == 0) {
        double z = 0.0;
        for (int w = 0; w < kFT / 32; ++w) z += red[w];
        a.loss_partials[blockIdx.x] = z;
    }
}

cudaError_t launch_fit(const FitArgs& a, int ntiles, bool delta4, int kind, cudaStream_t st) {
    if (a.steps < 1 || a.steps > kFitMaxSteps) return cudaErrorInvalidValue;
    dim3 g(ntiles), b(kFT);
    if (delta4) {
        if (kind == 0) fit_kernel<kFitMaxSteps, true, 0><<<g, b, 0, st>>>(a);
        else fit_kernel<kFitMaxSteps, true, 1><<<g, b, 0, st>>>(a);
    } else {
        if (kind == 0) fit_kernel<kFitMaxSteps, false, 0><<<g, b, 0, st>>>(a);
        else fit_kernel<kFitMaxSteps, false, 1><<<g, b, 0, st>>>(a);
    }
    return cudaGetLastError();
}

}  // namespace idm
