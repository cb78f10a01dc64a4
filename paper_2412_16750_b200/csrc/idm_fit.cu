// idm_fit.cu -- whole fits in one launch for short horizons.
//
// Waymo-shaped prediction fits the IDM parameters of every agent on a
// 1-second history (10 steps of 0.1 s) before rolling out.  With K <= kFitMaxSteps the whole
// state history, the observations and the Adam moments of a 512-vehicle lane tile fit on chip,
// so fit_kernel runs `iters` complete iterations (forward + Eq. 4 + reverse sweep + Adam) in
// one launch with no HBM traffic between iterations.
//
// Layout as the lane kernels: 256 threads, thread t owns the adjacent vehicles 2t, 2t + 1 as
// one float2 pair (packed f32x2 arithmetic); the Adam state of both vehicles stays in registers
// across iterations, the per-step history (speeds, gaps, dL/dP) and the observations live in
// this CTA's shared memory.  Arithmetic is the same device code as fwd_kernel<LOSS> /
// bwd_kernel<ADAM> (core, jac_record, bwd_from_record, loss term, Adam), in the same order, so
// the parameters come out bit-identical to `iters` idm_fit_step calls.
#include <climits>
#include <cstdint>
#include <cuda_runtime.h>

#include "idm_device.cuh"
#include "idm_internal.h"

namespace idm {

namespace {
constexpr int kFT = kCap / 2;  // 256 threads, two vehicles each

template <int KM>
constexpr size_t fit_smem_of() {  // speed pairs (+ sentinel) | gaps | dL/dP | observations
    return (size_t)(KM * (kFT + 1) + KM * kFT + 2 * (KM + 1) * kFT) * sizeof(float2);
}
}  // namespace

template <int KM, bool D4, int KIND>
__global__ void __launch_bounds__(kFT, 2) fit_kernel(FitArgs a) {
    extern __shared__ __align__(16) float2 smem_fit[];
    float2* hv = smem_fit;                        // [KM][kFT + 1] speed pairs; [kFT] = 0
    float2* sg = hv + KM * (kFT + 1);             // [KM][kFT]     gap pairs
    float2* gg = sg + KM * kFT;                   // [KM + 1][kFT] dL/dP pairs
    float2* ob = gg + (KM + 1) * kFT;             // [KM + 1][kFT] observation pairs
    __shared__ float fx[2][kFT + 1];              // follower -> leader adjoint term
    __shared__ double red[kFT / 32];
    const int tid = threadIdx.x;
    const int64_t base = a.tile_start[blockIdx.x];
    const int n_loc = (int)(a.tile_start[blockIdx.x + 1] - base);
    const int64_t N = a.n;
    const int K = a.steps;
    const Consts k = a.k;
    const int id0 = 2 * tid;
    const int64_t i0 = base + id0;
    const bool val[2] = {id0 < n_loc, id0 + 1 < n_loc};
    const float qnan = __int_as_float(0x7fc00000);

    const float pinf = __int_as_float(0x7f800000);
    float pj[2] = {0.f, 0.f}, vj[2] = {0.f, 0.f}, sj[2] = {pinf, pinf};  // no leader: gap +inf
    float x[2][6], m1[2][6], m2[2][6];
    int bad_it = INT_MAX;  // first iteration with a non-finite gradient (reported at the end)
    int64_t bad_e = 0;
#pragma unroll
    for (int j = 0; j < 2; ++j) {
        const int64_t i = i0 + j;
#pragma unroll
        for (int q = 0; q < 6; ++q) {
            x[j][q] = q == 5 ? 4.f : 1.f;
            m1[j][q] = 0.f;
            m2[j][q] = 0.f;
        }
        if (val[j]) {
            pj[j] = a.pos0[i];
            vj[j] = a.vel0[i];
            if (a.lead[i] != 0) sj[j] = (a.pos0[i + 1] - pj[j]) - a.length[i + 1];
#pragma unroll
            for (int q = 0; q < 6; ++q) {
                x[j][q] = a.params[q * N + i];
                m1[j][q] = a.adam_m[q * N + i];
                m2[j][q] = a.adam_v[q * N + i];
            }
            if (D4 && x[j][5] != 4.f)
                atomicMin(a.status, (unsigned long long)kBadDelta << 32 | (uint64_t)i);
        }
    }
    const float2 p0 = make_float2(pj[0], pj[1]), v0 = make_float2(vj[0], vj[1]);
    const float2 s0 = make_float2(sj[0], sj[1]);
    for (int t = 0; t <= KM; ++t) {  // absent vehicles observe NaN (= missing)
        const float* o = a.obs + (int64_t)min(t, K) * N + i0;
        ob[t * kFT + tid] = make_float2((val[0] && t <= K) ? o[0] : qnan,
                                        (val[1] && t <= K) ? o[1] : qnan);
    }
    if (tid == 0) {
        fx[0][0] = 0.f;
        fx[1][0] = 0.f;
    }
    if (tid < KM) hv[tid * (kFT + 1) + kFT] = f2(0.f);  // leader-read sentinel of thread kFT-1
    __syncthreads();

    float2 lsum = f2(0.f);
    int par = 0;
    for (int it = 0; it < a.iters; ++it) {
        const VehPT<float2> P =
            pack(make_vehp(x[0][0], x[0][1], x[0][2], x[0][3], x[0][4], x[0][5]),
                 make_vehp(x[1][0], x[1][1], x[1][2], x[1][3], x[1][4], x[1][5]));
        const VehAT<float2> B = pack(make_veha(x[0][0], x[0][1], x[0][4], x[0][5], k),
                                     make_veha(x[1][0], x[1][1], x[1][4], x[1][5], k));
        // ---- forward + Eq. 4 (as fwd_kernel<LOSS>)
        float2 s = s0, v = v0, D = f2(0.f);
        lsum = f2(0.f);
        gg[tid] = loss_term<KIND>(ob[tid], p0, lsum);
#pragma unroll
        for (int t = 0; t < KM; ++t) {
            if (t < K) {
                sg[t * kFT + tid] = s;
                hv[t * (kFT + 1) + tid] = v;
                __syncthreads();
                const float2 vl = make_float2(v.y, hv[t * (kFT + 1) + tid + 1].x);
                D = vfma(v, k.dt, D);
                fwd_step<D4>(s, v, vl, P, k);
                gg[(t + 1) * kFT + tid] =
                    loss_term<KIND>(ob[(t + 1) * kFT + tid], vadd(p0, D), lsum);
            }
        }
        // ---- reverse sweep (as bwd_kernel: local Jacobian of each step, then the update)
        // scaled adjoint as bwd_kernel: u = dt lambda_v, m = -dt lambda_s, e = dt^2 lambda_D
        float2 m = f2(0.f), u = f2(0.f), e = vmul(gg[K * kFT + tid], k.dt2);  // lambda_D^K = dL/dP(K)
        GradAccT<float2> G = {f2(0.f), f2(0.f), f2(0.f), f2(0.f), f2(0.f), f2(0.f)};
        // gaps as bwd_kernel sees them: the reverse recurrence from the final gap s_K, exact at
        // the first step of each 4-step segment with a gap checkpoint row (gap_row)
        constexpr int kSeg = 4;  // the fused backward's segment (ckpt_every)
        float2 sn = s;           // s_K
#pragma unroll
        for (int t = KM - 1; t >= 0; --t) {
            if (t < K) {
                const float2 vv = hv[t * (kFT + 1) + tid];
                const float2 vl = make_float2(vv.y, hv[t * (kFT + 1) + tid + 1].x);
                const float2 sv = (t % kSeg == 0 && gap_row(t / kSeg))
                                      ? sg[t * kFT + tid]
                                      : vfma(vsub(vv, vl), k.dt, sn);
                sn = sv;
                CoreT<float2> c;
                core<D4>(sv, vv, vl, P, k, c);
                const RecT<float2> R = jac_record<D4, !D4>(c, sv, vv, P, B, k);
                const float2 F = bwd_from_record<D4, !D4>(R, vv, vl, P, B, k, m, u, e, G);
                fx[par][tid + 1] = F.y;  // vehicle 2t + 1 -> its leader 2t + 2 (thread t + 1)
                __syncthreads();
                u = vadd(u, make_float2(fx[par][tid], F.x));
                e = vfma(gg[t * kFT + tid], k.dt2, e);
                par ^= 1;
            }
        }
        // ---- gradients (as bwd_kernel's epilogue) + Adam (as adam_update)
        unscale_acc(G, k);
        const float Sj[6][2] = {{G.S1.x, G.S1.y}, {G.S2.x, G.S2.y}, {G.S3.x, G.S3.y},
                                {G.S4.x, G.S4.y}, {G.S5.x, G.S5.y}, {G.S6.x, G.S6.y}};
        const float step_size = a.adam_table[2 * it], sqrt_bc2 = a.adam_table[2 * it + 1];
        float gr[2][6];
#pragma unroll
        for (int j = 0; j < 2; ++j) {
            const float Sv[6] = {Sj[0][j], Sj[1][j], Sj[2][j], Sj[3][j], Sj[4][j], Sj[5][j]};
            param_grads(x[j], Sv, gr[j]);
            if (!((a.opt_mask >> 5) & 1u)) gr[j][5] = 0.f;  // delta frozen: not computed
#pragma unroll
            for (int q = 0; q < 6; ++q) {
                if (!((a.opt_mask >> q) & 1u)) continue;
                // a NaN gradient would reset the parameter to its bound through the clamp
                if (val[j] && !isfinite(gr[j][q]) && bad_it == INT_MAX) {
                    bad_it = it;
                    bad_e = q * N + i0 + j;
                }
                float xn = leaf_adam(x[j][q], gr[j][q], m1[j][q], m2[j][q], step_size, sqrt_bc2,
                                     a.beta1, a.beta2, a.eps);
                if (q < 5) xn = fminf(fmaxf(xn, a.lo[q]), a.hi[q]);
                x[j][q] = xn;
            }
        }
        if (it + 1 == a.iters) {
            fx[par][tid + 1] = m.y;
            __syncthreads();
            const float2 gp0 = grad_p0(e, m, make_float2(fx[par][tid], m.x), k);
            const float2 gv0 = grad_v0(u, k);
            const float gpj[2] = {gp0.x, gp0.y}, lvj[2] = {gv0.x, gv0.y};
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                if (!val[j]) continue;
                const int64_t i = i0 + j;
#pragma unroll
                for (int q = 0; q < 6; ++q) a.grad_params[q * N + i] = gr[j][q];
                if (a.grad_state0) {
                    a.grad_state0[i] = gpj[j];
                    a.grad_state0[N + i] = lvj[j];
                }
            }
        }
    }
#pragma unroll
    for (int j = 0; j < 2; ++j) {
        if (!val[j]) continue;
        const int64_t i = i0 + j;
#pragma unroll
        for (int q = 0; q < 6; ++q) {
            a.params[q * N + i] = x[j][q];
            a.adam_m[q * N + i] = m1[j][q];
            a.adam_v[q * N + i] = m2[j][q];
        }
    }
    if (bad_it != INT_MAX) atomicMin(a.status, (unsigned long long)kBadGrad << 32 | (uint64_t)bad_e);
    // loss of the last iteration: fixed-order CTA sum -> partials[tile]
    double y = (double)lsum.x + (double)lsum.y;
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

template <bool D4, int KIND>
static cudaError_t launch_fit_v(const FitArgs& a, int ntiles, cudaStream_t st) {
    constexpr size_t smem = fit_smem_of<kFitMaxSteps>();
    static std::atomic<unsigned long long> optin{0};  // devices opted in (bit per device)
    cudaError_t e = smem_optin((const void*)fit_kernel<kFitMaxSteps, D4, KIND>, (int)smem, optin);
    if (e != cudaSuccess) return e;
    fit_kernel<kFitMaxSteps, D4, KIND><<<ntiles, kFT, smem, st>>>(a);
    return cudaSuccess;
}

cudaError_t launch_fit(const FitArgs& a, int ntiles, bool delta4, int kind, cudaStream_t st) {
    if (a.steps < 1 || a.steps > kFitMaxSteps) return cudaErrorInvalidValue;
    cudaError_t e;
    if (delta4) e = kind == 0 ? launch_fit_v<true, 0>(a, ntiles, st) : launch_fit_v<true, 1>(a, ntiles, st);
    else e = kind == 0 ? launch_fit_v<false, 0>(a, ntiles, st) : launch_fit_v<false, 1>(a, ntiles, st);
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}

}  // namespace idm
