// idm_internal.h -- kernel argument blocks and launchers shared by idm_kernels.cu and idm_capi.cu.
#pragma once
#include <atomic>
#include <cstdint>
#include <cuda_runtime.h>

#include "idm_device.cuh"

namespace idm {

// status word: UINT64_MAX = OK; otherwise (code_or_step << 32 | index), smallest wins.
constexpr unsigned kBadInput = 0xFFFFFFF0u;  // invalid pos0/vel0/length at vehicle index
constexpr unsigned kBadParam = 0xFFFFFFF1u;  // invalid parameter at flat index
constexpr unsigned kBadDelta = 0xFFFFFFF2u;  // delta != 4 in a delta=4-specialised kernel
constexpr unsigned kBadOrder = 0xFFFFFFF3u;  // lane member overlapping / behind its leader
constexpr unsigned kBadGrad = 0xFFFFFFF4u;   // non-finite parameter gradient (flat index)

// Opt `fn` into `bytes` of dynamic shared memory on the CURRENT device.  The attribute belongs
// to each device's context, so it is set once per device (bit d of `done`), thread-safely
// (a race only sets it twice), and its error is returned.
inline cudaError_t smem_optin(const void* fn, int bytes, std::atomic<unsigned long long>& done) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    const unsigned long long bit = dev < 64 ? 1ull << dev : 0ull;
    if (bit && (done.load(std::memory_order_acquire) & bit)) return cudaSuccess;
    e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (e == cudaSuccess && bit) done.fetch_or(bit, std::memory_order_release);
    return e;
}

struct ValidateArgs {
    const float *pos0, *vel0, *length, *params;
    const uint8_t* lead;  // lane mode: leader flags (order check); nullptr: no lane order
    int64_t n, n_par;
    unsigned long long* status;
    unsigned* delta_not4;
};

struct FwdVariant {
    bool delta4;  // every delta == 4 (two squarings instead of ex2/lg2)
    bool kahan;   // compensated displacement
    bool rec_v;   // record speeds
    int loss;     // 0, or fused Eq. 4 (1 = L1, 2 = L2): read obs, sum the loss (idm_fit_step)
    bool hist = true;  // store the state history for a backward (false: P rows only)
    int csize = 1;     // > 1: lanes longer than a tile, thread-block clusters of csize tiles
};

// Lane-mode state history in HBM, TILE-LOCAL layout (internal workspace):
//   vt  [tile][max_steps + 1][kCap]     speed of every vehicle slot at every step
//   ckt [tile][nck + 1][3][kCap]        (gap, displacement, Kahan compensation) at every
//                                       ckpt_every-th step (the gap only where gap_row(), the
//                                       final gap s_K in row nck's gap slot; see kGapCk)
// A tile's rows are kCap floats apart (compile-time), so a thread's vehicle pair is one
// aligned 8-byte access at an immediate offset, and slots past the tile's vehicles are
// private padding (stores need no predicate).
constexpr int kCkRows = 3;
// Gaps in the history: the gap row of checkpoint j is written only for j % kGapCk == 0, plus
// the final gap s_K in the gap row of checkpoint ceil(K / ckpt_every) (one row past the last
// segment's).  The backward rebuilds every other gap from the later one by the reverse
// recurrence s_t = s_{t+1} + dt (v_t - v_h,t) on the stored speeds, re-anchored on the exact
// row every kGapCk checkpoints (at most kGapCk ckpt_every steps of rounding, a few ulp): 7/8 of
// the gap rows' HBM traffic saved in both kernels.  gap_row() is the one
// rule the forward, the backward and the on-chip fit use.
constexpr int kGapCk = 8;
__host__ __device__ constexpr bool gap_row(int j) { return j % kGapCk == 0; }
//   sgn [tile][max_steps / 4 + 1][kCap / 2] u16, fused L1 only: dL/dP = -sign(obs - P) of a
//                                       thread's two vehicles as a 4-bit code per step (bits 0 / 2:
//                                       r != 0, bits 1 / 3: r < 0), steps 4j .. 4j + 3 in word j
constexpr int kSgnSteps = 4;  // steps per u16 code word
__host__ __device__ constexpr int64_t sgn_words_per_tile(int max_steps) {  // in u32 units
    return (int64_t)(max_steps / kSgnSteps + 1) * (kCap / 2) / 2;
}

struct FwdArgs {
    const int64_t* tile_start;
    const uint8_t* lead;
    const float *pos0, *vel0, *length, *params;
    int64_t n, n_par;
    float *traj, *vel_traj, *state_out;
    float *vt, *ckt;
    int64_t vt_stride, ck_stride;  // floats per tile
    uint32_t* sgn;                 // fused L1: sign codes (u16 words, see above)
    int64_t sg_stride;             // words per tile
    int tile0;                     // first tile of this launch (grid = a chunk of the tiles)
    int steps, ckpt_every;
    Consts k;
    unsigned long long* status;
    // fused loss (LOSS variant): Eq. 4 value only (the backward re-derives dL/dP)
    const float* obs;
    int kind;
    double* loss_partials;  // [ntiles]
    // programmatic dependent launch of the fused backward (nullable): tile_ready[tile] = epoch
    // (release) once the tile's history is written
    unsigned* tile_ready;
    unsigned epoch;
    // fused step (nullable): the last CTA to finish sums loss_partials[0 .. n_tiles) in
    // reduce_kernel's fixed order into *loss_out (done_count: zero between launches)
    double* loss_out;
    unsigned* done_count;
    int n_tiles;
};

struct AdamArgs {
    float *x, *m, *v;
    const float* grad;
    int64_t n_par;
    uint32_t opt_mask;
    float step_size, sqrt_bc2, beta1, beta2, eps;
    float lo[5], hi[5];
    unsigned long long* status;  // a non-finite gradient is reported here (kBadGrad)
};

struct BwdArgs {
    const int64_t* tile_start;
    const uint8_t* lead;
    const float* params;
    int64_t n, n_par;
    const float* grad_traj;        // dL/dP rows (API path)
    const float *obs, *pos0;       // fused path: dL/dP re-derived from obs and positions
    const float *vt, *ckt;
    int64_t vt_stride, ck_stride;
    const uint32_t* sgn;
    int64_t sg_stride;
    int tile0;  // first tile of this launch
    float *grad_params, *grad_state0;
    // shared mode: per-lane fp64 gradient sums -> lane_grads[lane][6] (lane = index into
    // lane_offsets [n_lanes + 1])
    const int32_t* lane_offsets;
    int32_t n_lanes;
    double* lane_grads;
    int steps, ckpt_every;
    Consts k;
    unsigned long long* status;
    AdamArgs adam;  // fused Adam epilogue (ADAM variant)
    // launched as a programmatic dependent of the forward (nullable): wait (acquire) for
    // tile_ready[tile] == epoch before reading the tile's history
    const unsigned* tile_ready;
    unsigned epoch;
    // GOBS >= 2 (nullable): this tile's Eq. 4 loss -> loss_partials[tile] (the forward did not)
    double* loss_partials;
};

// virtual-leader mode (idm_vl.cu)
struct VlArgs {
    const float *pos0, *vel0, *params;
    int64_t n, n_par;
    int steps, max_steps, ckpt_every;
    Consts k;
    const float *vl_dp, *vl_dv;
    float *vl_grad;  // [2][max_steps][N]
    float *vl_adam_m, *vl_adam_v;  // [2][max_steps][N] (fused leaf Adam)
    float *traj, *grad_traj, *state_out, *ckpt_v, *grad_params, *grad_state0;
    float* ckpt_d;  // [nseg][N] displacement checkpoints (history-only forward, loss = 3)
    float* vel_traj;  // nullable: record speeds
    const float* obs;
    double* loss_partials;
    unsigned long long* status;
    AdamArgs adam;
};

// whole fits in one launch (idm_fit.cu)
constexpr int kFitMaxSteps = 12;      // horizon limit of idm_fit (registers per vehicle)
constexpr int kFitMaxIters = 4096;    // per-launch iteration limit (Adam schedule table)
struct FitArgs {
    const int64_t* tile_start;
    const uint8_t* lead;
    const float *pos0, *vel0, *length, *obs;
    float *params, *adam_m, *adam_v, *grad_params, *grad_state0;
    int64_t n;
    int steps, iters;
    uint32_t opt_mask;
    Consts k;
    const float* adam_table;  // [iters][2] (step_size, sqrt_bc2) of each iteration
    float beta1, beta2, eps;
    float lo[5], hi[5];
    double* loss_partials;
    unsigned long long* status;
};

// every iteration of a long-horizon fit in one launch (fit_long_kernel)
struct FitLongArgs {
    int iters;
    const float* adam_table;  // [iters][2] (step_size, sqrt_bc2) of each iteration
};

struct LossArgs {
    const float *traj, *obs;
    const uint8_t* mask;
    float* grad;
    int64_t n_elem;
    int kind;
    double* partials;
};

cudaError_t launch_validate(const ValidateArgs& a, cudaStream_t st);
cudaError_t launch_fwd(const FwdArgs& a, int ntiles, const FwdVariant& var, cudaStream_t st);
cudaError_t kernels_configure(int ckpt_every);
// gobs = 0: dL/dP from grad_traj; 1: L1 from the forward's sign codes; 2 / 3: L2 / L1 re-derived
// from obs and the rebuilt positions (gobs != 0: fused idm_fit_step, ckpt_every == 4)
// pdl: launch as a programmatic dependent of the preceding kernel in the stream (the forward of
// the same tiles, which signals a.tile_ready)
// csize > 1: lanes longer than a tile, thread-block clusters of csize tiles (no pdl)
cudaError_t launch_bwd(const BwdArgs& a, int ntiles, bool delta4, bool shared, bool adam,
                       int gobs, bool kahan, cudaStream_t st, bool pdl = false, int csize = 1);
bool ckpt_supported(int k);
cudaError_t launch_loss(const LossArgs& a, int nblocks, cudaStream_t st);
cudaError_t launch_reduce(const double* partials, int64_t n, int width, double* out, float* out_f,
                          cudaStream_t st);
cudaError_t launch_adam(const AdamArgs& a, cudaStream_t st);
cudaError_t launch_vl_fwd(const VlArgs& a, bool delta4, int loss, cudaStream_t st);
// obs_kind = -1: dL/dP rows from grad_traj; 0 / 1: L1 / L2 derived from obs after the
// history-only forward (loss = 3), fused iteration (adam) only
cudaError_t launch_vl_bwd(const VlArgs& a, bool delta4, bool adam, cudaStream_t st,
                          int obs_kind = -1);
cudaError_t launch_adam_free(float* x, const float* g, float* m, float* v, int64_t n,
                             const AdamArgs& hp, cudaStream_t st);
int64_t vl_blocks(int64_t n);
cudaError_t launch_fit(const FitArgs& a, int ntiles, bool delta4, int kind, cudaStream_t st);
cudaError_t launch_fit_long(const FwdArgs& af, const BwdArgs& ab, const FitLongArgs& fl,
                            int ntiles, bool delta4, bool kahan, int kind, cudaStream_t st);
cudaError_t launch_state_from_obs(const float* obs, int64_t n, int steps, float dt, float* pos0,
                                  float* vel0, cudaStream_t st);

// Adam (Kingma & Ba, bias-corrected) + box clamp of one scalar;
// shared by adam_kernel and the fused backward epilogue so both paths agree bitwise.
#ifdef __CUDACC__
// Predicated streaming load / store (one instruction each, no branch: the compiler otherwise
// branches around guarded accesses and rebuilds every 64-bit row address from scratch).
__device__ __forceinline__ float ld_cs_if(const float* p, bool on, float dflt) {
    float r = dflt;
    asm("{\n .reg .pred q;\n setp.ne.b32 q, %2, 0;\n @q ld.global.cs.f32 %0, [%1];\n}"
        : "+f"(r)
        : "l"(p), "r"((int)on));
    return r;
}
__device__ __forceinline__ void st_cs_if(float* p, bool on, float x) {
    asm volatile("{\n .reg .pred q;\n setp.ne.b32 q, %2, 0;\n @q st.global.cs.f32 [%0], %1;\n}"
                 ::"l"(p), "f"(x), "r"((int)on)
                 : "memory");
}

__device__ __forceinline__ float leaf_adam(float x, float g, float& m, float& v, float step_size,
                                           float sqrt_bc2, float b1, float b2, float eps);

// The caller reports a non-finite g (report_bad_grad): a NaN gradient would otherwise reset the
// parameter to its lower bound through the clamp (fminf / fmaxf drop NaN) while the loss still
// looks finite.
__device__ __forceinline__ void adam_update(const AdamArgs& a, int q, int64_t e, float g) {
    float m = a.m[e], v = a.v[e];
    float x = leaf_adam(a.x[e], g, m, v, a.step_size, a.sqrt_bc2, a.beta1, a.beta2, a.eps);
    a.m[e] = m;
    a.v[e] = v;
    if (q < 5) x = fminf(fmaxf(x, a.lo[q]), a.hi[q]);
    a.x[e] = x;
}

__device__ __forceinline__ void report_bad_grad(unsigned long long* status, int64_t e) {
    atomicMin(status, (unsigned long long)kBadGrad << 32 | (uint64_t)e);
}

// Adam on one scalar (parameters and virtual-leader leaves), explicit roundings so the separate
// kernels, the fused backward and the whole-fit kernel produce the same bits.  The update
//   x - step m1 / (sqrt(m2) / c + eps)  ==  x - (step c) m1 / (sqrt(m2) + eps c),  c = sqrt(bc2)
// uses the MUFU sqrt and reciprocal (a few ulp on a step of size ~lr) instead of IEEE divide and
// square root, whose slow paths dominated the virtual-leader backward's instruction count.
__device__ __forceinline__ float leaf_adam(float x, float g, float& m, float& v, float step_size,
                                           float sqrt_bc2, float b1, float b2, float eps) {
    const float m1 = __fmaf_rn(__fsub_rn(1.f, b1), g, __fmul_rn(m, b1));
    const float m2 = __fmaf_rn(__fmul_rn(__fsub_rn(1.f, b2), g), g, __fmul_rn(v, b2));
    m = m1;
    v = m2;
    float sq;
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(sq) : "f"(m2));
    const float den = __fmaf_rn(eps, sqrt_bc2, sq);
    return __fmaf_rn(-__fmul_rn(step_size, sqrt_bc2), __fmul_rn(m1, rcp(den)), x);
}
#endif


constexpr int kLossBlocks = 148 * 8;  // fixed => deterministic loss reduction

}  // namespace idm
