// idm_kernels.cu -- sm_100a kernels of the differentiable IDM hot path (arXiv 2412.16750).
//
//   NK0 validate_kernel   input checks (finite, v >= 0, params > 0)            once per init
//   NK1 fwd_kernel        K fused steps per lane tile, state in registers;     Eqs. 1-3, III-C
//                         stores the speed history (+ fused Eq. 4 value, L1 sign bits)
//   NK2 loss_kernel       Eq. 4 L1/L2 + dL/dP, fixed-order fp64 partials
//   NK3 bwd_kernel        rebuild gaps from the stored history, local Jacobians, adjoint of NK1
//                         reverse sweep per lane tile (+ fused Adam epilogue)
//   NK4 reduce_kernel     fixed-order sum of per-block fp64 partials (loss / shared grads)
//   NK5 adam_kernel       Adam + linear lr + box clamp
//
// A lane tile is a run of WHOLE lanes of at most kCap = 512 vehicles (lanes are independent, so
// no tile ever needs another tile's data).  A CTA of kT = 256 threads owns one tile; thread t
// owns the adjacent local vehicles 2t, 2t + 1 as one float2 pair (packed f32x2 arithmetic), so
// vehicle 2t's leader is in the thread and 2t + 1's is thread t + 1's first vehicle (one
// shared-memory word and one barrier per step).  Segments are KS steps (compile-time,
// unrolled).  Lane-mode state history and its layout: idm_internal.h, DESIGN.md section 3.
#include <cstdlib>
#include <climits>
#include <cstdint>
#include <type_traits>
#include <utility>
#include <cuda_runtime.h>

#include "idm_device.cuh"
#include "idm_internal.h"

namespace idm {

// f(integral_constant<int, 0>) ... f(integral_constant<int, N - 1>): an unrolled loop whose index
// is a compile-time constant inside the body
template <class F, int... I>
__device__ __forceinline__ void static_for_impl(F& f, std::integer_sequence<int, I...>) {
    (f(std::integral_constant<int, I>{}), ...);
}
template <int N, class F>
__device__ __forceinline__ void static_for(F&& f) {
    static_for_impl(f, std::make_integer_sequence<int, N>{});
}

// ------------------------------------------------------------------------------ NK0
__global__ void validate_kernel(ValidateArgs a) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (; i < a.n; i += stride) {
        float p = a.pos0[i], v = a.vel0[i], l = a.length[i];
        bool ok = isfinite(p) && isfinite(v) && isfinite(l) && v >= 0.f && l >= 0.f;
        if (!ok) atomicMin(a.status, (unsigned long long)(kBadInput) << 32 | (uint64_t)i);
    }
    // lane order (the leader is the vehicle directly ahead in the same lane): a
    // lane member must be strictly behind its leader with a positive gap, else the input is
    // out of order or overlapping (gaps in (0, eps_gap) are valid and clamped, R#7)
    if (a.lead)
        for (i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < a.n; i += stride) {
            if (!a.lead[i]) continue;
            const float gap = (a.pos0[i + 1] - a.pos0[i]) - a.length[i + 1];  // as fwd_kernel
            if (!(gap > 0.f)) atomicMin(a.status, (unsigned long long)(kBadOrder) << 32 | (uint64_t)i);
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

constexpr int kVpt = 2;          // vehicles per thread (one float2 lane pair)
constexpr int kT = kCap / kVpt;   // 256 threads per CTA

// fixed-order CTA reduction of one double per thread (NT threads) -> *out (deterministic)
template <int NT = kT>
__device__ __forceinline__ void block_sum_to(double x, double* out) {
    __shared__ double red[NT / 32];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = x;
    __syncthreads();
    if (threadIdx.x == 0) {
        double y = 0.0;
        for (int w = 0; w < NT / 32; ++w) y += red[w];
        *out = y;
    }
}

// ------------------------------------------------------------------------------ tile handoff
// The fused backward may start while the forward's last wave drains (programmatic dependent
// launch, launch_bwd(pdl)): forward CTA j releases tile_ready[j] = epoch after its last global
// store, backward CTA j acquires it before its first read of the tile's history.  The forward
// allows the dependent launch at its start, so the backward grid launches only once every forward
// CTA is resident or done: a waiting backward CTA never blocks the forward it waits for.
__device__ __forceinline__ void tile_release(unsigned* flag, unsigned epoch) {
    __threadfence();  // every thread's history stores, at gpu scope
    __syncthreads();
    if (threadIdx.x == 0)
        asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(flag), "r"(epoch) : "memory");
}
// The wait is bounded: a forward CTA that has started finishes within its `steps` steps, so a
// handoff still missing after ~2^24 + 1024 * steps polls (seconds, orders of magnitude above any
// forward CTA's duration) is a bug, and it fails the launch instead of hanging the GPU.
__device__ __forceinline__ void tile_acquire(const unsigned* flag, unsigned epoch, int steps) {
    unsigned v;
    const long long bound = (1ll << 24) + 1024ll * steps;
    for (long long spins = 0;; ++spins) {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(flag) : "memory");
        if (v == epoch) break;
        if (spins > bound) __trap();
        __nanosleep(64);
    }
    // order the acquire before the bulk copies (async proxy) that read the history
    asm volatile("fence.proxy.async.global;" ::: "memory");
}

// ------------------------------------------------------------------------------ async copies
// 1-D bulk copies (global -> shared, completion counted on an mbarrier in bytes): the
// tile-local rows are 16-byte aligned and contiguous, so one elected thread moves a whole
// 2 KB row per instruction and no register holds data in flight.
namespace {
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_fence_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
        ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "IDM_WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra IDM_WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
// per-thread 4-byte async copy global -> shared (src_size 0: zero-fill, nothing read)
__device__ __forceinline__ void cp_async4(float* dst, const float* src, bool on) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(smem_u32(dst)), "l"(src),
                 "r"(on ? 4 : 0)
                 : "memory");
}
// 4-byte cp.async issued only when `on` (no zero-fill: the destination keeps its value)
__device__ __forceinline__ void cp_async4_if(float* dst, const float* src, bool on) {
    asm volatile("{\n .reg .pred q;\n setp.ne.b32 q, %2, 0;\n"
                 " @q cp.async.ca.shared.global [%0], [%1], 4;\n}" ::"r"(smem_u32(dst)),
                 "l"(src), "r"((int)on)
                 : "memory");
}
// 8-byte cp.async issued only when `on` (both addresses 8-byte aligned)
__device__ __forceinline__ void cp_async8_if(float* dst, const float* src, bool on) {
    asm volatile("{\n .reg .pred q;\n setp.ne.b32 q, %2, 0;\n"
                 " @q cp.async.ca.shared.global [%0], [%1], 8;\n}" ::"r"(smem_u32(dst)),
                 "l"(src), "r"((int)on)
                 : "memory");
}
// 16-byte cp.async bypassing L1 (streamed rows), issued only when `on` (16-byte aligned)
__device__ __forceinline__ void cp_async16_if(float* dst, const float* src, bool on) {
    asm volatile("{\n .reg .pred q;\n setp.ne.b32 q, %2, 0;\n"
                 " @q cp.async.cg.shared.global [%0], [%1], 16;\n}" ::"r"(smem_u32(dst)),
                 "l"(src), "r"((int)on)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() {
    asm volatile("cp.async.commit_group;" ::: "memory");
}
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// ------------------------------------------------------------------ thread-block clusters
// A lane longer than one tile (kCap vehicles) runs as consecutive full tiles of one cluster
// (idm_capi.cu plan_tiles): CTA r + 1 holds the vehicles ahead of CTA r's, so the leader of CTA
// r's last vehicle is CTA r + 1's first, read from its shared memory (DSMEM), and every step
// barrier is cluster-wide.  Tiles of whole lanes inside such a launch do the same with no peer.
__device__ __forceinline__ unsigned cluster_rank() {
    unsigned r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\t"
                 "barrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// shared-memory word `p` (a local address) of cluster CTA `rank`
__device__ __forceinline__ float ld_peer(const float* p, unsigned rank) {
    uint32_t ra;
    float v;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(smem_u32(p)), "r"(rank));
    asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(v) : "r"(ra) : "memory");
    return v;
}
__device__ __forceinline__ double ld_peer(const double* p, unsigned rank) {
    uint32_t ra;
    double v;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(smem_u32(p)), "r"(rank));
    asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(ra) : "memory");
    return v;
}
// the per-step barrier: CTA-wide, or cluster-wide for lanes split over a cluster (CL)
template <bool CL>
__device__ __forceinline__ void step_sync() {
    if constexpr (CL) cluster_sync_all();
    else __syncthreads();
}

// One-way per-step message channel between neighbouring cluster CTAs (the boundary vehicle's
// value of each step).  A cluster-wide barrier per step compiles to a GPU-scope MEMBAR (each
// thread waits for its streaming history stores) plus an L1 invalidate; instead the producer
// pushes the value with st.async into the consumer CTA's slot, completing on the consumer's
// mbarrier (no fence), and a cluster barrier every kChanQ messages bounds how far the producer
// may run ahead (flow control: a slot is rewritten only in the next window, after its reader
// passed the barrier).  The buffer sits at the same shared offset in every CTA of the kernel.
constexpr int kChanQ = 32;
struct ChanBuf {
    uint64_t bar[kChanQ];  // consumer-side: one completion (4 bytes + 1 arrival) per window
    float val[kChanQ];
};
__device__ __forceinline__ uint32_t mapa_u32(const void* p, unsigned rank) {
    uint32_t ra;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(smem_u32(p)), "r"(rank));
    return ra;
}
// consumer thread: initialise and arm every slot for the first window (call before the
// cluster barrier that precedes the first send)
__device__ __forceinline__ void chan_init(ChanBuf& c) {
    for (int q = 0; q < kChanQ; ++q) mbar_init(&c.bar[q], 1);
    mbar_fence_init();
    for (int q = 0; q < kChanQ; ++q) mbar_expect_tx(&c.bar[q], 4);
}
// producer thread: message seq into cluster CTA `rank`'s channel
__device__ __forceinline__ void chan_send(ChanBuf& c, unsigned rank, int seq, float v) {
    const int q = seq % kChanQ;
    asm volatile(
        "st.async.shared::cluster.mbarrier::complete_tx::bytes.b32 [%0], %1, [%2];" ::"r"(
            mapa_u32(&c.val[q], rank)),
        "r"(__float_as_uint(v)), "r"(mapa_u32(&c.bar[q], rank))
        : "memory");
}
// consumer thread: wait for message seq, read it, re-arm its slot for the next window
__device__ __forceinline__ float chan_recv(ChanBuf& c, int seq) {
    const int q = seq % kChanQ;
    mbar_wait(&c.bar[q], (uint32_t)(seq / kChanQ) & 1u);
    const float v = c.val[q];
    mbar_expect_tx(&c.bar[q], 4);
    return v;
}
}  // namespace

// ------------------------------------------------------------------------------ NK1
// One CTA = one lane tile; thread t owns VT = 2 NP adjacent local vehicles VT t .. VT t + VT - 1
// as NP float2 lane pairs (packed f32x2 arithmetic; NP = 2 by default: 128 threads per tile).
// Inside the thread a pair's second vehicle leads... its leader is the next pair's first vehicle;
// the thread's last vehicle's leader is thread t + 1's first vehicle, so one speed per thread
// crosses shared memory per step (one __syncthreads, double-buffered).  A lane head carries the
// gap +inf, which zeroes its interaction term whatever "leader" speed it reads.  Per vehicle the
// arithmetic does not depend on NP (same bits).
// All `steps` steps run in one launch, in segments of KS steps (compile-time, fully unrolled;
// the K mod KS tail runs as one predicated segment).  LOSS = 0: record P (idm_forward).
// LOSS = 1 (L1) / 2 (L2): fused Eq. 4 for idm_fit_step -- observation rows staged two segments
// ahead (cp.async ring); each step sums Eq. 4 against the fresh positions and, for L1, records
// dL/dP = -sign(obs - P) as a 4-bit code per pair-step; P and dL/dP are not written.
// LOSS = 3: fused iteration whose backward derives Eq. 4 from obs (L2 by default): only the
// tile history -- speeds, and gap + displacement checkpoints.
// CK = checkpoint interval (the backward's segment length); the forward's own prefetch
// segment is KS = max(4, CK) steps, so CK | KS and checkpoints fall at static positions.
#ifndef IDM_FWD_LOSS_MINB
#define IDM_FWD_LOSS_MINB 4  // CTAs per SM the NP = 1 fused (LOSS) forward is budgeted for
#endif
#ifndef IDM_FWD_MINB2
#define IDM_FWD_MINB2 4  // CTAs (of 128 threads) per SM the NP = 2 forward is budgeted for
#endif
// Vehicle pairs per forward thread (1: 256 threads, 2: 128 threads).  Measured at C4
// (DESIGN.md section 4): NP = 2 runs the fused forward in 1.062 against 1.102 ms and the
// prediction rollout in 0.797 against 0.820 ms, but the idm_forward that records P and the
// history in 0.904 against 0.891 ms, so that one keeps NP = 1.
#ifndef IDM_FWD_NP
#define IDM_FWD_NP 2
#endif
#ifndef IDM_FWD_NP_API
#define IDM_FWD_NP_API 1
#endif
template <int CK, int LOSS, int NP>
constexpr int fwd_min_blocks() {
    return NP == 1 ? (CK > 4 ? 2 : (LOSS ? IDM_FWD_LOSS_MINB : 4)) : (CK > 4 ? 3 : IDM_FWD_MINB2);
}
// store NP float2 of one thread (adjacent) as one access: 8 bytes (NP = 1) or 16 (NP = 2)
template <int NP>
__device__ __forceinline__ void st_pairs(float2* p, const float2 (&x)[NP]) {
    if constexpr (NP == 2) __stcs(reinterpret_cast<float4*>(p), make_float4(x[0].x, x[0].y, x[1].x, x[1].y));
    else __stcs(p, x[0]);
}
// HIST = false (LOSS = 0 only): a prediction rollout (idm_forward_ex IDM_FWD_NO_HISTORY) that
// writes only the P rows -- no speed history or checkpoints, nothing for a backward.
// The forward of lane tile a.tile0 + blockIdx.x (the body of fwd_kernel, and the forward phase
// of fit_long_kernel).
template <bool D4, bool KAHAN, bool RECV, int LOSS, int CK, bool HIST, bool CL, int NP>
__device__ __forceinline__ void fwd_tile(FwdArgs a) {
    static_assert(HIST || LOSS == 0, "the fused forward always feeds a backward");
    constexpr int VT = 2 * NP;        // vehicles per thread
    constexpr int kTf = kCap / VT;    // threads per CTA
    constexpr int KS = CK > 4 ? CK : 4;
    // LOSS = 3: the fused iteration whose backward derives Eq. 4 itself (from obs and the
    // rebuilt positions): only the tile history (speeds; gap + displacement checkpoints)
    constexpr bool OBSV = LOSS == 1 || LOSS == 2;  // reads the observations here
    constexpr bool DCK = LOSS == 2 || LOSS == 3;   // displacement checkpoints for the backward
    __shared__ float xv[2][kTf + 1];  // speed of each thread's first vehicle; [kTf] = 0 sentinel
    const int tid = threadIdx.x;
    const int tile = a.tile0 + (int)blockIdx.x;  // launches may cover a chunk of the tiles
    const int64_t base = a.tile_start[tile];
    const int n_loc = (int)(a.tile_start[tile + 1] - base);
    const Consts k = a.k;
    const int64_t N = a.n;
    const int steps = a.steps;
    const int nfull = steps / KS, tail = steps - nfull * KS;
    const int id0 = VT * tid;
    const int64_t i0 = base + id0;
    bool val[VT];
#pragma unroll
    for (int j = 0; j < VT; ++j) val[j] = id0 + j < n_loc;
    if (LOSS && a.tile_ready) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    // CL: this tile's last vehicle has a leader, the next cluster CTA's first vehicle (a lane
    // split over a cluster; the planner keeps such tiles a multiple of 4 vehicles, so the last
    // vehicle is the last one of thread n_loc / VT - 1)
    const unsigned crank = CL ? cluster_rank() : 0u;
    const bool peer_lead = CL && n_loc > 0 && n_loc % VT == 0 && a.lead[base + n_loc - 1] != 0;
    // ... and this tile's first vehicle is the previous CTA's last vehicle's leader
    const bool peer_follow = CL && base > 0 && n_loc > 0 && a.lead[base - 1] != 0;
    const int reader = peer_lead ? n_loc / VT - 1 : -1;  // the thread of the last vehicle
    // CL: the leader speed of the last vehicle arrives by a message channel each step
    __shared__ std::conditional_t<CL, ChanBuf, char> chanV;
    if constexpr (CL) {
        if (tid == reader) chan_init(chanV);
        cluster_sync_all();  // every channel armed before the first message
    }

    auto put = [&](float* row, const float2 (&x)[NP]) {  // row points at local vehicle VT tid
#pragma unroll
        for (int p = 0; p < NP; ++p) {
            st_cs_if(row + 2 * p, val[2 * p], x[p].x);
            st_cs_if(row + 2 * p + 1, val[2 * p + 1], x[p].y);
        }
    };
    // out: P row of the current step (LOSS = 0; the fused variant only sums Eq. 4)
    float* orow = LOSS ? nullptr : a.traj + i0;
    float* vrow = RECV ? a.vel_traj + i0 : nullptr;
    // tile-local state history: speed row of every step, (gap, D, compensation) every CK steps
    float2* vtp = reinterpret_cast<float2*>(a.vt + tile * a.vt_stride) + NP * tid;
    float2* ckp = reinterpret_cast<float2*>(a.ckt + tile * a.ck_stride) + NP * tid;
    constexpr int kR2 = kCap / 2;  // one row in float2 units
    const float* obs = OBSV ? a.obs + i0 : nullptr;
    const float qnan = __int_as_float(0x7fc00000);
    // LOSS: observation rows staged ahead (refilled after each segment) in a 3-buffer ring by
    // per-thread cp.async; the slots of absent vehicles hold NaN (= missing) from the start and
    // are never copied to; one commit group per segment (empty past the end) keeps
    // cp.async.wait_group<1> exact
#ifndef IDM_FWD_RING
#define IDM_FWD_RING 3  // observation ring slots (prefetch distance = slots - 1 segments)
#endif
    constexpr int OR = IDM_FWD_RING;
    __shared__ __align__(16) float obuf[OBSV ? OR : 1][OBSV ? KS : 1][kCap];
    float2 lseg[NP];  // loss of this thread's vehicles in this segment (fp32)
#pragma unroll
    for (int p = 0; p < NP; ++p) lseg[p] = f2(0.f);
    double lacc = 0.0;   // and across segments (fp64)
    // segment seg observes rows seg*KS + 1 .. seg*KS + KS; fetches run up to two segments ahead of
    // use, slots rotate 0, 1, 2 (fslot: next fetch, cslot: current use)
    const float* onext = OBSV ? obs + N : nullptr;  // first row of the next fetch
    int fslot = 0, cslot = 0;
    // pairs are 8-byte aligned in every row when the tile starts at an even vehicle, N is even
    // and the array is 8-byte aligned (CTA-uniform); a thread's 4 vehicles (NP = 2) are one
    // 16-byte block when the start and N are multiples of 4 and the array is 16-byte aligned
    const bool pair8 = OBSV && ((base | N) & 1) == 0 && ((uintptr_t)a.obs & 7) == 0;
    const bool quad16 = OBSV && NP == 2 && ((base | N) & 3) == 0 && ((uintptr_t)a.obs & 15) == 0;
    auto fetch_obs = [&](int seg) {
        const int r0 = seg * KS + 1;
        float* dst = &obuf[fslot][0][VT * tid];
        fslot = fslot == OR - 1 ? 0 : fslot + 1;
        if (r0 + KS - 1 <= steps) {  // whole segment inside the rollout (CTA-uniform)
            const float* o = onext;
            if (quad16 && val[VT - 1]) {  // the thread's 4 vehicles in one 16-byte copy (a
                                          // partial last thread takes the pair copies below)
#pragma unroll
                for (int tt = 0; tt < KS; ++tt, o += N) cp_async16_if(dst + tt * kCap, o, true);
            } else if (pair8) {  // both vehicles of a pair in one 8-byte copy (a lone last one: 4
                                 // bytes)
#pragma unroll
                for (int tt = 0; tt < KS; ++tt, o += N) {
#pragma unroll
                    for (int p = 0; p < NP; ++p) {
                        cp_async8_if(dst + tt * kCap + 2 * p, o + 2 * p, val[2 * p + 1]);
                        cp_async4_if(dst + tt * kCap + 2 * p, o + 2 * p,
                                     val[2 * p] && !val[2 * p + 1]);
                    }
                }
            } else {
#pragma unroll
                for (int tt = 0; tt < KS; ++tt, o += N) {
#pragma unroll
                    for (int j = 0; j < VT; ++j) cp_async4_if(dst + tt * kCap + j, o + j, val[j]);
                }
            }
            onext = o;
        } else {  // the tail / past the end: predicated, addresses kept inside the array
#pragma unroll
            for (int tt = 0; tt < KS; ++tt) {
                const bool on = r0 + tt <= steps;
                const float* o = on ? onext + (int64_t)tt * N : obs;
#pragma unroll
                for (int j = 0; j < VT; ++j) cp_async4_if(dst + tt * kCap + j, o + j, on && val[j]);
            }
        }
        cp_async_commit();
    };
    auto obs_at = [&](int tt, int p) {  // pair p of row seg*KS + 1 + tt (current segment)
        return *reinterpret_cast<const float2*>(&obuf[cslot][tt][VT * tid + 2 * p]);
    };
    if (OBSV) {
        float* ob = &obuf[0][0][0];
#pragma unroll
        for (int q = 0; q < OR * KS; ++q) {  // own slots only: no barrier needed
#pragma unroll
            for (int j = 0; j < VT; ++j)
                if (!val[j]) ob[q * kCap + VT * tid + j] = qnan;
        }
#pragma unroll
        for (int q = 0; q < OR - 1; ++q) fetch_obs(q);
    }
    // per-vehicle state and constants while the first observation rows are in flight
    const float pinf = __int_as_float(0x7f800000);
    float2 s[NP], v[NP], p0[NP], D[NP], cmp[NP];
    VehPT<float2> P[NP];
#pragma unroll
    for (int p = 0; p < NP; ++p) {
        float sj[2], vj[2], pj[2];
        VehP Pj[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int j = 2 * p + h;
            const int64_t i = i0 + j;
            RawP r = dummy_raw();
            sj[h] = pinf; vj[h] = 0.f; pj[h] = 0.f;  // no leader: gap +inf (see core_dv)
            if (val[j]) {
                pj[h] = a.pos0[i];
                vj[h] = a.vel0[i];
                if (a.lead[i] != 0) sj[h] = (a.pos0[i + 1] - pj[h]) - a.length[i + 1];
                r = load_raw(a.params, a.n_par, i);
                if (D4 && r.delta != 4.f)
                    atomicMin(a.status, (unsigned long long)kBadDelta << 32 | (uint64_t)i);
            }
            Pj[h] = make_vehp(r.a_max, r.a_pref, r.s_min, r.T, r.v_targ, r.delta);
        }
        s[p] = make_float2(sj[0], sj[1]);
        v[p] = make_float2(vj[0], vj[1]);
        p0[p] = make_float2(pj[0], pj[1]);
        P[p] = pack(Pj[0], Pj[1]);
        D[p] = f2(0.f);
        cmp[p] = f2(0.f);
    }
    if (tid == 0) { xv[0][kTf] = 0.f; xv[1][kTf] = 0.f; }
    // checkpoint rows the consumer reads: the gap (idm_backward); + displacement (fused
    // backward rebuilds positions); + compensation (and that with Kahan)
    auto put_ck = [&](int j) {  // checkpoint j (step j CK)
        if (!HIST) return;
        if (gap_row(j)) st_pairs<NP>(ckp, s);
        if (DCK) st_pairs<NP>(ckp + kR2, D);
        if (DCK && KAHAN) st_pairs<NP>(ckp + 2 * kR2, cmp);
    };
    // fused L1: dL/dP = -sign(obs - P) of a pair as a 4-bit code per step (bits 0 / 2: r != 0,
    // bits 1 / 3: r < 0) at bit 16 p + 4 (t mod 4), collected in a register and stored as one
    // word per 4 steps (steps 4j .. 4j + 3 -> word j): u16 per pair, so a row holds the pairs'
    // codes in vehicle order whatever NP (NP = 2 stores the thread's two as one u32)
    static_assert(LOSS != 1 || KS % kSgnSteps == 0, "code words align with segments");
    unsigned short* sgp =
        LOSS == 1 ? reinterpret_cast<unsigned short*>(a.sgn + tile * a.sg_stride) + NP * tid
                  : nullptr;
    unsigned code = 0;
    auto put_code = [&] {
        if constexpr (NP == 2) __stcs(reinterpret_cast<unsigned*>(sgp), code);
        else __stcs(sgp, (unsigned short)code);
    };
    // Eq. 4 term of the fused forward at a step t with t mod 4 = ph (compile-time): L2 sums r^2;
    // L1 sums |r| and records -sign(r) of the masked residual r (0 where unobserved), i.e.
    // exactly loss_term<0>'s dL/dP
    auto loss_step = [&](const float2 (&o)[NP], const float2 (&Pv)[NP], auto PH) {
        constexpr int ph = decltype(PH)::value;
#pragma unroll
        for (int p = 0; p < NP; ++p) {
            if (LOSS == 2) {
                (void)loss_term<1>(o[p], Pv[p], lseg[p]);
                continue;
            }
            const float2 rm = vsel(vge(vnabs(o[p]), -3.4e38f), vsub(o[p], Pv[p]), f2(0.f));
            lseg[p] = vadd(lseg[p], vabs(rm));
            const unsigned nib = (rm.x != 0.f ? 1u : 0u) | (rm.x < 0.f ? 2u : 0u) |
                                 (rm.y != 0.f ? 4u : 0u) | (rm.y < 0.f ? 8u : 0u);
            code |= nib << (16 * p + 4 * ph);
        }
        if (LOSS == 1 && ph == kSgnSteps - 1) {
            put_code();
            sgp += kCap / 2;
            code = 0;
        }
    };
    if (OBSV) {
        float2 o0[NP];
#pragma unroll
        for (int p = 0; p < NP; ++p)
            o0[p] = make_float2(ld_cs_if(obs + 2 * p, val[2 * p], qnan),
                                ld_cs_if(obs + 2 * p + 1, val[2 * p + 1], qnan));
        loss_step(o0, p0, std::integral_constant<int, 0>{});
    } else if (!LOSS) {
        put(orow, p0);
    }
    if (RECV) put(vrow, v);
    if (HIST) st_pairs<NP>(vtp, v);
    put_ck(0);
    int par = 0;
    // one synchronous step of the whole tile; o = this step's observations (LOSS)
    auto step = [&](int t, int tt, auto PH) {  // t = t0 + tt; PH: (index of the step computed) mod 4
        xv[par][tid] = v[0].x;
        if constexpr (CL) {  // the first vehicle's speed to the previous CTA's last vehicle
            if (peer_follow && tid == 0) chan_send(chanV, crank - 1, t, v[0].x);
        }
        __syncthreads();
        float nb = xv[par][tid + 1];  // the next thread's first vehicle ([kTf]: sentinel 0)
        if constexpr (CL) {
            if (tid == reader) nb = chan_recv(chanV, t);
        }
        float2 vl[NP];
#pragma unroll
        for (int p = 0; p < NP; ++p)
            vl[p] = make_float2(v[p].y, p + 1 < NP ? v[p + 1 < NP ? p + 1 : p].x : nb);
        par ^= 1;
        float2 Pv[NP];
#pragma unroll
        for (int p = 0; p < NP; ++p) {
            if (KAHAN) {  // compensated displacement for long horizons (C3)
                const float2 y = vfma(v[p], k.dt, vneg(cmp[p]));
                const float2 t2 = vadd(D[p], y);
                cmp[p] = vsub(vsub(t2, D[p]), y);
                D[p] = t2;
            } else {
                D[p] = vfma(v[p], k.dt, D[p]);
            }
            fwd_step<D4>(s[p], v[p], vl[p], P[p], k);
            Pv[p] = vadd(p0[p], D[p]);
        }
        if (!LOSS) orow += N;
        if (RECV) vrow += N;
        vtp += kR2;
        if (OBSV) {
            float2 o[NP];
#pragma unroll
            for (int p = 0; p < NP; ++p) o[p] = obs_at(tt, p);
            loss_step(o, Pv, PH);
        } else if (!LOSS) {
            put(orow, Pv);
        }
        if (HIST) st_pairs<NP>(vtp, v);
        if (RECV) put(vrow, v);
    };
    // first checkpoint step at which each vehicle's state was non-finite (INT_MAX: none); kept
    // in registers and reported once at the end, no branch or atomic per checkpoint
    int bad[VT];
#pragma unroll
    for (int j = 0; j < VT; ++j) bad[j] = INT_MAX;
    auto finite2 = [&](int t0) {  // gap: +inf is the no-leader value, only NaN is an error
#pragma unroll
        for (int p = 0; p < NP; ++p) {
            const bool ok0 = !isnan(s[p].x) && isfinite(v[p].x) && isfinite(D[p].x);
            const bool ok1 = !isnan(s[p].y) && isfinite(v[p].y) && isfinite(D[p].y);
            bad[2 * p] = (!ok0 && bad[2 * p] == INT_MAX) ? t0 : bad[2 * p];
            bad[2 * p + 1] = (!ok1 && bad[2 * p + 1] == INT_MAX) ? t0 : bad[2 * p + 1];
        }
    };
    auto checkpoint = [&](int t0) {  // (gap, D, compensation) at step t0 > 0 + finiteness check
        if (HIST) ckp += kCkRows * kR2;
        put_ck(t0 / CK);
        finite2(t0);
    };
    auto obs_ready = [&](int seg) {
        if (OBSV) {
            cp_async_wait<OR - 2>();  // this segment's group; later ones may stay in flight
        }
    };
    auto obs_done = [&] { cslot = cslot == OR - 1 ? 0 : cslot + 1; };
    auto fold_loss = [&] {
#pragma unroll
        for (int p = 0; p < NP; ++p) {
            lacc += (double)lseg[p].x + (double)lseg[p].y;
            lseg[p] = f2(0.f);
        }
    };
    for (int seg = 0; seg < nfull; ++seg) {
        const int t0 = seg * KS;
        obs_ready(seg);
        static_for<KS>([&](auto TT) {
            constexpr int tt = decltype(TT)::value;
            if (tt % CK == 0 && (tt > 0 || seg > 0)) checkpoint(t0 + tt);
            step(t0 + tt, tt, std::integral_constant<int, (tt + 1) % 4>{});
        });
        // CL: the channel's flow-control window (kChanQ steps, a multiple of KS)
        if (CL && (t0 + KS) % kChanQ == 0) cluster_sync_all();
        obs_done();
        if (OBSV) fold_loss();
        // refill after the segment's steps (its reads of the refilled slot are long done)
        if (OBSV) fetch_obs(seg + OR - 1);
    }
    if (tail > 0) {
        obs_ready(nfull);
        static_for<KS>([&](auto TT) {
            constexpr int tt = decltype(TT)::value;
            if (tt < tail) {  // CTA-uniform predicate
                if (tt % CK == 0 && (tt > 0 || nfull > 0)) checkpoint(nfull * KS + tt);
                step(nfull * KS + tt, tt, std::integral_constant<int, (tt + 1) % 4>{});
            }
        });
    }
    if (OBSV) cp_async_wait<0>();  // no copy outlives the CTA
    if (LOSS == 1 && steps % kSgnSteps != kSgnSteps - 1)
        put_code();  // the last, partial code word (holds step K)
    if (HIST)  // the final gap s_K: the backward's reverse gap recurrence starts from it
        st_pairs<NP>(reinterpret_cast<float2*>(a.ckt + tile * a.ck_stride +
                                               (int64_t)((steps + CK - 1) / CK) * kCkRows * kCap) +
                         NP * tid,
                     s);
    finite2(steps);
#pragma unroll
    for (int j = 0; j < VT; ++j)
        if (val[j] && bad[j] != INT_MAX) report_nonfinite(a.status, bad[j], i0 + j);
    if (a.state_out) {
        float2 pe[NP];
#pragma unroll
        for (int p = 0; p < NP; ++p) pe[p] = vadd(p0[p], D[p]);
        put(a.state_out + i0, pe);
        put(a.state_out + N + i0, v);
    }
    if (OBSV) {
        fold_loss();
        block_sum_to<kTf>(lacc, a.loss_partials + tile);
    }
    if (OBSV && a.loss_out) {  // the step's Eq. 4 loss, summed by the last CTA to finish
        bool mine = false;
        if (tid == 0) {
            __threadfence();  // this tile's partial precedes its ticket
            mine = atomicAdd(a.done_count, 1u) == (unsigned)(a.n_tiles - 1);
        }
        if (__syncthreads_or(mine)) {
            __threadfence();
            // reduce_kernel's order: 256 strided per-thread sums, then a fixed tree (each of
            // the kTf threads forms VT / 2 of the 256 sums)
            constexpr int kR = 256;
            double* lred = reinterpret_cast<double*>(&obuf[0][0][0]);  // the ring is idle now
#pragma unroll
            for (int w = tid; w < kR; w += kTf) {
                double x = 0.0;
                for (int r = w; r < a.n_tiles; r += kR) x += __ldcg(a.loss_partials + r);
                lred[w] = x;
            }
            __syncthreads();
            for (int st = kR / 2; st > 0; st >>= 1) {
                for (int w = tid; w < st; w += kTf) lred[w] += lred[w + st];
                __syncthreads();
            }
            if (tid == 0) {
                *a.loss_out = lred[0];
                *a.done_count = 0u;
            }
        }
    }
    if (LOSS && a.tile_ready) tile_release(a.tile_ready + tile, a.epoch);
    if (CL) cluster_sync_all();  // no CTA leaves while a peer may still read its shared memory
}

template <bool D4, bool KAHAN, bool RECV, int LOSS, int CK, bool HIST = true, bool CL = false,
          int NP = (LOSS == 0 && HIST ? IDM_FWD_NP_API : IDM_FWD_NP)>
__global__ void __launch_bounds__(kCap / (2 * NP), (fwd_min_blocks<CK, LOSS, NP>()))
    fwd_kernel(FwdArgs a) {
    fwd_tile<D4, KAHAN, RECV, LOSS, CK, HIST, CL, NP>(a);
}

// ------------------------------------------------------------------------------ NK3
// Per CTA (lane tile), segments of KS steps from last to first.  Thread t owns VT = 2 NP
// adjacent vehicles VT t .. VT t + VT - 1 as NP float2 lane pairs (packed f32x2 arithmetic;
// NP = 2 by default: 128 threads per 512-vehicle tile, so the per-step exchange, barrier and
// bookkeeping are paid once per 4 vehicles and every warp carries two independent adjoint
// chains).  The forward stored every vehicle's speed at every step and (gap, displacement,
// compensation) at every KS-th step in the tile-local rows, so nothing here is a long serial
// chain: inside a segment the displacements follow from the checkpoint by the forward's own
// one-FMA recurrence (bit-identical) and the gaps from the later segment's by the reverse one
// (re-anchored on the stored gap every kGapCk segments), every step's local Jacobian (core +
// jac_record) depends only on stored state, and the one sequential dependency left is the
// adjoint itself -- lambda^{t+1} -> lambda^t plus the follower -> leader term F of the
// thread's last vehicle, passed to thread t + 1 through shared memory (one barrier per step;
// inside the thread the terms pass in registers).  Per vehicle the arithmetic and its order do
// not depend on NP, so every NP gives the same bits.
//   GOBS = 0:      dL/dP rows from grad_traj (idm_backward after idm_loss_grad);
//   GOBS = 1:      fused idm_fit_step, L1 -- dL/dP = -sign(obs - P) from the forward's sign
//                  codes (2 bits per vehicle-step);
//   GOBS = 2 / 3:  fused idm_fit_step, L2 / L1 -- dL/dP re-derived from obs and the rebuilt
//                  positions P = p0 + D with the loss kernel's term (same bits as idm_loss_grad);
//                  with loss_partials set, this tile's Eq. 4 loss as well (LOSS = 3 forward).
// Gradient accumulators stay in registers for the whole rollout; ADAM: per-vehicle Adam in the
// epilogue (idm_fit_step).
#ifndef IDM_BWD_MINB
#define IDM_BWD_MINB 2  // CTAs per SM the NP = 1 backward is register-budgeted for (128 regs)
#endif
#ifndef IDM_BWD_MINB2
#define IDM_BWD_MINB2 3  // CTAs (of 128 threads) per SM the NP = 2 backward is budgeted for
#endif
template <int KS, int NP>
constexpr int bwd_min_blocks() {
    return NP == 1 ? (KS <= 4 ? IDM_BWD_MINB : 1) : (KS <= 4 ? IDM_BWD_MINB2 : 1);
}
// The backward of lane tile a.tile0 + blockIdx.x (the body of bwd_kernel, and the backward phase
// of fit_long_kernel).
template <bool D4, bool SHARED, bool ADAM, int KS, int GOBS, bool KAHAN, bool CL, int NP>
__device__ __forceinline__ void bwd_tile(const BwdArgs& a) {
    constexpr int VT = 2 * NP;          // vehicles per thread
    constexpr int kTb = kCap / VT;      // threads per CTA
    __shared__ float fx[2][kTb + 1];
    const int tid = threadIdx.x;
    const int tile = a.tile0 + (int)blockIdx.x;  // launches may cover a chunk of the tiles
    const int64_t base = a.tile_start[tile];
    const int n_loc = (int)(a.tile_start[tile + 1] - base);
    const Consts k = a.k;
    const int64_t N = a.n;
    const int steps = a.steps;
    const int id0 = VT * tid;
    const int64_t i0 = base + id0;
    bool val[VT];
#pragma unroll
    for (int j = 0; j < VT; ++j) val[j] = id0 + j < n_loc;
    // CL (a lane longer than a tile over a cluster): the last vehicle's leader is the next CTA's
    // first vehicle; the first vehicle's follower is the previous CTA's last vehicle
    const unsigned crank = CL ? cluster_rank() : 0u;
    const bool peer_lead = CL && n_loc > 0 && n_loc % VT == 0 && a.lead[base + n_loc - 1] != 0;
    const bool peer_follow = CL && base > 0 && n_loc > 0 && a.lead[base - 1] != 0;
    // the previous CTA's last vehicle writes its term to its fx[par][n_prev / VT]
    const int pslot = peer_follow ? (int)(base - a.tile_start[tile - 1]) / VT : 0;
    const int reader = peer_lead ? n_loc / VT - 1 : -1;  // the thread of the last vehicle
    // CL: the follower -> leader adjoint term crosses to the next CTA by a message channel
    __shared__ std::conditional_t<CL, ChanBuf, char> chanF;
    const int nseg = (steps + KS - 1) / KS;
    const int tail = steps - (nseg - 1) * KS;  // length of the last segment (1..KS)

    // Segment rows are staged in shared memory, one to two segments ahead, in a ring of 3
    // buffers (each refill is issued at the end of a segment):
    // speeds and the checkpoint by bulk copy (one thread, mbarrier-counted), dL/dP rows (or the
    // observation rows, plus one for the rollout's last step) by per-thread cp.async.  No
    // register holds data in flight.
    extern __shared__ __align__(16) float smem_b[];
#ifndef IDM_BWD_RING
#define IDM_BWD_RING 3  // staging ring buffers of the backward (rows NB - 1 segments ahead)
#endif
    constexpr int NB = IDM_BWD_RING;
    constexpr int VP = kCap + 4;  // speed row pitch: [kCap] = 0 is the leader read of slot 511
    constexpr bool SGN = GOBS == 1, OBS = GOBS >= 2;
    constexpr int OKIND = GOBS == 3 ? 0 : 1;  // OBS: Eq. 4 as L1 (GOBS 3) or L2 (GOBS 2)
    constexpr int kSW = kCap / 2;             // u16 sign-code words per tile row (per 4 steps)
    double lacc = 0.0;  // OBS: this thread's Eq. 4 terms (fp32 per segment, fp64 across)
    // fused iteration with delta frozen at 4: dL/d delta is not computed (row 5 written as 0)
    constexpr bool GD = !(D4 && GOBS != 0);
    constexpr int KO = GOBS ? KS + 1 : KS;             // + the rollout's last step (fused)
    float* vrow = smem_b;                              // [NB][KS][VP]
    float* ckrow = vrow + NB * KS * VP;                // [NB][3][kCap]
    float* orow = ckrow + NB * kCkRows * kCap;         // [NB][KO][kCap] (dL/dP or obs rows)
    // SGN: [NB][2][kSW] u16 code words (the segment's steps; + the next word, which holds step
    // K when the last segment is a whole one) and the 16-entry decode table code -> dL/dP pair.
    // Word w of a row is the code of vehicles 2w, 2w + 1, so a thread's NP words are adjacent.
    unsigned short* sbuf = reinterpret_cast<unsigned short*>(orow);
    __shared__ float2 glut[16];
    if (SGN && tid < 16) {
        auto gv = [](unsigned nz, unsigned neg) { return nz ? (neg ? 1.f : -1.f) : 0.f; };
        glut[tid] = make_float2(gv(tid & 1u, tid & 2u), gv(tid & 4u, tid & 8u));
    }
    __shared__ __align__(8) uint64_t mbar[NB];
    constexpr int nckr = OBS ? (KAHAN ? 3 : 2) : 1;    // checkpoint rows used
    if (tid == 0) {
#pragma unroll
        for (int q = 0; q < NB; ++q) mbar_init(&mbar[q], 1);
        mbar_fence_init();
        // fused step after a programmatic launch: the tile's history is complete
        if (GOBS && a.tile_ready) tile_acquire(a.tile_ready + tile, a.epoch, a.steps);
    }
    if (tid < NB * KS) vrow[tid * VP + kCap] = 0.f;
    if constexpr (CL) {
        if (peer_follow && tid == 0) chan_init(chanF);
        cluster_sync_all();  // every channel armed before the first message
    } else {
        __syncthreads();
    }
    uint32_t phase = 0;  // bit q: parity of buffer q's next completion
    auto fetch = [&](int seg, int len) {
        const int b = seg % NB;
        const int64_t t0 = (int64_t)seg * KS;
        if (tid == 0) {
            // buffer b was last read (generic proxy) before the barriers of an earlier
            // segment; order those reads before the async-proxy writes
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            // SGN: code word seg, + word seg + 1 (step K) when the last segment is whole
            const int swords = (seg == nseg - 1 && len == KS) ? 2 : 1;
            // CL: the last vehicle's leader is the next tile's first vehicle: the speed row
            // holds this tile's n_loc vehicles, then 16 bytes of the next tile's row (slot n_loc,
            // where the last vehicle reads its leader; 16-byte aligned: n_loc is a multiple of 4)
            const uint32_t vrow_b = (uint32_t)(peer_lead ? n_loc : kCap) * sizeof(float);
            // checkpoint rows: the gap row only where the forward wrote it (gap_row)
            const int ck0 = gap_row(seg) ? 0 : 1;
            const uint32_t bytes = (uint32_t)len * (vrow_b + (peer_lead ? 16u : 0u)) +
                                   (uint32_t)(nckr - ck0) * kCap * sizeof(float) +
                                   (SGN ? (uint32_t)swords * kSW * sizeof(unsigned short) : 0u);
            mbar_expect_tx(&mbar[b], bytes);
            if (SGN)
                bulk_g2s(sbuf + b * 2 * kSW,
                         reinterpret_cast<const unsigned short*>(a.sgn + tile * a.sg_stride) +
                             (int64_t)seg * kSW,
                         swords * kSW * sizeof(unsigned short), &mbar[b]);
            const float* src = a.vt + tile * a.vt_stride + t0 * kCap;
            for (int tt = 0; tt < len; ++tt) {
                bulk_g2s(vrow + (b * KS + tt) * VP, src + tt * kCap, vrow_b, &mbar[b]);
                if (CL && peer_lead)
                    bulk_g2s(vrow + (b * KS + tt) * VP + n_loc, src + a.vt_stride + tt * kCap, 16u,
                             &mbar[b]);
            }
            if (nckr > ck0)
                bulk_g2s(ckrow + (b * kCkRows + ck0) * kCap,
                         a.ckt + tile * a.ck_stride + ((int64_t)seg * kCkRows + ck0) * kCap,
                         (nckr - ck0) * kCap * sizeof(float), &mbar[b]);
        }
        if (!SGN) {
            const float* src = (OBS ? a.obs : a.grad_traj) + t0 * N + i0;
            float* dst = orow + b * KO * kCap + VT * tid;
#pragma unroll
            for (int tt = 0; tt < KO; ++tt, src += N) {
                const bool on = tt < len || (OBS && tt == len && seg == nseg - 1);
#pragma unroll
                for (int j = 0; j < VT; ++j) cp_async4(dst + tt * kCap + j, src + j, val[j] && on);
            }
            cp_async_commit();
        }
    };
    int par = 0;
    fetch(nseg - 1, tail);
#pragma unroll
    for (int q = 2; q <= NB - 1; ++q)
        if (nseg >= q) fetch(nseg - q, KS);
    // per-vehicle constants while the first two segments' rows are in flight
    float ldj[VT], pj[VT];
    VehPT<float2> P[NP];
    VehAT<float2> B[NP];
    float2 p0[NP], e[NP], m[NP], u[NP], sc[NP];
    GradAccT<float2> G[NP];
#pragma unroll
    for (int p = 0; p < NP; ++p) {
        VehP Pj[2];
        VehA Aj[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int j = 2 * p + h;
            const int64_t i = i0 + j;
            RawP r = dummy_raw();
            ldj[j] = 0.f;
            pj[j] = 0.f;
            if (val[j]) {
                r = load_raw(a.params, a.n_par, i);
                if (D4 && r.delta != 4.f)
                    atomicMin(a.status, (unsigned long long)kBadDelta << 32 | (uint64_t)i);
                if (!GOBS) ldj[j] = a.grad_traj[(int64_t)steps * N + i];  // lambda_D^K = dL/dP(K)
                if (GOBS >= 2) pj[j] = a.pos0[i];
            }
            Pj[h] = make_vehp(r.a_max, r.a_pref, r.s_min, r.T, r.v_targ, r.delta);
            Aj[h] = make_veha(r.a_max, r.a_pref, r.v_targ, r.delta, k);
        }
        p0[p] = make_float2(pj[2 * p], pj[2 * p + 1]);
        P[p] = pack(Pj[0], Pj[1]);
        B[p] = pack(Aj[0], Aj[1]);
        // scaled adjoint (bwd_from_record): u = dt lambda_v, m = -dt lambda_s, e = dt^2 lambda_D
        e[p] = vmul(make_float2(ldj[2 * p], ldj[2 * p + 1]), k.dt2);
        m[p] = f2(0.f);
        u[p] = f2(0.f);
        // the final gap s_K (written by the forward one row past the last segment's; L2 load:
        // after the handoff / the whole-fit barrier, an L1 line of an earlier iteration is stale)
        sc[p] = __ldcg(reinterpret_cast<const float2*>(a.ckt + tile * a.ck_stride +
                                                       (int64_t)nseg * kCkRows * kCap) +
                       NP * tid + p);
        G[p] = GradAccT<float2>{f2(0.f), f2(0.f), f2(0.f), f2(0.f), f2(0.f), f2(0.f)};
    }
    if (tid == 0) { fx[0][0] = 0.f; fx[1][0] = 0.f; }  // never written again (slots t+1 >= 1)
    auto segment = [&](const int seg, const int len, auto FULL) {
        constexpr bool kFull = decltype(FULL)::value;
        const int b = seg % NB;
        mbar_wait(&mbar[b], (phase >> b) & 1u);
        phase ^= 1u << b;
        if (!SGN) {
            // this segment's rows; the (up to NB - 2) later segments' may stay in flight
            if (NB >= 4 && seg >= 2) cp_async_wait<(NB >= 4 ? 2 : 1)>();
            else if (seg >= 1) cp_async_wait<1>();
            else cp_async_wait<0>();
        }
        const float* orr = orow + b * KO * kCap + VT * tid;
        float2 v[KS][NP], g[KO][NP], vl[KS][NP], sg[KS][NP];
        const float* vr = vrow + b * KS * VP + VT * tid;
#pragma unroll
        for (int tt = 0; tt < KS; ++tt) {
#pragma unroll
            for (int p = 0; p < NP; ++p) {
                if (kFull || tt < len) {
                    v[tt][p] = *reinterpret_cast<const float2*>(vr + tt * VP + 2 * p);
                    // the leader of the pair's second vehicle: the next pair's first, or the
                    // next thread's first vehicle (slot kCap: the 0 sentinel; CL: slot n_loc
                    // holds the next tile's first vehicle)
                    vl[tt][p] = make_float2(v[tt][p].y, vr[tt * VP + 2 * p + 2]);
                } else {
                    v[tt][p] = f2(0.f);
                    vl[tt][p] = f2(0.f);
                }
            }
        }
        unsigned cw0 = 0, cw1 = 0;  // SGN: this thread's code words (steps t0 .. t0 + 4)
        if (SGN) {
            static_assert(!SGN || KS == kSgnSteps, "one code word per segment");
            if (NP == 1) {
                cw0 = sbuf[b * 2 * kSW + tid];
                if (seg == nseg - 1 && len == KS) cw1 = sbuf[b * 2 * kSW + kSW + tid];
            } else {  // NP = 2: the two adjacent u16 words as one u32 (pair p at bit 16 p)
                cw0 = reinterpret_cast<const unsigned*>(sbuf + b * 2 * kSW)[tid];
                if (seg == nseg - 1 && len == KS)
                    cw1 = reinterpret_cast<const unsigned*>(sbuf + b * 2 * kSW + kSW)[tid];
            }
        }
#pragma unroll
        for (int tt = 0; tt < KO; ++tt) {
#pragma unroll
            for (int p = 0; p < NP; ++p) {
                if (SGN) {  // -sign(obs - P) of the pair's two vehicles: 4-bit code -> table
                    const unsigned c = ((tt < KS ? cw0 : cw1) >> (16 * p + 4 * (tt % KS))) & 15u;
                    g[tt][p] = (kFull || tt <= len) ? glut[c] : f2(0.f);
                } else {
                    g[tt][p] = (kFull || tt <= len)
                                   ? *reinterpret_cast<const float2*>(orr + tt * kCap + 2 * p)
                                   : f2(0.f);
                }
            }
        }
        // positions inside the segment (OBS): the forward's recurrence from the checkpoint,
        // bitwise; gaps: the reverse recurrence from the later segment's first gap sc (s_K for
        // the last), the segment's first gap replaced by the exact row where there is one
        const float* cr = ckrow + b * kCkRows * kCap + VT * tid;
        const bool ck_gap = gap_row(seg);  // CTA-uniform
#pragma unroll
        for (int p = 0; p < NP; ++p) {
            float2 D = f2(0.f), cmp = f2(0.f), lsum = f2(0.f);
            if (OBS) D = *reinterpret_cast<const float2*>(cr + kCap + 2 * p);
            if (OBS && KAHAN) cmp = *reinterpret_cast<const float2*>(cr + 2 * kCap + 2 * p);
#pragma unroll
            for (int tt = 0; tt < KO; ++tt) {
                if (OBS) {
                    // dL/dP at step t0 + tt (the forward's loss term on the same P bits); the
                    // rollout's last step K adds its term to lambda_D^K below.  Each row's Eq. 4
                    // term is counted once: rows t0 .. t0 + len - 1, and row K in the last
                    // segment
                    float2 lt = f2(0.f);
                    if (kFull || tt <= len) g[tt][p] = loss_term<OKIND>(g[tt][p], vadd(p0[p], D), lt);
                    if (tt < len || (tt == len && seg == nseg - 1)) lsum = vadd(lsum, lt);
                }
                if (tt < KS) {
                    if (kFull || tt < len) {
                        if (OBS) {
                            if (KAHAN) {
                                const float2 y = vfma(v[tt][p], k.dt, vneg(cmp));
                                const float2 t2 = vadd(D, y);
                                cmp = vsub(vsub(t2, D), y);
                                D = t2;
                            } else {
                                D = vfma(v[tt][p], k.dt, D);
                            }
                        }
                    }
                }
            }
            if (OBS) {  // absent vehicles' slots are zero-filled, not NaN: their terms drop here
                lacc += (val[2 * p] ? (double)lsum.x : 0.0) +
                        (val[2 * p + 1] ? (double)lsum.y : 0.0);
            }
            float2 sr = sc[p];  // s_t = s_{t+1} + dt (v_t - v_h,t), t = t0 + len - 1 .. t0
#pragma unroll
            for (int tt = KS - 1; tt >= 0; --tt) {
                if (kFull || tt < len) sr = vfma(vsub(v[tt][p], vl[tt][p]), k.dt, sr);
                sg[tt][p] = sr;
            }
            if (ck_gap) sg[0][p] = *reinterpret_cast<const float2*>(cr + 2 * p);
            sc[p] = sg[0][p];  // this segment's first gap, for the segment before it
        }
        if (GOBS && seg == nseg - 1) {  // lambda_D^K = dL/dP(K) (static selects, no indexing)
#pragma unroll
            for (int tt = 0; tt < KO; ++tt)
                if (tt == len)
#pragma unroll
                    for (int p = 0; p < NP; ++p) e[p] = vmul(g[tt][p], k.dt2);
        }
        // reverse sweep t = t0 + len - 1 ... t0; the local Jacobians of the next step down are
        // independent of the adjoint chain, so the scheduler overlaps them with this one
#pragma unroll
        for (int tt = KS - 1; tt >= 0; --tt) {
            if (kFull || tt < len) {  // CTA-uniform
                float2 F[NP];
#pragma unroll
                for (int p = 0; p < NP; ++p) {
                    CoreT<float2> c;
                    core<D4>(sg[tt][p], v[tt][p], vl[tt][p], P[p], k, c);
                    const RecT<float2> R = jac_record<D4, GD>(c, sg[tt][p], v[tt][p], P[p], B[p], k);
                    F[p] = bwd_from_record<D4, GD>(R, v[tt][p], vl[tt][p], P[p], B[p], k, m[p],
                                                   u[p], e[p], G[p]);
                }
                // the thread's last vehicle -> its leader, thread t + 1's first vehicle
                fx[par][tid + 1] = F[NP - 1].y;
                // CL: message seq of the reverse sweep (steps done before this one)
                const int seq = steps - 1 - (seg * KS + tt);
                (void)seq;
                if constexpr (CL) {  // the tile's last vehicle -> the next CTA's first
                    if (tid == reader) chan_send(chanF, crank + 1, seq, F[NP - 1].y);
                }
                // in-thread follower terms and lambda_D^t = g^t + lambda_D^{t+1} need no barrier
#pragma unroll
                for (int p = 1; p < NP; ++p) u[p] = vadd(u[p], make_float2(F[p - 1].y, F[p].x));
#pragma unroll
                for (int p = 0; p < NP; ++p) e[p] = vfma(g[tt][p], k.dt2, e[p]);
                __syncthreads();
                // F of the first vehicle's follower: thread t - 1's last vehicle
                float ff = fx[par][tid];
                if constexpr (CL) {
                    if (peer_follow && tid == 0) ff = chan_recv(chanF, seq);
                    if (seq % kChanQ == kChanQ - 1) cluster_sync_all();  // flow-control window
                }
                u[0] = vadd(u[0], make_float2(ff, F[0].x));
                par ^= 1;
            }
        }
        // refill the ring after the sweep: the elected thread's bulk-copy issue (~20
        // instructions) sits off the first step's barrier, where it held every warp
        // (backward 1.61 -> 1.51 ms); the rows still arrive a segment ahead of their use
        if (seg > NB - 2) fetch(seg - (NB - 1), KS);
    };
    int seg = nseg - 1;
    if (tail < KS) segment(seg--, tail, std::false_type{});
    for (; seg >= 0; --seg) segment(seg, KS, std::true_type{});
    // dL/dp0_i = lambda_D - lambda_s_i + lambda_s_{follower}; dL/dv0 = lambda_v (unscaled)
    fx[par][tid + 1] = m[NP - 1].y;
    step_sync<CL>();
    float mpeer = fx[par][tid];
    if (CL && peer_follow && tid == 0) mpeer = ld_peer(&fx[par][pslot], crank - 1);
    float gpj[VT], lvj[VT], Sj[6][VT];
#pragma unroll
    for (int p = 0; p < NP; ++p) {
        const float mf0 = p == 0 ? mpeer : m[p - 1].y;
        const float2 gp0 = grad_p0(e[p], m[p], make_float2(mf0, m[p].x), k);
        const float2 gv0 = grad_v0(u[p], k);
        gpj[2 * p] = gp0.x;
        gpj[2 * p + 1] = gp0.y;
        lvj[2 * p] = gv0.x;
        lvj[2 * p + 1] = gv0.y;
        // parameter gradients from the factored accumulators
        unscale_acc(G[p], k);
        const float2 Sp[6] = {G[p].S1, G[p].S2, G[p].S3, G[p].S4, G[p].S5, G[p].S6};
#pragma unroll
        for (int q = 0; q < 6; ++q) {
            Sj[q][2 * p] = Sp[q].x;
            Sj[q][2 * p + 1] = Sp[q].y;
        }
    }
    float gr[VT][6];
#pragma unroll
    for (int j = 0; j < VT; ++j) {
#pragma unroll
        for (int q = 0; q < 6; ++q) gr[j][q] = 0.f;
        if (!val[j]) continue;
        const int64_t i = i0 + j;
        const RawP r = load_raw(a.params, a.n_par, i);
        const float rr[6] = {r.a_max, r.a_pref, r.s_min, r.T, r.v_targ, r.delta};
        const float Sv[6] = {Sj[0][j], Sj[1][j], Sj[2][j], Sj[3][j], Sj[4][j], Sj[5][j]};
        param_grads(rr, Sv, gr[j]);
        if (GOBS && !((a.adam.opt_mask >> 5) & 1u)) gr[j][5] = 0.f;  // delta frozen: not computed
        if (a.grad_state0) {
            a.grad_state0[i] = gpj[j];
            a.grad_state0[N + i] = lvj[j];
        }
        if (!(isfinite(lvj[j]) && isfinite(gpj[j]))) report_nonfinite(a.status, 0, i);
    }
    if (!SHARED) {
#pragma unroll
        for (int j = 0; j < VT; ++j) {
            if (!val[j]) continue;
            const int64_t i = i0 + j;
            int bq = -1;  // first optimised parameter with a non-finite gradient
#pragma unroll
            for (int q = 0; q < 6; ++q) {
                a.grad_params[q * N + i] = gr[j][q];
                // fused iteration: Adam on this vehicle's parameters right here (idm_fit_step)
                if (ADAM && ((a.adam.opt_mask >> q) & 1u)) {
                    if (bq < 0 && !isfinite(gr[j][q])) bq = q;
                    adam_update(a.adam, q, q * N + i, gr[j][q]);
                }
            }
            if (ADAM && bq >= 0) report_bad_grad(a.status, bq * N + i);
        }
    } else {
        // Per-LANE fp64 sums in vehicle order -> lane_grads[lane][6]: a lane is whole on every
        // rank and in every tile plan, so these rows (and their fixed-order sum over the global
        // lane index, idm_reduce_shared) do not depend on the tiling or the sharding.  The
        // staging ring is idle after the sweep (the barrier above ordered its last reads).
        double* vg = reinterpret_cast<double*>(smem_b);  // [kCap][6]
#pragma unroll
        for (int j = 0; j < VT; ++j)
#pragma unroll
            for (int q = 0; q < 6; ++q) vg[(id0 + j) * 6 + q] = (double)gr[j][q];
        step_sync<CL>();  // CL: a lane's later vehicles sit in the next CTAs' vg
#pragma unroll
        for (int j = 0; j < VT; ++j) {
            const int li = id0 + j;
            if (!val[j] || (li == 0 && peer_follow) || !(li == 0 || a.lead[base + li - 1] == 0))
                continue;  // lane starts (a lane split over CTAs is summed by its first one)
            double acc[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
            // the lane's vehicles up to its head (no leader); a lane split over a cluster
            // continues in CTAs crank + c, whose vehicles start at tile_start[tile + c]
            int c = 0, e = li, nc = n_loc;
            for (int64_t gi = base + li;; ++gi, ++e) {
                if (CL && e == nc) {
                    ++c;
                    e = 0;
                    nc = (int)(a.tile_start[tile + c + 1] - a.tile_start[tile + c]);
                }
                if (!CL || c == 0) {
#pragma unroll
                    for (int q = 0; q < 6; ++q) acc[q] += vg[e * 6 + q];
                } else {
#pragma unroll
                    for (int q = 0; q < 6; ++q) acc[q] += ld_peer(vg + e * 6 + q, crank + c);
                }
                if (a.lead[gi] == 0) break;
            }
            // lane index: the last l with lane_offsets[l] <= i (empty lanes skipped)
            const int64_t gi = base + li;
            int lo = 0, hi = a.n_lanes;  // lane_offsets[lo] <= gi < lane_offsets[hi]
            while (hi - lo > 1) {
                const int mid = (lo + hi) >> 1;
                if (a.lane_offsets[mid] <= gi) lo = mid;
                else hi = mid;
            }
#pragma unroll
            for (int q = 0; q < 6; ++q) a.lane_grads[(int64_t)lo * 6 + q] = acc[q];
        }
    }
    if (OBS && a.loss_partials) block_sum_to<kTb>(lacc, a.loss_partials + tile);  // Eq. 4 here
    if (CL) cluster_sync_all();  // no CTA leaves while a peer may still read its shared memory
}

template <bool D4, bool SHARED, bool ADAM, int KS, int GOBS, bool KAHAN, bool CL, int NP>
__global__ void __launch_bounds__(kCap / (2 * NP), (bwd_min_blocks<KS, NP>()))
    bwd_kernel(const __grid_constant__ BwdArgs a) {
    // How the argument block reaches the body changes the code around the staging: the
    // single-CTA observation variants read it in place (L2 fused backward 2.00 -> 1.82 ms), the
    // others from a copy (fused L1 backward 1.48 -> 1.42 ms, C4L 3.61 -> 3.57 ms; same-box A/B,
    // DESIGN.md section 4)
    if constexpr (GOBS >= 2 && !CL) {
        bwd_tile<D4, SHARED, ADAM, KS, GOBS, KAHAN, CL, NP>(a);
    } else {
        const BwdArgs c = a;
        bwd_tile<D4, SHARED, ADAM, KS, GOBS, KAHAN, CL, NP>(c);
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
// Sums `n` rows of `width` fp64 partials in fixed order (per thread strided, then a fixed tree;
// a function of n only); out_f (nullable) gets a float copy.  Block b sums column b.
__global__ void reduce_kernel(const double* __restrict__ partials, int64_t n, int width,
                              double* __restrict__ out, float* __restrict__ out_f) {
    __shared__ double red[256];
    {
        const int c = blockIdx.x;
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
    }
}

// ------------------------------------------------------------------------------ NK5
__global__ void __launch_bounds__(256) adam_kernel(AdamArgs a) {
    const int64_t m = 6 * a.n_par;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < m;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int q = (int)(e / a.n_par);
        if ((a.opt_mask >> q) & 1u) {
            const float g = a.grad[e];
            if (!isfinite(g)) report_bad_grad(a.status, e);
            adam_update(a, q, e, g);
        }
    }
}

// ------------------------------------------------------------------------------ NK6
// Initial state of a fit from its observations ("p(0) and v(0) ... set to 0 and
// (Delta P) / Delta t, where Delta P is the distance between the first two data points"; R#13):
// per vehicle the first two observed rows t1 < t2 of the step-major [(steps+1)][N] array (NaN
// = missing) give v0 = max(0, (P_t2 - P_t1) / ((t2 - t1) dt)) and p0 = P_t1 - t1 dt v0 (the
// first data point carried back to step 0 at that speed; = P_t1 when t1 = 0).  One observation:
// v0 = 0, p0 = P_t1; none: 0, 0.  Coalesced: thread i reads column i row by row.
__global__ void state_from_obs_kernel(const float* __restrict__ obs, int64_t n, int steps,
                                      float dt, float* __restrict__ pos0,
                                      float* __restrict__ vel0) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        int t1 = -1, t2 = -1;
        float o1 = 0.f, o2 = 0.f;
        for (int t = 0; t <= steps; ++t) {
            const float o = __ldcs(obs + (int64_t)t * n + i);
            if (!isfinite(o)) continue;
            if (t1 < 0) {
                t1 = t;
                o1 = o;
            } else {
                t2 = t;
                o2 = o;
                break;
            }
        }
        float v = 0.f, p = 0.f;
        if (t2 >= 0) v = fmaxf(0.f, __fdiv_rn(__fsub_rn(o2, o1), __fmul_rn((float)(t2 - t1), dt)));
        if (t1 >= 0) p = __fsub_rn(o1, __fmul_rn(__fmul_rn((float)t1, dt), v));
        pos0[i] = p;
        vel0[i] = v;
    }
}

template <int KS, int GOBS>
constexpr size_t bwd_smem_of() {  // ring of NB: speed + checkpoint + dL/dP/obs (or sign) rows
    return (size_t)IDM_BWD_RING *
           (KS * (kCap + 4) + kCkRows * kCap +
            (GOBS == 1 ? kCap / 2 : (GOBS ? KS + 1 : KS) * kCap)) *
           sizeof(float);
}

// ------------------------------------------------------------------------------ NK7
// NEXT-4, any horizon: iterations it0 .. it0 + iters - 1 of the fused iteration in ONE launch.
// Lane tiles are independent across iterations too -- tile j's next forward needs only tile
// j's parameters, which its own backward's Adam epilogue wrote -- so each CTA runs its tile's
// whole fit: fused forward (Eq. 4 in-kernel), then the backward with Adam, iters times, with
// no grid-wide synchronisation.  The state history still goes through memory (K = 300 does not
// fit on chip), but it is re-read by the same CTA right after it was
// written, and the two resident CTAs of an SM drift into different phases, so the HBM-bound
// forward of one overlaps the FP32-bound backward of the other.  Same device code and the same
// per-vehicle order as idm_fit_step (fwd_tile / bwd_tile, one vehicle pair per thread in both):
// parameters, moments and gradients are bit-identical to the loop of idm_fit_step calls.
//   L1 (KIND 0): forward with sign codes (LOSS 1) -> backward from the codes (GOBS 1);
//   L2 (KIND 1): history-only forward (LOSS 3) -> backward deriving Eq. 4 from obs (GOBS 2).
// The Eq. 4 loss of the last iteration: L1 summed by the forward's last CTA, L2 as per-tile
// partials from the backward (reduce_kernel after the launch).
template <bool D4, bool KAHAN, int KIND>
__global__ void __launch_bounds__(kT, 2) fit_long_kernel(FwdArgs af, BwdArgs ab, FitLongArgs fl) {
    double* const loss_out = af.loss_out;
    double* const bwd_partials = ab.loss_partials;
    for (int it = 0; it < fl.iters; ++it) {
        const bool last = it + 1 == fl.iters;
        if (KIND == 0) {
            af.loss_out = last ? loss_out : nullptr;  // the last CTA sums the last iteration's
            fwd_tile<D4, KAHAN, false, 1, 4, true, false, 1>(af);
        } else {
            fwd_tile<D4, KAHAN, false, 3, 4, true, false, 1>(af);
        }
        // the tile's history (this CTA's generic stores) -> the backward's bulk copies (async
        // proxy, issued by thread 0): every store visible, then the proxy fence
        __threadfence();
        __syncthreads();
        if (threadIdx.x == 0) asm volatile("fence.proxy.async.global;" ::: "memory");
        ab.adam.step_size = fl.adam_table[2 * it];
        ab.adam.sqrt_bc2 = fl.adam_table[2 * it + 1];
        if (KIND == 0) {
            bwd_tile<D4, false, true, 4, 1, false, false, 1>(ab);
        } else {
            ab.loss_partials = last ? bwd_partials : nullptr;
            bwd_tile<D4, false, true, 4, 2, KAHAN, false, 1>(ab);
        }
        // the Adam epilogue's parameters are the next forward's inputs; the backward's last
        // staging reads are done before the next forward overwrites the history
        __syncthreads();
    }
}

template <bool D4, bool KH, int KIND>
static cudaError_t launch_fit_long_v(const FwdArgs& af, const BwdArgs& ab, const FitLongArgs& fl,
                                     int ntiles, cudaStream_t st) {
    constexpr size_t smem = bwd_smem_of<4, KIND == 0 ? 1 : 2>();
    static std::atomic<unsigned long long> optin{0};
    cudaError_t e = smem_optin((const void*)fit_long_kernel<D4, KH, KIND>, (int)smem, optin);
    if (e != cudaSuccess) return e;
    fit_long_kernel<D4, KH, KIND><<<ntiles, kT, smem, st>>>(af, ab, fl);
    return cudaGetLastError();
}

cudaError_t launch_fit_long(const FwdArgs& af, const BwdArgs& ab, const FitLongArgs& fl,
                            int ntiles, bool delta4, bool kahan, int kind, cudaStream_t st) {
    if (af.ckpt_every != 4 || ab.ckpt_every != 4) return cudaErrorInvalidValue;
    if (delta4) {
        if (kahan) return kind == 0 ? launch_fit_long_v<true, true, 0>(af, ab, fl, ntiles, st)
                                    : launch_fit_long_v<true, true, 1>(af, ab, fl, ntiles, st);
        return kind == 0 ? launch_fit_long_v<true, false, 0>(af, ab, fl, ntiles, st)
                         : launch_fit_long_v<true, false, 1>(af, ab, fl, ntiles, st);
    }
    if (kahan) return kind == 0 ? launch_fit_long_v<false, true, 0>(af, ab, fl, ntiles, st)
                                : launch_fit_long_v<false, true, 1>(af, ab, fl, ntiles, st);
    return kind == 0 ? launch_fit_long_v<false, false, 0>(af, ab, fl, ntiles, st)
                     : launch_fit_long_v<false, false, 1>(af, ab, fl, ntiles, st);
}

// ------------------------------------------------------------------------------ launchers
cudaError_t launch_state_from_obs(const float* obs, int64_t n, int steps, float dt, float* pos0,
                                  float* vel0, cudaStream_t st) {
    int64_t blocks = (n + 255) / 256;
    if (blocks > 148 * 8) blocks = 148 * 8;
    state_from_obs_kernel<<<(int)blocks, 256, 0, st>>>(obs, n, steps, dt, pos0, vel0);
    return cudaGetLastError();
}

cudaError_t launch_validate(const ValidateArgs& a, cudaStream_t st) {
    validate_kernel<<<148 * 4, 256, 0, st>>>(a);
    return cudaGetLastError();
}

bool ckpt_supported(int k) { return k == 2 || k == 4 || k == 8; }

// One launch: plain <<<>>> unless it needs attributes -- a thread-block cluster of csize CTAs
// (lanes longer than a tile) and / or programmatic stream serialization (the fused backward).
// IDM_SMEM_PAD=<bytes> (measurement only): extra dynamic shared memory
// on every forward / backward launch, which caps the resident CTAs per SM -- the occupancy an
// on-chip state history would leave (the on-chip-history experiment of NEXT-4).
static size_t smem_pad() {
    static const size_t pad = [] {
        const char* e = std::getenv("IDM_SMEM_PAD");
        return e ? (size_t)std::strtoull(e, nullptr, 10) : (size_t)0;
    }();
    return pad;
}

template <class A>
static cudaError_t launch_cfg(void (*kern)(A), const A& a, int grid, int block, size_t smem,
                              cudaStream_t st, int csize, bool pdl) {
    if (const size_t pad = smem_pad()) {
        smem += pad;
        const cudaError_t e = cudaFuncSetAttribute((const void*)kern,
                                                   cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                   (int)smem);
        if (e != cudaSuccess) return e;
    }
    if (csize <= 1 && !pdl) {
        kern<<<grid, block, smem, st>>>(a);
        return cudaSuccess;  // launch errors: cudaGetLastError in the caller
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(block);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    int na = 0;
    if (pdl) {
        attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[na].val.programmaticStreamSerializationAllowed = 1;
        ++na;
    }
    if (csize > 1) {
        attr[na].id = cudaLaunchAttributeClusterDimension;
        attr[na].val.clusterDim.x = (unsigned)csize;
        attr[na].val.clusterDim.y = 1;
        attr[na].val.clusterDim.z = 1;
        ++na;
    }
    cfg.attrs = attr;
    cfg.numAttrs = na;
    return cudaLaunchKernelEx(&cfg, kern, a);
}

template <bool D4, bool KH, int KS, bool CL>
static cudaError_t launch_fwd_k(const FwdArgs& a, int ntiles, const FwdVariant& var,
                                cudaStream_t st) {
    const int b = kCap / (2 * IDM_FWD_NP);
    const int b_api = kCap / (2 * IDM_FWD_NP_API);  // idm_forward with history
    const int cs = CL ? var.csize : 1;
    if constexpr (KS == 4) {  // the fused idm_fit_step forward exists for 4-step segments
        // (with clusters only the history-only variant: ptxas 12.9 crashes on the observation-
        // staging ones combined with the cluster message channel; the host uses LOSS 3 there)
        if constexpr (!CL) {
            if (var.loss == 1) return launch_cfg(fwd_kernel<D4, KH, false, 1, KS, true, CL>, a, ntiles, b, 0, st, cs, false);
            if (var.loss == 2) return launch_cfg(fwd_kernel<D4, KH, false, 2, KS, true, CL>, a, ntiles, b, 0, st, cs, false);
        } else {
            if (var.loss == 1 || var.loss == 2) return cudaErrorInvalidValue;
        }
        if (var.loss == 3) return launch_cfg(fwd_kernel<D4, KH, false, 3, KS, true, CL>, a, ntiles, b, 0, st, cs, false);
    }
    if (!var.hist) {  // prediction rollout: P rows only (the segment length is immaterial)
        if (var.rec_v) return launch_cfg(fwd_kernel<D4, KH, true, 0, 4, false, CL>, a, ntiles, b, 0, st, cs, false);
        return launch_cfg(fwd_kernel<D4, KH, false, 0, 4, false, CL>, a, ntiles, b, 0, st, cs, false);
    }
    if (var.rec_v) return launch_cfg(fwd_kernel<D4, KH, true, 0, KS, true, CL>, a, ntiles, b_api, 0, st, cs, false);
    return launch_cfg(fwd_kernel<D4, KH, false, 0, KS, true, CL>, a, ntiles, b_api, 0, st, cs, false);
}

template <bool D4, bool KH>
static cudaError_t launch_fwd_dk(const FwdArgs& a, int ntiles, const FwdVariant& var,
                                 cudaStream_t st) {
    if (var.csize > 1)  // lanes split over clusters: 4-step segments only (idm_init checks)
        return a.ckpt_every == 4 ? launch_fwd_k<D4, KH, 4, true>(a, ntiles, var, st)
                                 : cudaErrorInvalidValue;
    switch (a.ckpt_every) {
        case 2: return launch_fwd_k<D4, KH, 2, false>(a, ntiles, var, st);
        case 8: return launch_fwd_k<D4, KH, 8, false>(a, ntiles, var, st);
        default: return launch_fwd_k<D4, KH, 4, false>(a, ntiles, var, st);
    }
}

cudaError_t launch_fwd(const FwdArgs& a, int ntiles, const FwdVariant& var, cudaStream_t st) {
    if (!ckpt_supported(a.ckpt_every)) return cudaErrorInvalidValue;
    cudaError_t e;
    if (var.delta4) e = var.kahan ? launch_fwd_dk<true, true>(a, ntiles, var, st)
                                  : launch_fwd_dk<true, false>(a, ntiles, var, st);
    else e = var.kahan ? launch_fwd_dk<false, true>(a, ntiles, var, st)
                       : launch_fwd_dk<false, false>(a, ntiles, var, st);
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}

cudaError_t kernels_configure(int ckpt_every) {
    return ckpt_supported(ckpt_every) ? cudaSuccess : cudaErrorInvalidValue;
}


#ifndef IDM_BWD_NP
#define IDM_BWD_NP 1  // vehicle pairs per backward thread (1: 256 threads, 2: 128 threads; 2 measured 3.7% slower)
#endif
template <bool D4, bool SH, bool AD, int KS, int GO, bool KH, bool CL = false>
static cudaError_t launch_bwd_v(const BwdArgs& a, int ntiles, cudaStream_t st, bool pdl = false,
                                int csize = 1) {
    constexpr int NP = IDM_BWD_NP;
    constexpr int kTb = kCap / (2 * NP);
    constexpr size_t smem = bwd_smem_of<KS, GO>();
    static std::atomic<unsigned long long> optin{0};  // devices opted in (bit per device)
    cudaError_t e =
        smem_optin((const void*)bwd_kernel<D4, SH, AD, KS, GO, KH, CL, NP>, (int)smem, optin);
    if (e != cudaSuccess) return e;
    return launch_cfg(bwd_kernel<D4, SH, AD, KS, GO, KH, CL, NP>, a, ntiles, kTb, smem, st,
                      CL ? csize : 1, pdl);
}

// API backward (idm_backward): dL/dP rows from grad_traj, Adam by its own kernel
template <bool D4, int KS>
static cudaError_t launch_bwd_k(const BwdArgs& a, int ntiles, bool shared, cudaStream_t st,
                                int csize) {
    if constexpr (KS == 4) {
        if (csize > 1) {
            if (shared) return launch_bwd_v<D4, true, false, KS, 0, false, true>(a, ntiles, st, false, csize);
            return launch_bwd_v<D4, false, false, KS, 0, false, true>(a, ntiles, st, false, csize);
        }
    }
    if (csize > 1) return cudaErrorInvalidValue;
    if (shared) return launch_bwd_v<D4, true, false, KS, 0, false>(a, ntiles, st);
    return launch_bwd_v<D4, false, false, KS, 0, false>(a, ntiles, st);
}

// fused idm_fit_step backward (ckpt_every == 4): dL/dP from obs
template <bool D4, int GO, bool KH>
static cudaError_t launch_bwd_obs(const BwdArgs& a, int ntiles, bool shared, cudaStream_t st,
                                  bool pdl, int csize) {
    if (csize > 1) {  // no programmatic launch with clusters (idm_capi.cu use_pdl)
        if (shared) return launch_bwd_v<D4, true, false, 4, GO, KH, true>(a, ntiles, st, false, csize);
        return launch_bwd_v<D4, false, true, 4, GO, KH, true>(a, ntiles, st, false, csize);
    }
    if (shared) return launch_bwd_v<D4, true, false, 4, GO, KH>(a, ntiles, st, pdl);
    return launch_bwd_v<D4, false, true, 4, GO, KH>(a, ntiles, st, pdl);
}

template <bool D4>
static cudaError_t launch_bwd_d(const BwdArgs& a, int ntiles, bool shared, bool adam, int gobs,
                                bool kahan, cudaStream_t st, bool pdl, int csize) {
    if (gobs) {
        if (a.ckpt_every != 4) return cudaErrorInvalidValue;
        if (gobs == 1)  // sign codes: no positions needed, compensation irrelevant
            return launch_bwd_obs<D4, 1, false>(a, ntiles, shared, st, pdl, csize);
        if (gobs == 3) {  // L1 re-derived from obs and the rebuilt positions
            if (kahan) return launch_bwd_obs<D4, 3, true>(a, ntiles, shared, st, pdl, csize);
            return launch_bwd_obs<D4, 3, false>(a, ntiles, shared, st, pdl, csize);
        }
        if (kahan) return launch_bwd_obs<D4, 2, true>(a, ntiles, shared, st, pdl, csize);
        return launch_bwd_obs<D4, 2, false>(a, ntiles, shared, st, pdl, csize);
    }
    if (pdl || adam) return cudaErrorInvalidValue;  // API backward: after the loss kernel, no Adam
    switch (a.ckpt_every) {
        case 2: return launch_bwd_k<D4, 2>(a, ntiles, shared, st, csize);
        case 4: return launch_bwd_k<D4, 4>(a, ntiles, shared, st, csize);
        case 8: return launch_bwd_k<D4, 8>(a, ntiles, shared, st, csize);
        default: return cudaErrorInvalidValue;
    }
}

cudaError_t launch_bwd(const BwdArgs& a, int ntiles, bool delta4, bool shared, bool adam,
                       int gobs, bool kahan, cudaStream_t st, bool pdl, int csize) {
    cudaError_t e = delta4 ? launch_bwd_d<true>(a, ntiles, shared, adam, gobs, kahan, st, pdl, csize)
                           : launch_bwd_d<false>(a, ntiles, shared, adam, gobs, kahan, st, pdl, csize);
    if (e != cudaSuccess) return e;
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
    reduce_kernel<<<width, 256, 0, st>>>(partials, n, width, out, out_f);
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
