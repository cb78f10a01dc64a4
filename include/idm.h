/*
 * idm.h -- C-ABI of the B200-native differentiable IDM hot path (arXiv 2412.16750).
 *
 * One optimizer iteration of the paper's trajectory fitting is
 *
 *     idm_forward(h, K)            Eqs. 1-3 + Sec. III-C bounds, K synchronous Euler steps
 *     idm_loss_grad(h, obs, ...)   Eq. 4 loss and dL/dP
 *     idm_backward(h)              reverse-mode adjoint to the parameters and initial state
 *     idm_adam_step(h, it, ...)    Adam + linear lr decay + box clamp
 *
 * Citations "PAPER.md:N" are lines of the paper's LaTeX; "R#n" are the readings of silent or
 * ambiguous passages listed in DESIGN.md.
 *
 * Conventions (all calls):
 *   - Every array pointer in idm_desc is a DEVICE pointer owned by the caller (the Python
 *     binding keeps torch tensors alive for the handle's lifetime).  The library owns only the
 *     opaque handle and the caller-allocated workspace it is given (idm_workspace_bytes).
 *   - fp32 arrays; SoA layout; vehicles are LANE-SORTED: lane l owns the index range
 *     [lane_offsets[l], lane_offsets[l+1]) in ascending position, so the leader h(i) of
 *     vehicle i is i+1 when i+1 is in the same lane, and the lane head has no
 *     leader (exact free road, R#8).  Lanes never change (no lane changes, R#9).
 *   - Parameters are SoA [6][n_par] in the order
 *         0 a_max  1 a_pref  2 s_min  3 T_pref  4 v_targ  5 delta
 *     (delta = IDM exponent, R#1), n_par = N (IDM_PARAMS_PER_VEHICLE,
 *     "fixed for each trajectory") or 1 (IDM_PARAMS_SHARED).
 *   - Trajectory arrays are step-major [(steps+1)][N]: row t holds P(t) = p_i(t), absolute
 *     positions in m (the array P of Eq. 4).
 *   - Every call is ordered on desc->stream (a cudaStream_t); only idm_init, idm_loss_grad
 *     with loss_host != NULL, idm_check and idm_step_host synchronize it.
 *   - Return value: an idm_status.  On failure idm_last_error(h) holds a sticky message.
 *     Calls out of order (e.g. idm_backward before idm_loss_grad) return IDM_ESTATE.
 *   - No CPU fallback: without a usable sm_100a device every call returns IDM_ECUDA.
 */
#ifndef IDM_H
#define IDM_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct idm_handle idm_handle; /* opaque */

typedef enum {
    IDM_OK = 0,
    IDM_EINVAL = 1,   /* invalid argument or input data (SPEC "data error", exit 1) */
    IDM_ENUMERIC = 2, /* non-finite state or gradient (SPEC "numerical failure", exit 2) */
    IDM_ECUDA = 3,    /* CUDA runtime error / no device */
    IDM_ESTATE = 4    /* call-order violation */
} idm_status;

typedef enum { IDM_PARAMS_PER_VEHICLE = 0, IDM_PARAMS_SHARED = 1 } idm_param_mode;
typedef enum { IDM_LOSS_L1 = 0 /* Eq. 4 */, IDM_LOSS_L2 = 1 /* smooth variant */ } idm_loss_kind;
typedef enum {
    IDM_LEADER_LANE = 0,    /* leader = next vehicle ahead in the lane */
    IDM_LEADER_VIRTUAL = 1  /* free per-step leader terms (Delta p_k, Delta v_k) */
} idm_leader_mode;

typedef struct {
    int64_t n_vehicles;          /* N >= 1 */
    int32_t n_lanes;             /* L >= 1 */
    const int32_t* lane_offsets; /* [L+1], non-decreasing, [0] = 0, [L] = N */
    float* pos0;                 /* [N] initial absolute position p_i(0) (m); written only by
                                    idm_step_host (upload) */
    float* vel0;                 /* [N] initial speed v_i(0) >= 0 (m/s); idem */
    const float* length;         /* [N] body length of each vehicle (m) */
    float* params;               /* [6][n_par] IDM parameters; updated by idm_adam_step */
    float* grad_params;          /* [6][n_par] dL/dtheta written by idm_backward */
    float* adam_m;               /* [6][n_par] Adam first moment (caller zero-initialises) */
    float* adam_v;               /* [6][n_par] Adam second moment (caller zero-initialises) */
    float* grad_state0;          /* [2][N] dL/dp(0), dL/dv(0) from idm_backward (nullable) */
    float* traj;                 /* [(max_steps+1)][N] positions P(t) (required for the loss) */
    float* vel_traj;             /* [(max_steps+1)][N] speeds v(t) (nullable; diagnostics) */
    float* grad_traj;            /* [(max_steps+1)][N] dL/dP from idm_loss_grad */
    float* state_out;            /* [2][N] final position and speed (nullable) */
    float* obs_stage;            /* [(max_steps+1)][N] device staging for idm_step_host (nullable) */
    uint8_t* mask_stage;         /* [(max_steps+1)][N] staging for the mask (nullable) */
    int32_t max_steps;           /* K_max >= 1 */
    int32_t ckpt_every;          /* k: backward checkpoint interval, 2, 4 (recommended) or 8 --
                                    compile-time segment lengths of the kernels
                                    (idm_workspace_bytes returns 0 otherwise) */
    float dt;                    /* Delta t > 0 (0.1 s) */
    float a_min;                 /* < 0, maximum deceleration (-10) */
    float eps_gap;               /* > 0, gap clamp (0.1 m, R#7) */
    int32_t param_mode;          /* idm_param_mode */
    uint32_t opt_mask;           /* bit k set = parameter k optimized by Adam; the paper's five:
                                    0x1F (delta frozen) */
    void* stream;                /* cudaStream_t (NULL = legacy default stream) */
    void* workspace;             /* device, >= idm_workspace_bytes(desc), 256-B aligned */
    size_t workspace_bytes;
    /* Virtual-leader mode ("We also optimize the lists of Delta p_k and Delta v_k
       for each simulation step k, initializing them to 10 and 0"): each vehicle is fitted alone
       and its leader terms at step k are the free variables below (lanes are ignored; gaps
       below eps_gap are clamped with zero gradient, R#7).  idm_backward writes their
       gradients, idm_adam_step / idm_fit_step update them with the same Adam schedule (no
       box; idm_fit_step applies it inside the backward sweep and does not write vl_grad).
       Requires ckpt_every == 4. */
    int32_t leader_mode;         /* idm_leader_mode (0 = lane leader) */
    float* vl_dp;                /* [max_steps][N] Delta p_k */
    float* vl_dv;                /* [max_steps][N] Delta v_k */
    float* vl_grad;              /* [2][max_steps][N] dL/dDelta p_k, dL/dDelta v_k */
    float* vl_adam_m;            /* [2][max_steps][N] Adam moments of the leaves (zeroed) */
    float* vl_adam_v;            /* [2][max_steps][N] */
    float* obs_stage2;           /* [(max_steps+1)][N] second observation staging buffer
                                    (nullable): idm_step_host(_async) alternate between the two
                                    when no mask is given, so an upload never waits for the
                                    previous step's loss kernel */
    double* lane_grads;          /* shared mode: [n_lanes][6] fp64, row l = the sum of lane l's
                                    vehicles' dL/dtheta in vehicle order, written by
                                    idm_backward / idm_fit_step (empty lanes: 0) -- the unit of
                                    the shard-count-invariant reduction (idm_reduce_shared).
                                    Nullable: then kept in the workspace */
} idm_desc;

/* Bytes of device workspace idm_init needs for this descriptor (reads lane_offsets to plan the
   tiles): lane mode -- the state history (every vehicle's speed at every step and (gap,
   displacement) every ckpt_every steps, in a tile-local layout sized for the plan's tile count,
   about (max_steps + 1) N floats), the L1 sign codes; virtual-leader mode -- speed and
   displacement checkpoints; both -- the lane-tile plan, leader flags, reduction partials,
   per-lane shared-gradient rows (shared mode without desc.lane_grads), status word.
   Returns 0 if the descriptor is malformed. */
size_t idm_workspace_bytes(const idm_desc* d);

/* The lane -> CTA tile plan idm_init builds (host only, no device needed): whole lanes per
   tile, at most idm_max_lane_vehicles() vehicles per tile, packed greedily in lane order, so two
   consecutive tiles always hold more than that many vehicles.  lane_offsets: HOST [n_lanes+1].
   Writes the n_tiles+1 tile starts (vehicle indices, last = n_vehicles) to tile_start (HOST,
   nullable: count only) and returns n_tiles, or -1 for malformed offsets or a lane longer than
   idm_max_lane_length().  With a lane longer than a tile the plan holds empty padding tiles
   (equal consecutive starts) so that such lanes start at multiples of the cluster size. */
int64_t idm_plan_tiles(const int32_t* lane_offsets, int32_t n_lanes, int64_t n_vehicles,
                       int64_t* tile_start);

/* Initial state of a fit from its observations, the paper's initialisation (PAPER.md:267:
   "the initial position p(0) and speed v(0) for each trajectory were set to 0 and
   (Delta P) / Delta t, where Delta P is the distance between the first two data points"; R#13:
   with lanes, p(0) is the vehicle's own first observation).  obs: DEVICE [(steps+1)][N]
   step-major positions, NaN = not observed (as idm_loss_grad).  Per vehicle, the first two
   observed rows t1 < t2 give
       vel0 = max(0, (obs[t2] - obs[t1]) / ((t2 - t1) dt)),   pos0 = obs[t1] - t1 dt vel0
   (the first data point carried back to step 0 at that speed: obs[t1] when t1 = 0); one
   observation: vel0 = 0, pos0 = obs[t1]; none: 0, 0.  pos0, vel0: DEVICE [N] outputs (e.g. the
   arrays a descriptor will point to).  No handle needed (call before idm_init); ordered on
   `stream` (cudaStream_t, NULL = legacy); IDM_EINVAL for bad arguments, IDM_ECUDA if the launch
   fails. */
int idm_state_from_obs(const float* obs, int64_t n_vehicles, int32_t steps, float dt,
                       float* pos0, float* vel0, void* stream);

/* Validate the descriptor and input data (finite, v(0) >= 0, lengths >= 0, a_max, a_pref,
   v_targ, delta > 0, lane offsets well formed, every lane at most idm_max_lane_length()
   vehicles, and -- lane mode -- every lane member strictly behind its
   leader: pos0[i+1] - pos0[i] - length[i+1] > 0, the ordering PAPER.md:106 presumes ("the
   vehicle directly ahead"); gaps in (0, eps_gap) are valid and clamped, R#7), build the
   lane -> CTA tile plan and leader flags in the workspace.  IDM_EINVAL on any violation, with
   the first offending vehicle in the message.  Virtual-leader mode has no lanes: no plan, no
   lane-size limit, no order check.  Synchronizes the stream.  *out receives the handle (NULL
   on failure).  The desc is copied; the arrays it points to must stay valid until idm_destroy.
   The handle belongs to the CUDA device current here; every later call runs on that device
   (made current for the call, the caller's current device restored after). */
int idm_init(idm_handle** out, const idm_desc* d);

/* Simulate `steps` (1..max_steps) synchronous steps from (pos0, vel0) (Eqs. 1-3, Sec. III-B/C,
   PAPER.md:106-152): one fused launch, state in registers; traj rows 0..steps (and vel_traj,
   state_out if given); the workspace gets every vehicle's speed at every step, its gap every
   8 ckpt_every steps and its final gap, which idm_backward reads back.
   Non-finite states are detected at checkpoints and reported by the next synchronizing call. */
int idm_forward(idm_handle* h, int32_t steps);

/* Flags of idm_forward_ex. */
enum {
    IDM_FWD_NO_HISTORY = 1 /* prediction rollout: write traj (and vel_traj, state_out) only, no
                              state history -- half the HBM bytes of idm_forward; idm_loss_grad
                              may follow, idm_backward then returns IDM_ESTATE */
};

/* idm_forward with flags (0 = idm_forward).  The same arithmetic, so traj is bit-identical. */
int idm_forward_ex(idm_handle* h, int32_t steps, uint32_t flags);

/* Eq. 4 over rows 0..steps of traj:
     L1: L = sum_{observed (t,i)} |obs - P|,  dL/dP = -sign(obs - P), sign(0) = 0 (R#11)
     L2: L = sum (obs - P)^2,                 dL/dP = -2 (obs - P)
   obs: device [(steps+1)][N]; mask: device uint8 [(steps+1)][N], nonzero = observed, or NULL.
   (t,i) is observed iff the mask is set (or NULL) and obs is finite (NaN = missing).  Writes grad_traj; the loss (fixed-order fp64 reduction, deterministic) to
   *loss_dev (device double, nullable) and, if loss_host != NULL, to *loss_host (synchronizes;
   also reports a pending non-finite status as IDM_ENUMERIC). */
int idm_loss_grad(idm_handle* h, const float* obs, const uint8_t* mask, int32_t kind,
                  double* loss_dev, double* loss_host);

/* Reverse-mode adjoint of the last idm_forward through grad_traj -- the derivative of the
   simulator that PAPER.md:134 makes "differentiable" and PAPER.md:227 obtains by autograd:
   the full coupled BPTT of Eqs. 1-3 with the Sec. III-C bounds (leader states included,
   R#23), given dL/dP from idm_loss_grad (Eq. 4).  Per lane tile it rebuilds
   each checkpoint segment's gaps from the stored speeds on chip (backwards from the final gap,
   re-anchored on the stored gap every 8 segments) and sweeps it backwards.
   Writes
     grad_params  [6][n_par]  dL/d(a_max, a_pref, s_min, T_pref, v_targ, delta), row 5 = the
                  true dL/d delta on this call (the fused optimizer calls write 0 there when
                  delta is frozen, see idm_fit_step);  in shared mode the fixed-order sum of
                  lane_grads over this handle's lanes (one rank: the whole gradient);
     lane_grads   (shared mode) the per-lane sums, for idm_reduce_shared across ranks;
     grad_state0  [2][N]  dL/dp(0), dL/dv(0) (nullable).
   IDM_ESTATE unless the last forward kept its history (idm_forward, not IDM_FWD_NO_HISTORY)
   and idm_loss_grad followed it.  No atomics: fixed-order reductions, bitwise deterministic. */
int idm_backward(idm_handle* h);

/* Shared-parameter mode across ranks (north_star: NCCL only for the shared gradients and the
   loss): grad_params = the fixed-order fp64 sum over rows 0..n_rows-1 of lane_grads (device
   [n_rows][6], the rows of ALL ranks' lanes in global lane order, e.g. each rank's own rows
   placed in a zeroed buffer and all-reduced -- disjoint rows make that all-reduce exact), rounded
   to fp32.  The result depends only on the global rows, so it is bitwise the same for any
   number of ranks.  Call between idm_backward and idm_adam_step. */
int idm_reduce_shared(idm_handle* h, const double* lane_grads, int64_t n_rows);

/* Adam step (Kingma & Ba; beta1 0.9, beta2 0.999, eps 1e-8, bias-corrected, R#14) on the
   parameters selected by opt_mask with lr = lr0 + (lr1 - lr0) * iter / (total_iters - 1)
   (0.1 -> 0.01 over 500), then clamp (a_max, a_pref, s_min, T_pref, v_targ) to
   [5,10], [0.1,5], [1,10], [0.1,5], [20,60] (R#15).  iter is 0-based. */
int idm_adam_step(idm_handle* h, int32_t iter, int32_t total_iters, float lr0, float lr1);

/* One whole optimizer iteration, fused: exactly forward(steps) -> loss_grad(obs, kind) ->
   backward -> adam_step(iter, ...) (same arithmetic; grad_params, grad_state0, Adam moments and
   parameters bit for bit -- except grad_params row 5, dL/d delta: on the optimizer calls
   (idm_fit_step, idm_fit, idm_fit_steps) it is written as 0 when delta is frozen (opt_mask
   bit 5 clear), because the optimizer never reads it and the delta = 4 kernels skip the
   per-step log2 it needs; idm_backward always writes the true value), when ckpt_every == 4 in
   two kernels writing only
   the internal state history, the backward launched as a programmatic dependent of the forward
   (each CTA waits for its own tile's history) and applying Adam + box clamp per vehicle in its
   epilogue.  L1: the forward sums Eq. 4 against each fresh position row and records
   dL/dP = -sign as 2 bits per vehicle-step; its last CTA sums the per-tile losses (2 launches).
   L2: the forward only records the history; the backward derives the loss terms and dL/dP
   from obs and the rebuilt positions, and one fixed-order reduction sums the losses (3
   launches) (shared mode: + reduce + Adam launches; the shared gradient is THIS
   process's sum, so with several ranks use the separate calls and all-reduce between
   idm_backward and idm_adam_step -- the Python binding refuses the fused calls there).  traj
   and grad_traj are NOT written on this path.  With any other ckpt_every, and for
   latency-bound shapes (lane tiles <= half the SMs and >= 1000 steps, e.g. C3's 6 tiles x
   27,000 steps, where the separate kernels are faster), the defining sequence runs as is (and
   writes them); IDM_FUSED_ALWAYS=1 disables the latter.
   obs: device [(steps+1)][N]; missing observations are NaN (mask must be NULL).  Loss to
   *loss_dev / *loss_host as in idm_loss_grad. */
int idm_fit_step(idm_handle* h, int32_t steps, const float* obs, const uint8_t* mask,
                 int32_t kind, int32_t iter, int32_t total_iters, float lr0, float lr1,
                 double* loss_dev, double* loss_host);

/* Whole fit in one launch (NEXT-4): iterations iter0 .. iter0+iters-1 of exactly
   idm_fit_step(steps, obs, kind, it, total_iters, lr0, lr1) -- parameters, Adam moments and
   gradients (incl. the zero delta row of a frozen delta) come out bit-identical.  Lane tiles are
   independent across iterations (tile j's next forward needs only the parameters its own
   backward updated), so each CTA runs its tile's whole fit with no grid-wide synchronisation:
     steps <= idm_fit_max_steps(): state history, observations and Adam moments on chip (Waymo-
       shaped prediction histories of 10 steps);
     longer horizons: per iteration the fused forward (Eq. 4 in-kernel) then the backward with
       Adam, the state history through memory (written and re-read by the same CTA; needs
       ckpt_every == 4).
   Lane-leader mode with per-vehicle parameters and lanes within one tile; iters <= 4096 per
   call; traj / grad_traj are not written.  The loss of the last iteration (same Eq. 4, summed in
   a different fixed order) goes to *loss_dev / *loss_host. */
int idm_fit(idm_handle* h, int32_t steps, const float* obs, int32_t kind, int32_t iter0,
            int32_t iters, int32_t total_iters, float lr0, float lr1, double* loss_dev,
            double* loss_host);

/* Largest horizon of idm_fit's on-chip variant (longer ones run the long-horizon kernel). */
int32_t idm_fit_max_steps(void);

/* Iterations iter0 .. iter0+iters-1 of idm_fit_step(steps, obs, kind, it, total_iters, lr0, lr1)
   for any horizon, launched as ONE CUDA graph: the calls are captured on the handle's stream
   (each iteration's Adam step size baked into its kernel nodes) and the graph is launched once,
   which removes the per-launch host overhead that dominates small configurations.  Same
   kernels, same order: parameters, moments and gradients are bit-identical to the loop of
   idm_fit_step calls.  The loss of the last iteration goes to *loss_dev / *loss_host.  The
   instantiated graph is kept by the handle until the next call or idm_destroy. */
int idm_fit_steps(idm_handle* h, int32_t steps, const float* obs, int32_t kind, int32_t iter0,
                  int32_t iters, int32_t total_iters, float lr0, float lr1, double* loss_dev,
                  double* loss_host);

/* One whole optimizer iteration from HOST buffers (end-to-end path): async-copies pos0/vel0
   (nullable = keep), obs (required) and mask (nullable = all observed) from host memory
   (pinned for overlap) into desc->pos0/vel0/obs_stage/mask_stage, runs forward(steps) ->
   loss_grad -> backward -> adam_step(iter, total_iters, lr0, lr1) and copies the loss back to
   *loss_host (synchronizes).  The obs upload overlaps the forward kernel on a second stream. */
int idm_step_host(idm_handle* h, int32_t steps, const float* pos0_host, const float* vel0_host,
                  const float* obs_host, const uint8_t* mask_host, int32_t kind, int32_t iter,
                  int32_t total_iters, float lr0, float lr1, double* loss_host);

/* Pipelined form of idm_step_host for a stream of iterations: enqueues the same uploads and
   kernels plus an asynchronous read of the loss and status, and returns without synchronizing,
   so the next call's observation upload (which still waits for this step's loss kernel, the
   staging buffer's last reader) overlaps this step's backward and Adam.  At most two steps may
   be in flight; idm_step_host_wait retires the oldest.  Same arithmetic as idm_step_host. */
int idm_step_host_async(idm_handle* h, int32_t steps, const float* pos0_host,
                        const float* vel0_host, const float* obs_host, const uint8_t* mask_host,
                        int32_t kind, int32_t iter, int32_t total_iters, float lr0, float lr1);

/* Waits for the oldest idm_step_host_async step; its loss to *loss_host (nullable).  A pending
   non-finite or invalid status drains the pipeline and is returned as by idm_check.
   IDM_ESTATE if no step is in flight. */
int idm_step_host_wait(idm_handle* h, double* loss_host);

/* Kernel classes for idm_timing_read. */
enum {
    IDM_K_FWD = 0,      /* forward (fused with Eq. 4 in idm_fit_step) */
    IDM_K_LOSS = 1,     /* Eq. 4 loss kernel (idm_loss_grad) */
    IDM_K_REDUCE = 2,   /* fixed-order reductions (loss, shared gradients) */
    IDM_K_BWD = 3,      /* backward (with the Adam epilogue in idm_fit_step) */
    IDM_K_ADAM = 4,     /* Adam kernel */
    IDM_K_OTHER = 5,    /* validation */
    IDM_NKERNELS = 6
};

/* Launch timing for benchmarks: while enabled, every kernel launch of this handle is bracketed
   by CUDA events recorded on desc->stream.  idm_timing_read synchronizes, writes the summed
   device milliseconds and launch counts per class (arrays of IDM_NKERNELS, nullable) and resets
   the accumulators. */
int idm_timing_enable(idm_handle* h, int enable);
int idm_timing_read(idm_handle* h, double* ms, int64_t* launches);

/* Synchronize the stream and report a pending non-finite status (IDM_ENUMERIC: a non-finite
   state at a checkpoint, or a non-finite parameter gradient reaching Adam) or CUDA error. */
int idm_check(idm_handle* h);

/* Number of kernel launches the library issued on this handle since idm_init. */
int64_t idm_launch_count(const idm_handle* h);

/* Largest lane (vehicles) one lane tile holds (one CTA). */
int32_t idm_max_lane_vehicles(void);

/* Largest lane (vehicles) supported: idm_max_lane_vehicles() x 8.  A lane longer than one tile
   runs over a thread-block cluster of consecutive tiles (up to 8, the portable cluster size):
   the boundary vehicles' leader speeds and adjoint terms cross CTAs through distributed shared
   memory and every step barrier is cluster-wide.  Such a plan needs ckpt_every == 4, runs
   every launch in clusters (slower steps), and idm_fit rejects it. */
int32_t idm_max_lane_length(void);

/* Sticky last error message of h ("" if none; a static message if h is NULL). */
const char* idm_last_error(const idm_handle* h);

/* Release the handle (not the caller's arrays).  NULL is a no-op. */
void idm_destroy(idm_handle* h);

#ifdef __cplusplus
}
#endif
#endif /* IDM_H */
