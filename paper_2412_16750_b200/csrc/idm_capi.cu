// idm_capi.cu -- host side of the C-ABI (include/idm.h): validation, lane-tile plan,
// workspace carving, call-order state machine and kernel launches.  No compute happens here.
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/idm.h"
#include "idm_internal.h"

using namespace idm;

struct idm_handle {
    idm_desc d;
    int device;  // the CUDA device current at idm_init; every entry point runs on it
    cudaStream_t st;
    int64_t n, n_par;
    int ntiles, nck;
    int csize;    // > 1: a lane is longer than a tile; every launch runs clusters of csize tiles
    int num_sms;  // of the handle's device
    // workspace carve-outs
    int64_t* tile_start;
    uint8_t* lead;
    float *vt, *ckt, *ckpt_v;     // lane-mode state history (tile-local), VL speed checkpoints
    float* ckpt_d;                // VL displacement checkpoints (fused iteration)
    uint32_t* sgn;                // fused L1 sign codes (tile-local)
    int64_t vt_stride, ck_stride, sg_stride;
    double *loss_partials, *loss_scalar;
    double* lane_grads;  // shared mode: [n_lanes][6] per-lane gradient sums (desc or workspace)
    bool hist_ok;        // the last forward kept its state history (a backward may follow)
    unsigned long long* status;
    unsigned* flags;  // [0] = some delta != 4 (set by the validation kernel)
    unsigned* tile_ready;  // [ntiles] forward -> backward handoff epochs of idm_fit_step (PDL)
    unsigned epoch;        // last epoch used
    unsigned* done_count;  // fused backward's finished-tile ticket (0 between launches)
    float* adam_table;  // [kFitMaxIters][2] per-iteration Adam step sizes for idm_fit
    float* adam_table_host;  // pinned staging of the above
    bool delta4;      // all delta == 4 and delta frozen => specialised kernels
    // host-side resources for idm_step_host / synchronous reads
    cudaStream_t copy_st;
    cudaEvent_t ev_obs, ev_loss_done, ev_loss_done2;  // last reader of obs_stage / obs_stage2
    int stage_next;  // staging buffer of the next host step (0 / 1 with obs_stage2)
    cudaEvent_t ev_step[2];  // idm_step_host_async: completion of the (up to) two steps in flight
    int async_head, async_n;
    // fused iteration in tile chunks: backward of chunk c on st2 overlaps forward of chunk c+1
    cudaStream_t st2;
    cudaEvent_t ev_fork, ev_join, ev_chunk[16];
    cudaGraphExec_t graph_exec;  // last idm_fit_steps graph (kept until the next call / destroy)
    cudaStream_t cap_st;         // capture stream (capture is not allowed on the legacy stream)
    cudaEvent_t ev_gfork, ev_gjoin;
    double* pinned;  // [0] loss, [1] status (as bits), [2] flags
    int stage;       // 0 = initialised, 1 = forward done, 2 = loss done, 3 = backward done
    int32_t steps;
    int64_t launches;
    char err[512];
    // launch timing (idm_timing_enable)
    bool timing;
    std::vector<cudaEvent_t>* ev_pool;
    std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>>* ev_rec;
};

namespace {

const char* kNoHandle = "idm: NULL handle";

int fail(idm_handle* h, int code, const char* fmt, ...) {
    if (h) {
        va_list ap;
        va_start(ap, fmt);
        vsnprintf(h->err, sizeof(h->err), fmt, ap);
        va_end(ap);
    }
    return code;
}

#define CK(h, call)                                                                       \
    do {                                                                                  \
        cudaError_t e_ = (call);                                                          \
        if (e_ != cudaSuccess)                                                            \
            return fail((h), IDM_ECUDA, "CUDA error %s at %s:%d (%s)", cudaGetErrorString(e_), \
                        __FILE__, __LINE__, #call);                                       \
    } while (0)

size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

struct Layout {
    size_t tile_start, lead, vt, ckt, sgn, ckpt_v, ckpt_d, loss_partials, loss_scalar, shared_partials,
        status, flags, adam_table, tile_ready, done_count, total;
    int64_t vt_stride, ck_stride, sg_stride;  // elements per tile
};

bool lane_mode(const idm_desc* d) { return d->leader_mode != IDM_LEADER_VIRTUAL; }

constexpr int kMaxCluster = 8;  // portable thread-block cluster size: lanes <= 8 kCap vehicles

int64_t max_tiles_for(const idm_desc* d) {
    if (!lane_mode(d)) return 1;  // virtual leader: independent trajectories, no lane tiles
    const int64_t n = d->n_vehicles;
    // greedy packing: <= 2N/kCap + 1; each lane longer than a tile (< N/kCap of them) adds at
    // most 2 (kMaxCluster - 1) empty padding tiles, and the end pads to a cluster multiple
    int64_t by_size = 2 * ((n + kCap - 1) / kCap) + 1 + 2 * (kMaxCluster - 1) * (n / kCap + 1) +
                      kMaxCluster;
    return d->n_lanes + 2 * (kMaxCluster - 1) * (n / kCap + 1) + kMaxCluster < by_size
               ? d->n_lanes + 2 * (kMaxCluster - 1) * (n / kCap + 1) + kMaxCluster
               : by_size;
}

// Lane-tile plan (cold path, host): whole lanes per tile, <= kCap vehicles; greedy, so two
// consecutive tiles always hold > kCap vehicles.  A lane longer than kCap (up to kMaxCluster
// kCap vehicles) runs over one thread-block cluster of cs consecutive tiles, cs = the longest
// lane's tile count: it starts at a tile index that is a multiple of cs (empty padding tiles
// before it), fills full tiles of kCap vehicles (the last one the remainder, then empty ones up
// to cs), and no other lane shares its tiles; the tile count is padded to a multiple of cs.
// Every launch of such a plan uses clusters of cs CTAs (csize_out; 1 = no long lane).  Fills
// tile starts and leader flags (if given); returns the tile count, or -1 with *err set.
// chunk (a multiple of 4, <= kCap): lanes longer than chunk are split into tiles of chunk
// vehicles (kCap: only lanes that do not fit a tile; smaller: latency-bound shapes spread over
// more SMs, see split_chunk_for).
int64_t plan_tiles(const std::vector<int32_t>& off, int32_t n_lanes, int64_t n,
                   std::vector<int64_t>* tiles, std::vector<uint8_t>* lead, std::string* err,
                   int* csize_out = nullptr, int64_t chunk = kCap) {
    char buf[256];
    if (off[0] != 0 || off.back() != n) {
        std::snprintf(buf, sizeof buf, "lane_offsets must start at 0 and end at N=%lld (got %d..%d)",
                      (long long)n, off[0], off.back());
        *err = buf;
        return -1;
    }
    int64_t longest = 0;
    for (int32_t l = 0; l < n_lanes; ++l) {
        const int64_t a = off[l], b = off[l + 1];
        if (b < a) {
            std::snprintf(buf, sizeof buf, "lane_offsets decrease at lane %d", l);
            *err = buf;
            return -1;
        }
        if (b - a > kMaxCluster * chunk) {
            std::snprintf(buf, sizeof buf,
                          "lane %d has %lld vehicles; at most %lld per lane are supported (%d "
                          "tiles of %lld in one thread-block cluster)", l, (long long)(b - a),
                          (long long)(kMaxCluster * chunk), kMaxCluster, (long long)chunk);
            *err = buf;
            return -1;
        }
        longest = b - a > longest ? b - a : longest;
    }
    const int cs = longest > chunk ? (int)((longest + chunk - 1) / chunk) : 1;
    if (csize_out) *csize_out = cs;
    std::vector<int64_t> t(1, 0);  // tile starts; the last entry is the open tile
    int64_t cur = 0;               // vehicles in the open tile
    for (int32_t l = 0; l < n_lanes; ++l) {
        const int64_t a = off[l], b = off[l + 1];
        const int64_t sz = b - a;
        if (sz == 0) continue;
        if (sz > chunk) {  // a cluster of its own, starting at a multiple of cs
            if (cur > 0) t.push_back(a);
            while ((t.size() - 1) % (size_t)cs != 0) t.push_back(a);  // empty tiles [a, a)
            for (int c = 1; c < cs; ++c) t.push_back(a + c * chunk < b ? a + c * chunk : b);
            cur = kCap;  // closed: the next lane opens a new tile
        } else {
            if (cur + sz > kCap) {
                t.push_back(a);
                cur = 0;
            }
            cur += sz;
        }
        if (lead)
            for (int64_t i = a; i + 1 < b; ++i) (*lead)[(size_t)i] = 1;
    }
    t.push_back(n);
    while ((t.size() - 1) % (size_t)cs != 0) t.push_back(n);  // empty tiles [n, n)
    const int64_t count = (int64_t)t.size() - 1;
    if (tiles) *tiles = std::move(t);
    return count;
}

// Split chunk of the lane plan.  A latency-bound shape -- few tiles and a long horizon, e.g.
// C3's 6 lanes of 333 vehicles over 27,000 steps on 148 SMs -- steps at the pace of one CTA's
// per-step chain, so its lanes can be spread over thread-block clusters of smaller tiles
// (IDM_SPLIT_LANES=auto | <vehicles per tile> | 0 = off, the default).
int64_t split_chunk_for(const std::vector<int32_t>& off, int32_t n_lanes, int64_t n,
                        int32_t max_steps, int num_sms) {
    const char* e = std::getenv("IDM_SPLIT_LANES");
    if (!e || e[0] == '0' || e[0] == 0) return kCap;
    int64_t longest = 0;
    for (int32_t l = 0; l < n_lanes; ++l)
        longest = off[l + 1] - off[l] > longest ? off[l + 1] - off[l] : longest;
    int64_t chunk;
    if (std::strcmp(e, "auto") == 0) {
        std::string err;
        const int64_t nt = plan_tiles(off, n_lanes, n, nullptr, nullptr, &err);
        if (nt < 0 || 4 * nt > num_sms || max_steps < 1000 || longest <= 8) return kCap;
        int64_t c = num_sms / nt;
        c = c > kMaxCluster ? kMaxCluster : (c < 1 ? 1 : c);
        chunk = (longest + c - 1) / c;
    } else {
        chunk = std::atoll(e);
    }
    chunk = (chunk + 3) / 4 * 4;  // tiles of a split lane hold a multiple of 4 vehicles
    if (chunk < 4) chunk = 4;
    if (chunk > kCap) chunk = kCap;
    if (longest > kMaxCluster * chunk) chunk = kCap;  // the lane would need a larger cluster
    return chunk;
}

// Tile count of the descriptor's lane plan (reads lane_offsets), or the bound if unreadable.
int64_t tiles_of(const idm_desc* d) {
    if (!d || !d->lane_offsets || d->n_lanes < 1) return -1;
    if (!lane_mode(d)) return 1;
    std::vector<int32_t> off((size_t)d->n_lanes + 1);
    if (cudaMemcpy(off.data(), d->lane_offsets, sizeof(int32_t) * off.size(), cudaMemcpyDefault) !=
        cudaSuccess) {
        cudaGetLastError();
        return -1;
    }
    std::string err;
    int num_sms = 148, dev = 0;
    if (cudaGetDevice(&dev) == cudaSuccess)
        cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, dev);
    cudaGetLastError();
    return plan_tiles(off, d->n_lanes, d->n_vehicles, nullptr, nullptr, &err, nullptr,
                      split_chunk_for(off, d->n_lanes, d->n_vehicles, d->max_steps, num_sms));
}

// ntiles: the plan's tile count (< 0: size for the bound max_tiles_for)
bool layout_for(const idm_desc* d, int64_t ntiles, Layout* L) {
    if (!d || d->n_vehicles < 1 || d->n_lanes < 1 || d->max_steps < 1 ||
        !ckpt_supported(d->ckpt_every))
        return false;
    int64_t n = d->n_vehicles;
    int64_t mt = ntiles > 0 ? ntiles : max_tiles_for(d);
    int64_t nck = (d->max_steps + d->ckpt_every - 1) / d->ckpt_every;
    size_t off = 0;
    const bool lane = lane_mode(d);
    L->tile_start = off; off += align256(sizeof(int64_t) * (mt + 1));
    L->lead = off; off += align256((size_t)n);
    // lane mode only: tile-local state history (idm_internal.h), sized for the plan's tiles
    L->vt_stride = lane ? (int64_t)(d->max_steps + 1) * kCap : 0;
    L->ck_stride = lane ? (nck + 1) * kCkRows * kCap : 0;  // + the final gap's row (kGapCk)
    L->sg_stride = lane ? sgn_words_per_tile(d->max_steps) : 0;
    L->vt = off; if (lane) off += align256(sizeof(float) * ((size_t)(mt * L->vt_stride) + 64));
    L->ckt = off; off += align256(sizeof(float) * (size_t)(mt * L->ck_stride));
    L->sgn = off; off += align256(sizeof(uint32_t) * (size_t)(mt * L->sg_stride));
    // virtual-leader mode only: speed and displacement checkpoints every 4 steps
    L->ckpt_v = off; if (!lane) off += align256(sizeof(float) * (size_t)(nck * n));
    L->ckpt_d = off; if (!lane) off += align256(sizeof(float) * (size_t)(nck * n));
    L->loss_partials = off;
    int64_t np_ = kLossBlocks > mt ? kLossBlocks : mt;
    if (vl_blocks(n) > np_) np_ = vl_blocks(n);
    off += align256(sizeof(double) * np_);
    L->loss_scalar = off; off += align256(sizeof(double));
    L->shared_partials = off;  // per-lane gradient sums, unless the caller gives lane_grads
    if (d->param_mode == IDM_PARAMS_SHARED && !d->lane_grads)
        off += align256(sizeof(double) * 6 * (size_t)d->n_lanes);
    L->status = off; off += align256(sizeof(unsigned long long));
    L->flags = off; off += align256(sizeof(unsigned));
    L->adam_table = off; off += align256(sizeof(float) * 2 * kFitMaxIters);
    L->tile_ready = off; off += align256(sizeof(unsigned) * (size_t)mt);  // fused-step handoff
    L->done_count = off; off += align256(sizeof(unsigned));  // fused-step last-CTA ticket
    L->total = off;
    return true;
}

Consts consts_of(const idm_desc& d) {
    Consts k;
    k.dt = d.dt;
    k.inv_dt = 1.0f / d.dt;
    k.a_min = d.a_min;
    k.eps = d.eps_gap;
    k.dt_ln2 = (float)((double)d.dt * 0.6931471805599453);
    k.a_min2 = (float)((double)d.a_min * 1.4426950408889634);
    k.ninv_dt2 = (float)(-1.4426950408889634 / (double)d.dt);
    k.dt_amin = d.dt * d.a_min;  // fp32 product, as the device would round it
    k.dt2 = d.dt * d.dt;
    return k;
}

// Reads and clears the device status word; returns IDM_OK / IDM_ENUMERIC / IDM_EINVAL.
int consume_status(idm_handle* h, unsigned long long st) {
    if (st == ~0ull) return IDM_OK;
    unsigned hi = (unsigned)(st >> 32), lo = (unsigned)(st & 0xffffffffu);
    if (hi == kBadInput)
        return fail(h, IDM_EINVAL, "invalid initial state at vehicle %u (non-finite, v < 0 or "
                                   "length < 0)", lo);
    if (hi == kBadDelta)
        return fail(h, IDM_EINVAL, "delta of vehicle %u is not 4 but the handle was specialised for "
                                   "delta = 4 at idm_init (delta frozen by opt_mask); re-create "
                                   "the handle after changing delta", lo);
    if (hi == kBadParam)
        return fail(h, IDM_EINVAL, "invalid IDM parameter %u of vehicle %lld (must be finite "
                                   "and > 0)", (unsigned)(lo / (h->n_par)),
                    (long long)(lo % h->n_par));
    if (hi == kBadOrder)
        return fail(h, IDM_EINVAL, "vehicle %u is not strictly behind its leader %u in its lane "
                                   "(gap pos0[i+1] - pos0[i] - length[i+1] <= 0: lanes must be "
                                   "sorted by ascending position without overlap)", lo, lo + 1);
    if (hi == kBadGrad)
        return fail(h, IDM_ENUMERIC, "non-finite gradient of IDM parameter %u of vehicle %lld",
                    (unsigned)(lo / (h->n_par)), (long long)(lo % h->n_par));
    return fail(h, IDM_ENUMERIC, "non-finite state detected at step %u (checkpoint), vehicle %u",
                hi, lo);
}

// Launch timing: events around a launch on the handle's stream (no-op unless enabled).
cudaEvent_t pool_event(idm_handle* h) {
    if (!h->ev_pool->empty()) {
        cudaEvent_t e = h->ev_pool->back();
        h->ev_pool->pop_back();
        return e;
    }
    cudaEvent_t e = nullptr;
    cudaEventCreate(&e);
    return e;
}
struct TimedLaunch {
    idm_handle* h;
    int kind;
    cudaStream_t st;
    cudaEvent_t a = nullptr, b = nullptr;
    TimedLaunch(idm_handle* h_, int kind_, cudaStream_t st_ = nullptr)
        : h(h_), kind(kind_), st(st_ ? st_ : h_->st) {
        if (h->timing) {
            a = pool_event(h);
            b = pool_event(h);
            cudaEventRecord(a, st);
        }
    }
    ~TimedLaunch() {
        if (h->timing && a && b) {
            cudaEventRecord(b, st);
            h->ev_rec->push_back({kind, {a, b}});
        }
    }
};

// Tile chunks of the fused iteration (IDM_FUSED_CHUNKS, default 1 = no split).
int fused_chunks(const idm_handle* h) {
    static const int env = [] {
        const char* e = std::getenv("IDM_FUSED_CHUNKS");
        return e ? std::atoi(e) : 1;
    }();
    int c = env < 1 ? 1 : (env > 16 ? 16 : env);
    if (h->csize > 1) return 1;  // chunks would split clusters
    return c > h->ntiles ? h->ntiles : c;
}

// Backward of idm_fit_step as a programmatic dependent launch of the forward (per-tile handoff,
// idm_kernels.cu "tile handoff"); IDM_PDL=0 turns it off.  Not with tile chunks (the backward runs
// on the second stream there) nor under launch timing (events between the two kernels).
bool use_pdl(const idm_handle* h, int nch) {
    static const bool env = [] {
        const char* e = std::getenv("IDM_PDL");
        return !(e && e[0] == '0');
    }();
    return env && nch == 1 && !h->timing && h->csize <= 1;  // not with clusters (long lanes)
}

int sync_status(idm_handle* h) {
    CK(h, cudaMemcpyAsync(&h->pinned[1], h->status, sizeof(unsigned long long),
                          cudaMemcpyDeviceToHost, h->st));
    CK(h, cudaStreamSynchronize(h->st));
    unsigned long long st;
    std::memcpy(&st, &h->pinned[1], sizeof(st));
    if (st != ~0ull) {
        CK(h, cudaMemsetAsync(h->status, 0xff, sizeof(unsigned long long), h->st));
        return consume_status(h, st);
    }
    return IDM_OK;
}

VlArgs vl_args(idm_handle* h, int32_t steps) {
    VlArgs a;
    std::memset(&a, 0, sizeof(a));
    a.pos0 = h->d.pos0;
    a.vel0 = h->d.vel0;
    a.params = h->d.params;
    a.n = h->n;
    a.n_par = h->n_par;
    a.steps = steps;
    a.max_steps = h->d.max_steps;
    a.ckpt_every = h->d.ckpt_every;
    a.k = consts_of(h->d);
    a.vl_dp = h->d.vl_dp;
    a.vl_dv = h->d.vl_dv;
    a.vl_grad = h->d.vl_grad;
    a.vl_adam_m = h->d.vl_adam_m;
    a.vl_adam_v = h->d.vl_adam_v;
    a.traj = h->d.traj;
    a.vel_traj = h->d.vel_traj;
    a.grad_traj = h->d.grad_traj;
    a.state_out = h->d.state_out;
    a.ckpt_v = h->ckpt_v;
    a.ckpt_d = h->ckpt_d;
    a.grad_params = h->d.grad_params;
    a.grad_state0 = h->d.grad_state0;
    a.loss_partials = h->loss_partials;
    a.status = h->status;
    return a;
}

bool is_vl(const idm_handle* h) { return h->d.leader_mode == IDM_LEADER_VIRTUAL; }

// Makes the handle's device current for the duration of one C-ABI call and restores the
// caller's (the handle's stream, workspace and kernels all belong to that device).
struct OnDevice {
    int prev = -1;
    bool switched = false;
    explicit OnDevice(const idm_handle* h) {
        if (h && h->device >= 0 && cudaGetDevice(&prev) == cudaSuccess && prev != h->device)
            switched = cudaSetDevice(h->device) == cudaSuccess;
    }
    ~OnDevice() {
        if (switched) cudaSetDevice(prev);
    }
};

}  // namespace

extern "C" {

int64_t idm_plan_tiles(const int32_t* lane_offsets, int32_t n_lanes, int64_t n_vehicles,
                       int64_t* tile_start) {
    if (!lane_offsets || n_lanes < 1 || n_vehicles < 1) return -1;
    std::vector<int32_t> off(lane_offsets, lane_offsets + (size_t)n_lanes + 1);
    std::vector<int64_t> tiles;
    std::string err;
    const int64_t nt = plan_tiles(off, n_lanes, n_vehicles, &tiles, nullptr, &err);
    if (nt >= 0 && tile_start) std::memcpy(tile_start, tiles.data(), sizeof(int64_t) * tiles.size());
    return nt;
}

size_t idm_workspace_bytes(const idm_desc* d) {
    Layout L;
    return layout_for(d, tiles_of(d), &L) ? L.total : 0;
}

int32_t idm_max_lane_vehicles(void) { return kCap; }

int32_t idm_max_lane_length(void) { return kMaxCluster * kCap; }

int idm_state_from_obs(const float* obs, int64_t n_vehicles, int32_t steps, float dt,
                       float* pos0, float* vel0, void* stream) {
    if (!obs || !pos0 || !vel0 || n_vehicles < 1 || steps < 0 || !(dt > 0.f) ||
        !std::isfinite(dt))
        return IDM_EINVAL;
    if (launch_state_from_obs(obs, n_vehicles, steps, dt, pos0, vel0, (cudaStream_t)stream) !=
        cudaSuccess)
        return IDM_ECUDA;
    return IDM_OK;
}

const char* idm_last_error(const idm_handle* h) { return h ? h->err : kNoHandle; }

int64_t idm_launch_count(const idm_handle* h) { return h ? h->launches : 0; }

void idm_destroy(idm_handle* h) {
    if (!h) return;
    OnDevice on_dev(h);
    if (h->st) cudaStreamSynchronize(h->st);
    if (h->ev_rec) {
        for (auto& r : *h->ev_rec) {
            cudaEventDestroy(r.second.first);
            cudaEventDestroy(r.second.second);
        }
        delete h->ev_rec;
    }
    if (h->ev_pool) {
        for (auto e : *h->ev_pool) cudaEventDestroy(e);
        delete h->ev_pool;
    }
    if (h->copy_st) cudaStreamDestroy(h->copy_st);
    if (h->graph_exec) cudaGraphExecDestroy(h->graph_exec);
    if (h->cap_st) cudaStreamDestroy(h->cap_st);
    if (h->ev_gfork) cudaEventDestroy(h->ev_gfork);
    if (h->ev_gjoin) cudaEventDestroy(h->ev_gjoin);
    if (h->st2) cudaStreamDestroy(h->st2);
    if (h->ev_fork) cudaEventDestroy(h->ev_fork);
    if (h->ev_join) cudaEventDestroy(h->ev_join);
    for (cudaEvent_t e : h->ev_chunk)
        if (e) cudaEventDestroy(e);
    if (h->ev_obs) cudaEventDestroy(h->ev_obs);
    if (h->ev_loss_done) cudaEventDestroy(h->ev_loss_done);
    if (h->ev_loss_done2) cudaEventDestroy(h->ev_loss_done2);
    for (int q = 0; q < 2; ++q)
        if (h->ev_step[q]) cudaEventDestroy(h->ev_step[q]);
    if (h->pinned) cudaFreeHost(h->pinned);
    if (h->adam_table_host) cudaFreeHost(h->adam_table_host);
    delete h;
}

int idm_init(idm_handle** out, const idm_desc* d) {
    if (!out) return IDM_EINVAL;
    *out = nullptr;
    idm_handle* h = new idm_handle();
    std::memset(h, 0, sizeof(*h));
    h->ev_pool = new std::vector<cudaEvent_t>();
    h->ev_rec = new std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>>();
    int rc = IDM_OK;
    auto bail = [&](int code) { rc = code; };
    do {
        Layout L;
        if (!d) { bail(fail(h, IDM_EINVAL, "NULL descriptor")); break; }
        h->d = *d;
        if (!layout_for(d, -1, &L)) {
            bail(fail(h, IDM_EINVAL, "malformed descriptor (need N >= 1, L >= 1, max_steps >= 1, "
                                     "ckpt_every in {2, 4, 8})"));
            break;
        }
        if (!(d->dt > 0.f) || !(d->a_min < 0.f) || !(d->eps_gap > 0.f) || !std::isfinite(d->dt) ||
            !std::isfinite(d->a_min) || !std::isfinite(d->eps_gap)) {
            bail(fail(h, IDM_EINVAL, "need dt > 0, a_min < 0, eps_gap > 0 (finite)"));
            break;
        }
        if (d->param_mode != IDM_PARAMS_PER_VEHICLE && d->param_mode != IDM_PARAMS_SHARED) {
            bail(fail(h, IDM_EINVAL, "bad param_mode %d", d->param_mode));
            break;
        }
        if (d->leader_mode != IDM_LEADER_LANE && d->leader_mode != IDM_LEADER_VIRTUAL) {
            bail(fail(h, IDM_EINVAL, "bad leader_mode %d", d->leader_mode));
            break;
        }
        if (d->leader_mode == IDM_LEADER_VIRTUAL &&
            (!d->vl_dp || !d->vl_dv || !d->vl_grad || !d->vl_adam_m || !d->vl_adam_v ||
             d->ckpt_every != 4 || d->param_mode != IDM_PARAMS_PER_VEHICLE)) {
            bail(fail(h, IDM_EINVAL, "virtual-leader mode needs vl_dp, vl_dv, vl_grad, vl_adam_m, "
                                     "vl_adam_v, ckpt_every == 4 and per-vehicle parameters"));
            break;
        }
        if (!d->lane_offsets || !d->pos0 || !d->vel0 || !d->length || !d->params ||
            !d->grad_params || !d->adam_m || !d->adam_v || !d->grad_traj || !d->traj) {
            bail(fail(h, IDM_EINVAL, "required device array is NULL"));
            break;
        }
        h->device = -1;
        // ---- lane plan on the host (cold path); the workspace is sized for its tile count.
        // Virtual-leader mode has no lanes (every trajectory alone): no plan.
        cudaError_t ce = cudaSuccess;
        std::vector<int64_t> tiles;
        std::vector<uint8_t> lead((size_t)d->n_vehicles, 0);
        int64_t nt = 1;
        if (lane_mode(d)) {
            std::vector<int32_t> off((size_t)d->n_lanes + 1);
            ce = cudaMemcpyAsync(off.data(), d->lane_offsets, sizeof(int32_t) * off.size(),
                                 cudaMemcpyDefault, (cudaStream_t)d->stream);
            if (ce == cudaSuccess) ce = cudaStreamSynchronize((cudaStream_t)d->stream);
            if (ce != cudaSuccess) {
                bail(fail(h, IDM_ECUDA, "reading lane_offsets: %s", cudaGetErrorString(ce)));
                break;
            }
            std::string perr;
            int num_sms = 148, dv = 0;
            if (cudaGetDevice(&dv) == cudaSuccess)
                cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, dv);
            cudaGetLastError();
            const int64_t chunk =
                split_chunk_for(off, d->n_lanes, d->n_vehicles, d->max_steps, num_sms);
            nt = plan_tiles(off, d->n_lanes, d->n_vehicles, &tiles, &lead, &perr, &h->csize,
                            chunk);
            if (nt < 0) {
                bail(fail(h, IDM_EINVAL, "%s", perr.c_str()));
                break;
            }
            if (h->csize > 1 && d->ckpt_every != 4) {
                bail(fail(h, IDM_EINVAL, "lanes longer than %d vehicles (thread-block clusters) "
                                         "need ckpt_every == 4", kCap));
                break;
            }
        } else {
            tiles = {0, d->n_vehicles};
            h->csize = 1;
        }
        if (!layout_for(d, nt, &L)) {
            bail(fail(h, IDM_EINVAL, "internal: tile plan exceeds bound"));
            break;
        }
        if (!d->workspace || d->workspace_bytes < L.total || ((uintptr_t)d->workspace & 255)) {
            bail(fail(h, IDM_EINVAL, "workspace must be >= %zu bytes and 256-byte aligned",
                      L.total));
            break;
        }
        int dev = -1;
        ce = cudaGetDevice(&dev);
        cudaDeviceProp prop;
        if (ce == cudaSuccess) ce = cudaGetDeviceProperties(&prop, dev);
        if (ce != cudaSuccess) {
            bail(fail(h, IDM_ECUDA, "no CUDA device: %s", cudaGetErrorString(ce)));
            break;
        }
        if (prop.major != 10) {
            bail(fail(h, IDM_ECUDA, "device %s is sm_%d%d; this library is built for sm_100a",
                      prop.name, prop.major, prop.minor));
            break;
        }
        h->device = dev;
        h->st = (cudaStream_t)d->stream;
        h->n = d->n_vehicles;
        h->n_par = d->param_mode == IDM_PARAMS_SHARED ? 1 : d->n_vehicles;
        char* ws = (char*)d->workspace;
        h->tile_start = (int64_t*)(ws + L.tile_start);
        h->lead = (uint8_t*)(ws + L.lead);
        h->vt = (float*)(ws + L.vt);
        h->ckt = (float*)(ws + L.ckt);
        h->vt_stride = L.vt_stride;
        h->ck_stride = L.ck_stride;
        h->sgn = (uint32_t*)(ws + L.sgn);
        h->sg_stride = L.sg_stride;
        h->ckpt_v = (float*)(ws + L.ckpt_v);
        h->ckpt_d = (float*)(ws + L.ckpt_d);
        h->loss_partials = (double*)(ws + L.loss_partials);
        h->loss_scalar = (double*)(ws + L.loss_scalar);
        h->lane_grads = d->lane_grads ? d->lane_grads : (double*)(ws + L.shared_partials);
        h->status = (unsigned long long*)(ws + L.status);
        h->flags = (unsigned*)(ws + L.flags);
        h->adam_table = (float*)(ws + L.adam_table);
        h->tile_ready = (unsigned*)(ws + L.tile_ready);
        h->done_count = (unsigned*)(ws + L.done_count);
        h->epoch = 0;

        h->nck = (int)((d->max_steps + d->ckpt_every - 1) / d->ckpt_every);

        h->ntiles = (int)nt;
        const char* what = "upload tile plan";
        ce = cudaMemcpyAsync(h->tile_start, tiles.data(), sizeof(int64_t) * tiles.size(),
                             cudaMemcpyHostToDevice, h->st);
        if (ce == cudaSuccess) {
            what = "upload leader flags";
            ce = cudaMemcpyAsync(h->lead, lead.data(), lead.size(), cudaMemcpyHostToDevice, h->st);
        }
        if (ce == cudaSuccess) { what = "memset status"; ce = cudaMemsetAsync(h->status, 0xff, 8, h->st); }
        if (ce == cudaSuccess) { what = "memset loss"; ce = cudaMemsetAsync(h->loss_scalar, 0, 8, h->st); }
        if (ce == cudaSuccess) { what = "memset flags"; ce = cudaMemsetAsync(h->flags, 0, 4, h->st); }
        if (ce == cudaSuccess) {
            what = "memset tile handoff";
            ce = cudaMemsetAsync(h->tile_ready, 0, sizeof(unsigned) * (size_t)nt, h->st);
        }
        if (ce == cudaSuccess) {
            what = "memset ticket";
            ce = cudaMemsetAsync(h->done_count, 0, sizeof(unsigned), h->st);
        }
        if (ce == cudaSuccess) { what = "smem attributes"; ce = kernels_configure(d->ckpt_every); }
        if (ce == cudaSuccess) {
            what = "device attributes";
            int dev = 0;
            ce = cudaGetDevice(&dev);
            if (ce == cudaSuccess)
                ce = cudaDeviceGetAttribute(&h->num_sms, cudaDevAttrMultiProcessorCount, dev);
        }
        if (ce == cudaSuccess) {
            what = "copy stream";
            ce = cudaStreamCreateWithFlags(&h->copy_st, cudaStreamNonBlocking);
        }
        if (ce == cudaSuccess) {
            what = "events";
            ce = cudaEventCreateWithFlags(&h->ev_obs, cudaEventDisableTiming);
        }
        if (ce == cudaSuccess)
            ce = cudaEventCreateWithFlags(&h->ev_loss_done, cudaEventDisableTiming);
            if (ce == cudaSuccess)
                ce = cudaEventCreateWithFlags(&h->ev_loss_done2, cudaEventDisableTiming);
        if (ce == cudaSuccess) {
            what = "chunk stream / events";
            ce = cudaStreamCreateWithFlags(&h->st2, cudaStreamNonBlocking);
            if (ce == cudaSuccess) ce = cudaEventCreateWithFlags(&h->ev_fork, cudaEventDisableTiming);
            if (ce == cudaSuccess) ce = cudaEventCreateWithFlags(&h->ev_join, cudaEventDisableTiming);
            for (cudaEvent_t& e : h->ev_chunk)
                if (ce == cudaSuccess) ce = cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
            if (ce == cudaSuccess) ce = cudaStreamCreateWithFlags(&h->cap_st, cudaStreamNonBlocking);
            if (ce == cudaSuccess) ce = cudaEventCreateWithFlags(&h->ev_gfork, cudaEventDisableTiming);
            for (int q = 0; q < 2 && ce == cudaSuccess; ++q)
                ce = cudaEventCreateWithFlags(&h->ev_step[q], cudaEventDisableTiming);
            if (ce == cudaSuccess) ce = cudaEventCreateWithFlags(&h->ev_gjoin, cudaEventDisableTiming);
        }
        if (ce == cudaSuccess) {
            what = "pinned buffer";
            // [0] loss, [1] status, [2] flags, [4..5] / [6..7] loss / status of the async ring
            ce = cudaMallocHost((void**)&h->pinned, 8 * sizeof(double));
        }
        if (ce != cudaSuccess) {
            bail(fail(h, IDM_ECUDA, "init (%s): %s", what, cudaGetErrorString(ce)));
            break;
        }
        ValidateArgs va{d->pos0,  d->vel0,      d->length, d->params, lane_mode(d) ? h->lead : nullptr,
                        h->n,     h->n_par, h->status, h->flags};
        ce = launch_validate(va, h->st);
        h->launches++;
        if (ce != cudaSuccess) {
            bail(fail(h, IDM_ECUDA, "validate launch: %s", cudaGetErrorString(ce)));
            break;
        }
        ce = cudaMemcpyAsync(&h->pinned[2], h->flags, sizeof(unsigned), cudaMemcpyDeviceToHost,
                             h->st);
        if (ce != cudaSuccess) {
            bail(fail(h, IDM_ECUDA, "init (flags): %s", cudaGetErrorString(ce)));
            break;
        }
        int s = sync_status(h);  // synchronizes (also keeps tiles/lead host vectors alive)
        if (s != IDM_OK) { bail(s); break; }
        unsigned fl;
        std::memcpy(&fl, &h->pinned[2], sizeof(fl));
        h->delta4 = fl == 0 && !((d->opt_mask >> 5) & 1u);

    } while (0);
    if (rc != IDM_OK) {
        // keep the message reachable: the caller gets no handle, so print it
        fprintf(stderr, "idm_init: %s\n", h->err);
        idm_destroy(h);
        return rc;
    }
    *out = h;
    return IDM_OK;
}

namespace {
FwdArgs fwd_args(idm_handle* h, int32_t steps) {
    FwdArgs a;
    std::memset(&a, 0, sizeof(a));
    a.tile_start = h->tile_start;
    a.lead = h->lead;
    a.pos0 = h->d.pos0;
    a.vel0 = h->d.vel0;
    a.length = h->d.length;
    a.params = h->d.params;
    a.n = h->n;
    a.n_par = h->n_par;
    a.state_out = h->d.state_out;
    a.vt = h->vt;
    a.ckt = h->ckt;
    a.vt_stride = h->vt_stride;
    a.ck_stride = h->ck_stride;
    a.sgn = h->sgn;
    a.sg_stride = h->sg_stride;
    a.steps = steps;
    a.ckpt_every = h->d.ckpt_every;
    a.k = consts_of(h->d);
    a.status = h->status;
    return a;
}

BwdArgs bwd_args(idm_handle* h, int32_t steps) {
    BwdArgs a;
    std::memset(&a, 0, sizeof(a));
    a.tile_start = h->tile_start;
    a.lead = h->lead;
    a.params = h->d.params;
    a.n = h->n;
    a.n_par = h->n_par;
    a.vt = h->vt;
    a.ckt = h->ckt;
    a.vt_stride = h->vt_stride;
    a.ck_stride = h->ck_stride;
    a.sgn = h->sgn;
    a.sg_stride = h->sg_stride;
    a.grad_params = h->d.grad_params;
    a.grad_state0 = h->d.grad_state0;
    a.lane_offsets = h->d.lane_offsets;
    a.n_lanes = h->d.n_lanes;
    a.lane_grads = h->lane_grads;
    a.steps = steps;
    a.ckpt_every = h->d.ckpt_every;
    a.k = consts_of(h->d);
    a.status = h->status;
    return a;
}
}  // namespace

int idm_forward(idm_handle* h, int32_t steps) { return idm_forward_ex(h, steps, 0u); }

int idm_forward_ex(idm_handle* h, int32_t steps, uint32_t flags) {
    if (!h) return IDM_EINVAL;
    OnDevice on_dev(h);
    if (steps < 1 || steps > h->d.max_steps)
        return fail(h, IDM_EINVAL, "steps=%d outside [1, max_steps=%d]", steps, h->d.max_steps);
    if (flags & ~(uint32_t)IDM_FWD_NO_HISTORY)
        return fail(h, IDM_EINVAL, "unknown idm_forward_ex flags 0x%x", flags);
    const bool hist = !(flags & IDM_FWD_NO_HISTORY);
    if (is_vl(h)) {
        VlArgs va = vl_args(h, steps);
        {
            TimedLaunch tl(h, IDM_K_FWD);
            CK(h, launch_vl_fwd(va, h->delta4, 0, h->st));
        }
        h->launches++;
        h->steps = steps;
        h->stage = 1;
        h->hist_ok = true;  // (its speed checkpoints are a small fraction of the traffic)
        return IDM_OK;
    }
    FwdArgs a = fwd_args(h, steps);
    a.traj = h->d.traj;
    a.vel_traj = h->d.vel_traj;
    FwdVariant var;
    var.delta4 = h->delta4;
    var.kahan = steps > 2000;  // compensated displacement for long horizons (C3)
    var.rec_v = h->d.vel_traj != nullptr;
    var.loss = 0;
    var.hist = hist;
    var.csize = h->csize;
    {
        TimedLaunch tl(h, IDM_K_FWD);
        CK(h, launch_fwd(a, h->ntiles, var, h->st));
    }
    h->launches++;
    h->steps = steps;
    h->stage = 1;
    h->hist_ok = hist;
    return IDM_OK;
}

int idm_loss_grad(idm_handle* h, const float* obs, const uint8_t* mask, int32_t kind,
                  double* loss_dev, double* loss_host) {
    if (!h) return IDM_EINVAL;
    OnDevice on_dev(h);
    if (h->stage < 1) return fail(h, IDM_ESTATE, "idm_loss_grad before idm_forward");
    if (!obs) return fail(h, IDM_EINVAL, "obs is NULL");
    if (kind != IDM_LOSS_L1 && kind != IDM_LOSS_L2)
        return fail(h, IDM_EINVAL, "bad loss kind %d", kind);
    LossArgs a;
    a.traj = h->d.traj;
    a.obs = obs;
    a.mask = mask;
    a.grad = h->d.grad_traj;
    a.n_elem = (int64_t)(h->steps + 1) * h->n;
    a.kind = kind;
    a.partials = h->loss_partials;
    {
        TimedLaunch tl(h, IDM_K_LOSS);
        CK(h, launch_loss(a, kLossBlocks, h->st));
    }
    {
        TimedLaunch tl(h, IDM_K_REDUCE);
        CK(h, launch_reduce(h->loss_partials, kLossBlocks, 1, h->loss_scalar, nullptr, h->st));
    }
    h->launches += 2;
    if (loss_dev)
        CK(h, cudaMemcpyAsync(loss_dev, h->loss_scalar, sizeof(double), cudaMemcpyDeviceToDevice,
                              h->st));
    h->stage = 2;
    if (loss_host) {
        CK(h, cudaMemcpyAsync(&h->pinned[0], h->loss_scalar, sizeof(double),
                              cudaMemcpyDeviceToHost, h->st));
        int s = sync_status(h);
        *loss_host = h->pinned[0];
        if (s != IDM_OK) return s;
    }
    return IDM_OK;
}

int idm_backward(idm_handle* h) {
    if (!h) return IDM_EINVAL;
    OnDevice on_dev(h);
    if (h->stage < 2) return fail(h, IDM_ESTATE, "idm_backward before idm_loss_grad");
    if (!h->hist_ok)
        return fail(h, IDM_ESTATE, "idm_backward after a forward without state history "
                                   "(IDM_FWD_NO_HISTORY): run idm_forward");
    if (is_vl(h)) {
        VlArgs va = vl_args(h, h->steps);
        {
            TimedLaunch tl(h, IDM_K_BWD);
            CK(h, launch_vl_bwd(va, h->delta4, false, h->st));
        }
        h->launches++;
        h->stage = 3;
        return IDM_OK;
    }
    BwdArgs a = bwd_args(h, h->steps);
    a.grad_traj = h->d.grad_traj;
    bool shared = h->d.param_mode == IDM_PARAMS_SHARED;
    std::memset(&a.adam, 0, sizeof(a.adam));
    if (shared)  // rows of empty lanes stay 0
        CK(h, cudaMemsetAsync(h->lane_grads, 0, sizeof(double) * 6 * (size_t)h->d.n_lanes, h->st));
    {
        TimedLaunch tl(h, IDM_K_BWD);
        CK(h, launch_bwd(a, h->ntiles, h->delta4, shared, false, 0, false, h->st, false,
                         h->csize));
    }
    h->launches++;
    if (shared) {  // this handle's lanes (one rank: the whole sum; ranks: idm_reduce_shared)
        TimedLaunch tl(h, IDM_K_REDUCE);
        CK(h, launch_reduce(h->lane_grads, h->d.n_lanes, 6, nullptr, h->d.grad_params, h->st));
        h->launches++;
    }
    h->stage = 3;
    return IDM_OK;
}

int idm_reduce_shared(idm_handle* h, const double* lane_grads, int64_t n_rows) {
    if (!h) return IDM_EINVAL;
    OnDevice on_dev(h);
    if (h->d.param_mode != IDM_PARAMS_SHARED)
        return fail(h, IDM_EINVAL, "idm_reduce_shared needs shared-parameter mode");
    if (!lane_grads || n_rows < h->d.n_lanes)
        return fail(h, IDM_EINVAL, "idm_reduce_shared: lane_grads NULL or fewer rows (%lld) "
                                   "than this handle's lanes (%d)", (long long)n_rows,
                    h->d.n_lanes);
    if (h->stage < 3) return fail(h, IDM_ESTATE, "idm_reduce_shared before idm_backward");
    {
        TimedLaunch tl(h, IDM_K_REDUCE);
        CK(h, launch_reduce(lane_grads, n_rows, 6, nullptr, h->d.grad_params, h->st));
    }
    h->launches++;
    return IDM_OK;
}

}  // extern "C"

namespace {
// Adam + schedule arguments of iteration `iter` (R#14-R#16).
AdamArgs make_adam(idm_handle* h, int32_t iter, int32_t total_iters, float lr0, float lr1) {
    const double b1 = 0.9, b2 = 0.999;
    double lr = total_iters > 1 ? lr0 + (double)(lr1 - lr0) * iter / (double)(total_iters - 1)
                                : lr0;
    double bc1 = 1.0 - std::pow(b1, iter + 1);
    double bc2 = 1.0 - std::pow(b2, iter + 1);
    AdamArgs a;
    a.x = h->d.params;
    a.m = h->d.adam_m;
    a.v = h->d.adam_v;
    a.grad = h->d.grad_params;
    a.n_par = h->n_par;
    a.opt_mask = h->d.opt_mask;
    a.step_size = (float)(lr / bc1);
    a.sqrt_bc2 = (float)std::sqrt(bc2);
    a.beta1 = (float)b1;
    a.beta2 = (float)b2;
    a.eps = 1e-8f;
    a.status = h->status;
    // boxes of PAPER.md:208 in parameter order (a_max, a_pref, s_min, T_pref, v_targ)
    const float lo[5] = {5.f, 0.1f, 1.f, 0.1f, 20.f}, hi[5] = {10.f, 5.f, 10.f, 5.f, 60.f};
    for (int q = 0; q < 5; ++q) { a.lo[q] = lo[q]; a.hi[q] = hi[q]; }
    return a;
}
}  // namespace

extern "C" {

}  // extern "C"

namespace {
// Adam over the virtual-leader leaves of the last `steps` rows (dp plane, dv plane).
int adam_leaves(idm_handle* h, const AdamArgs& a) {
    const int64_t kn = (int64_t)h->d.max_steps * h->n, n = (int64_t)h->steps * h->n;
    TimedLaunch tl(h, IDM_K_ADAM);
    CK(h, launch_adam_free(h->d.vl_dp, h->d.vl_grad, h->d.vl_adam_m, h->d.vl_adam_v, n, a, h->st));
    CK(h, launch_adam_free(h->d.vl_dv, h->d.vl_grad + kn, h->d.vl_adam_m + kn,
                           h->d.vl_adam_v + kn, n, a, h->st));
    h->launches += 2;
    return IDM_OK;
}
}  // namespace

extern "C" {

int idm_adam_step(idm_handle* h, int32_t iter, int32_t total_iters, float lr0, float lr1) {
    if (!h) return IDM_EINVAL;
    OnDevice on_dev(h);
    if (h->stage < 3) return fail(h, IDM_ESTATE, "idm_adam_step before idm_backward");
    if (iter < 0 || total_iters < 1 || iter >= total_iters)
        return fail(h, IDM_EINVAL, "iter=%d outside [0, total_iters=%d)", iter, total_iters);
    AdamArgs a = make_adam(h, iter, total_iters, lr0, lr1);
    {
        TimedLaunch tl(h, IDM_K_ADAM);
        CK(h, launch_adam(a, h->st));
    }
    h->launches++;
    if (is_vl(h)) {
        int s = adam_leaves(h, a);
        if (s != IDM_OK) return s;
    }
    h->stage = 0;  // parameters changed: a new forward is required
    return IDM_OK;
}

int idm_fit_step(idm_handle* h, int32_t steps, const float* obs, const uint8_t* mask,
                 int32_t kind, int32_t iter, int32_t total_iters, float lr0, float lr1,
                 double* loss_dev, double* loss_host) {
    if (!h) return IDM_EINVAL;
    OnDevice on_dev(h);
    if (steps < 1 || steps > h->d.max_steps)
        return fail(h, IDM_EINVAL, "steps=%d outside [1, max_steps=%d]", steps, h->d.max_steps);
    if (!obs) return fail(h, IDM_EINVAL, "obs is NULL");
    if (mask)
        return fail(h, IDM_EINVAL, "idm_fit_step takes no mask: mark missing observations as NaN");
    if (kind != IDM_LOSS_L1 && kind != IDM_LOSS_L2)
        return fail(h, IDM_EINVAL, "bad loss kind %d", kind);
    if (iter < 0 || total_iters < 1 || iter >= total_iters)
        return fail(h, IDM_EINVAL, "iter=%d outside [0, total_iters=%d)", iter, total_iters);
    if (is_vl(h)) {
        VlArgs va = vl_args(h, steps);
        va.obs = obs;
        va.adam = make_adam(h, iter, total_iters, lr0, lr1);
        // the forward writes only speed and displacement checkpoints; the backward derives
        // Eq. 4 and dL/dP from obs and the rebuilt positions (no dL/dP rows through HBM)
        {
            TimedLaunch tl(h, IDM_K_FWD);
            CK(h, launch_vl_fwd(va, h->delta4, 3, h->st));
        }
        {
            TimedLaunch tl(h, IDM_K_BWD);
            CK(h, launch_vl_bwd(va, h->delta4, true, h->st, kind));
        }
        {
            TimedLaunch tl(h, IDM_K_REDUCE);
            CK(h, launch_reduce(h->loss_partials, vl_blocks(h->n), 1, h->loss_scalar, nullptr,
                                h->st));
        }
        h->launches += 3;  // the leaves' Adam runs in the backward's reverse sweep
        h->steps = steps;
        h->stage = 0;
        if (loss_dev)
            CK(h, cudaMemcpyAsync(loss_dev, h->loss_scalar, sizeof(double),
                                  cudaMemcpyDeviceToDevice, h->st));
        if (loss_host) {
            CK(h, cudaMemcpyAsync(&h->pinned[0], h->loss_scalar, sizeof(double),
                                  cudaMemcpyDeviceToHost, h->st));
            int st2 = sync_status(h);
            *loss_host = h->pinned[0];
            if (st2 != IDM_OK) return st2;
        }
        return IDM_OK;
    }
    // Latency-bound shapes (a few lane tiles, long horizon: C3's 6 tiles x 27,000 steps) run
    // faster as the defining sequence: there each warp's in-order instruction stream sets the
    // pace, and the fused forward's Eq. 4 work lengthens it (C3: 11.8 vs 12.6 ms).
    const bool latency_bound = 2 * h->ntiles <= h->num_sms && steps >= 1000 && h->d.traj &&
                               h->d.grad_traj && !std::getenv("IDM_FUSED_ALWAYS");
    if (h->d.ckpt_every != 4 || latency_bound) {
        // the fused kernels are specialised to 4-step segments; any other interval (and a
        // latency-bound shape) runs the defining sequence itself (same arithmetic, same bits)
        int s = idm_forward(h, steps);
        if (s == IDM_OK) s = idm_loss_grad(h, obs, nullptr, kind, loss_dev, nullptr);
        if (s == IDM_OK) s = idm_backward(h);
        if (s == IDM_OK) s = idm_adam_step(h, iter, total_iters, lr0, lr1);
        if (s != IDM_OK) return s;
        if (!((h->d.opt_mask >> 5) & 1u))  // dL/d delta of a frozen delta is not reported
            CK(h, cudaMemsetAsync(h->d.grad_params + 5 * h->n_par, 0, h->n_par * sizeof(float),
                                  h->st));
        if (loss_host) {
            CK(h, cudaMemcpyAsync(&h->pinned[0], h->loss_scalar, sizeof(double),
                                  cudaMemcpyDeviceToHost, h->st));
            int st2 = sync_status(h);
            *loss_host = h->pinned[0];
            if (st2 != IDM_OK) return st2;
        }
        return IDM_OK;
    }
    // forward + Eq. 4 value fused (the state history goes to the tile-local rows; no P or
    // dL/dP round trip through HBM)
    FwdArgs f = fwd_args(h, steps);
    f.obs = obs;
    f.kind = kind;
    f.loss_partials = h->loss_partials;
    FwdVariant var;
    var.delta4 = h->delta4;
    var.kahan = steps > 2000;
    var.rec_v = false;
    var.csize = h->csize;
    // Two schemes, same arithmetic: the forward sums Eq. 4 and records the L1 sign codes (L1
    // default: 2 bits per vehicle-step cross to the backward), or the forward writes only the
    // tile history and the backward derives Eq. 4 from obs and the rebuilt positions (L2
    // default: L2's dL/dP needs the residual, so obs would otherwise be read twice).  C4: L1
    // 2.61 (codes) vs 2.75 ms, L2 3.13 vs 2.70 ms (obs).  IDM_FUSED_OBS_BWD=0/1 forces one.
    static const int obs_env = [] {
        const char* e = std::getenv("IDM_FUSED_OBS_BWD");
        return e ? (e[0] == '1' ? 1 : 0) : -1;
    }();
    // lanes over clusters: always the history-only forward (its observation-staging variants
    // are not built with the cluster channel, idm_kernels.cu launch_fwd_k)
    const bool obs_bwd = h->csize > 1 || (obs_env >= 0 ? obs_env == 1 : kind == 1);
    var.loss = obs_bwd ? 3 : 1 + kind;
    const int gobs = obs_bwd ? (kind == 0 ? 3 : 2) : 1 + kind;
    h->steps = steps;
    // backward: dL/dP from the forward's sign words (L1) or re-derived from obs and rebuilt
    // positions (L2); per-vehicle parameters get Adam in the same kernel's epilogue
    BwdArgs b = bwd_args(h, steps);
    b.obs = obs;
    b.pos0 = h->d.pos0;
    b.adam = make_adam(h, iter, total_iters, lr0, lr1);
    const bool shared = h->d.param_mode == IDM_PARAMS_SHARED;
    // Tiles are independent, so the iteration can run in tile chunks: the backward of chunk c
    // (second stream) overlaps the forward of chunk c + 1; every chunk does the same
    // arithmetic on the same tiles, so the results do not depend on the chunking.
    const int nch = fused_chunks(h);
    cudaStream_t sb = nch > 1 ? h->st2 : h->st;
    const bool pdl = use_pdl(h, nch);
    if (!obs_bwd) {  // the loss: summed by the forward's last CTA (no reduce launch)
        f.loss_out = h->loss_scalar;
        f.done_count = h->done_count;
        f.n_tiles = h->ntiles;
    } else {  // per-tile losses from the backward, then one fixed-order reduction
        b.loss_partials = h->loss_partials;
    }
    if (pdl) {
        f.tile_ready = h->tile_ready;
        b.tile_ready = h->tile_ready;
        if (++h->epoch == 0) h->epoch = 1;  // 0 = never signalled
        f.epoch = b.epoch = h->epoch;
    }
    if (shared)  // rows of empty lanes stay 0 (before the forward: the backward follows it directly)
        CK(h, cudaMemsetAsync(h->lane_grads, 0, sizeof(double) * 6 * (size_t)h->d.n_lanes, h->st));
    if (nch > 1) {
        CK(h, cudaEventRecord(h->ev_fork, h->st));
        CK(h, cudaStreamWaitEvent(h->st2, h->ev_fork, 0));
    }
    for (int c = 0; c < nch; ++c) {
        const int t0 = (int)((int64_t)h->ntiles * c / nch);
        const int t1 = (int)((int64_t)h->ntiles * (c + 1) / nch);
        if (t1 <= t0) continue;
        f.tile0 = t0;
        b.tile0 = t0;
        {
            TimedLaunch tl(h, IDM_K_FWD);
            CK(h, launch_fwd(f, t1 - t0, var, h->st));
        }
        if (nch > 1) {
            CK(h, cudaEventRecord(h->ev_chunk[c], h->st));
            CK(h, cudaStreamWaitEvent(h->st2, h->ev_chunk[c], 0));
        }
        {
            TimedLaunch tl(h, IDM_K_BWD, sb);
            CK(h, launch_bwd(b, t1 - t0, h->delta4, shared, !shared, gobs, var.kahan, sb, pdl,
                             h->csize));
        }
        h->launches += 2;
    }
    if (nch > 1) {
        CK(h, cudaEventRecord(h->ev_join, h->st2));
        CK(h, cudaStreamWaitEvent(h->st, h->ev_join, 0));
    }
    if (obs_bwd) {
        TimedLaunch tl(h, IDM_K_REDUCE);
        CK(h, launch_reduce(h->loss_partials, h->ntiles, 1, h->loss_scalar, nullptr, h->st));
        h->launches++;
    }
    if (shared) {
        {
            TimedLaunch tl(h, IDM_K_REDUCE);
            CK(h, launch_reduce(h->lane_grads, h->d.n_lanes, 6, nullptr, h->d.grad_params,
                                h->st));
        }
        {
            TimedLaunch tl(h, IDM_K_ADAM);
            CK(h, launch_adam(b.adam, h->st));
        }
        h->launches += 2;
    }
    h->stage = 0;
    if (loss_dev)
        CK(h, cudaMemcpyAsync(loss_dev, h->loss_scalar, sizeof(double), cudaMemcpyDeviceToDevice,
                              h->st));
    if (loss_host) {
        CK(h, cudaMemcpyAsync(&h->pinned[0], h->loss_scalar, sizeof(double),
                              cudaMemcpyDeviceToHost, h->st));
        int st2 = sync_status(h);
        *loss_host = h->pinned[0];
        if (st2 != IDM_OK) return st2;
    }
    return IDM_OK;
}

int32_t idm_fit_max_steps(void) { return kFitMaxSteps; }

int idm_fit_steps(idm_handle* h, int32_t steps, const float* obs, int32_t kind, int32_t iter0,
                  int32_t iters, int32_t total_iters, float lr0, float lr1, double* loss_dev,
                  double* loss_host) {
    if (!h) return IDM_EINVAL;
    OnDevice on_dev(h);
    if (iters < 1 || iter0 < 0 || (int64_t)iter0 + iters > total_iters)
        return fail(h, IDM_EINVAL, "idm_fit_steps: iterations %d..%d outside [0, %d)", iter0,
                    iter0 + iters - 1, total_iters);
    // the iteration loop as ONE CUDA graph: capture `iters` idm_fit_step calls on the handle's
    // stream (each with its own schedule step baked into its kernel nodes), launch it once
    if (h->graph_exec) {
        CK(h, cudaStreamSynchronize(h->cap_st));  // the previous graph may still be running
        cudaGraphExecDestroy(h->graph_exec);
        h->graph_exec = nullptr;
    }
    // capture on the handle's private stream, ordered after the work already queued on the
    // handle's stream (fork before the capture), and order the handle's stream after the
    // graph (join)
    cudaStream_t orig = h->st;
    CK(h, cudaEventRecord(h->ev_gfork, orig));
    CK(h, cudaStreamWaitEvent(h->cap_st, h->ev_gfork, 0));
    const bool timing = h->timing;
    h->timing = false;  // no timing events inside a capture
    h->st = h->cap_st;
    cudaError_t ce = cudaStreamBeginCapture(h->st, cudaStreamCaptureModeThreadLocal);
    if (ce != cudaSuccess) {
        h->st = orig;
        h->timing = timing;
        return fail(h, IDM_ECUDA, "graph capture: %s", cudaGetErrorString(ce));
    }
    int rc = IDM_OK;
    for (int32_t it = iter0; it < iter0 + iters && rc == IDM_OK; ++it)
        rc = idm_fit_step(h, steps, obs, nullptr, kind, it, total_iters, lr0, lr1,
                          it + 1 == iter0 + iters ? loss_dev : nullptr, nullptr);
    cudaGraph_t graph = nullptr;
    ce = cudaStreamEndCapture(h->st, &graph);
    h->st = orig;
    h->timing = timing;
    if (rc != IDM_OK) {
        if (graph) cudaGraphDestroy(graph);
        return rc;
    }
    if (ce == cudaSuccess) ce = cudaGraphInstantiate(&h->graph_exec, graph, 0);
    if (graph) cudaGraphDestroy(graph);
    if (ce == cudaSuccess) ce = cudaGraphLaunch(h->graph_exec, h->cap_st);
    if (ce == cudaSuccess) ce = cudaEventRecord(h->ev_gjoin, h->cap_st);
    if (ce == cudaSuccess) ce = cudaStreamWaitEvent(orig, h->ev_gjoin, 0);
    if (ce != cudaSuccess) return fail(h, IDM_ECUDA, "graph launch: %s", cudaGetErrorString(ce));
    if (loss_host) {
        CK(h, cudaMemcpyAsync(&h->pinned[0], h->loss_scalar, sizeof(double),
                              cudaMemcpyDeviceToHost, h->st));
        int st2 = sync_status(h);
        *loss_host = h->pinned[0];
        if (st2 != IDM_OK) return st2;
    }
    return IDM_OK;
}

int idm_fit(idm_handle* h, int32_t steps, const float* obs, int32_t kind, int32_t iter0,
            int32_t iters, int32_t total_iters, float lr0, float lr1, double* loss_dev,
            double* loss_host) {
    if (!h) return IDM_EINVAL;
    OnDevice on_dev(h);
    if (steps < 1 || steps > h->d.max_steps)
        return fail(h, IDM_EINVAL, "idm_fit: steps=%d outside [1, max_steps=%d]", steps,
                    h->d.max_steps);
    const bool on_chip = steps <= kFitMaxSteps;  // else the long-horizon kernel (NEXT-4)
    if (!on_chip && h->d.ckpt_every != 4)
        return fail(h, IDM_EINVAL, "idm_fit beyond %d steps needs ckpt_every == 4", kFitMaxSteps);
    if (!obs) return fail(h, IDM_EINVAL, "obs is NULL");
    if (kind != IDM_LOSS_L1 && kind != IDM_LOSS_L2)
        return fail(h, IDM_EINVAL, "bad loss kind %d", kind);
    if (is_vl(h) || h->d.param_mode != IDM_PARAMS_PER_VEHICLE)
        return fail(h, IDM_EINVAL, "idm_fit supports lane-leader mode with per-vehicle parameters");
    if (h->csize > 1)
        return fail(h, IDM_EINVAL, "idm_fit: lanes longer than %d vehicles are not supported (use "
                                   "idm_fit_step)", kCap);
    if (iters < 1 || iters > kFitMaxIters || iter0 < 0 || iter0 + iters > total_iters)
        return fail(h, IDM_EINVAL, "idm_fit: iterations [%d, %d) outside [0, total_iters=%d) or "
                                   "more than %d per call", iter0, iter0 + iters, total_iters,
                    kFitMaxIters);
    if (!h->adam_table_host)
        CK(h, cudaMallocHost((void**)&h->adam_table_host, sizeof(float) * 2 * kFitMaxIters));
    // the host-side schedule of idm_adam_step, one entry per iteration (bit-identical values)
    CK(h, cudaStreamSynchronize(h->st));  // the staging buffer may still feed a prior copy
    for (int j = 0; j < iters; ++j) {
        AdamArgs ad = make_adam(h, iter0 + j, total_iters, lr0, lr1);
        h->adam_table_host[2 * j] = ad.step_size;
        h->adam_table_host[2 * j + 1] = ad.sqrt_bc2;
    }
    CK(h, cudaMemcpyAsync(h->adam_table, h->adam_table_host, sizeof(float) * 2 * iters,
                          cudaMemcpyHostToDevice, h->st));
    AdamArgs ad = make_adam(h, iter0, total_iters, lr0, lr1);
    if (!on_chip) {
        // every iteration in one launch, each CTA its tile's whole fit (fit_long_kernel): the
        // arguments of idm_fit_step's two kernels, without the programmatic handoff
        FwdArgs f = fwd_args(h, steps);
        f.obs = obs;
        f.kind = kind;
        f.loss_partials = h->loss_partials;
        if (kind == IDM_LOSS_L1) {  // the forward's last CTA sums the last iteration's loss
            f.loss_out = h->loss_scalar;
            f.done_count = h->done_count;
            f.n_tiles = h->ntiles;
        }
        BwdArgs b = bwd_args(h, steps);
        b.obs = obs;
        b.pos0 = h->d.pos0;
        b.adam = ad;
        if (kind == IDM_LOSS_L2) b.loss_partials = h->loss_partials;
        FitLongArgs fl;
        fl.iters = iters;
        fl.adam_table = h->adam_table;
        {
            TimedLaunch tl(h, IDM_K_FWD);
            CK(h, launch_fit_long(f, b, fl, h->ntiles, h->delta4, steps > 2000, kind, h->st));
        }
        h->launches++;
        if (kind == IDM_LOSS_L2) {
            TimedLaunch tl(h, IDM_K_REDUCE);
            CK(h, launch_reduce(h->loss_partials, h->ntiles, 1, h->loss_scalar, nullptr, h->st));
            h->launches++;
        }
        h->steps = steps;
        h->stage = 0;
        if (loss_dev)
            CK(h, cudaMemcpyAsync(loss_dev, h->loss_scalar, sizeof(double),
                                  cudaMemcpyDeviceToDevice, h->st));
        if (loss_host) {
            CK(h, cudaMemcpyAsync(&h->pinned[0], h->loss_scalar, sizeof(double),
                                  cudaMemcpyDeviceToHost, h->st));
            int st2 = sync_status(h);
            *loss_host = h->pinned[0];
            if (st2 != IDM_OK) return st2;
        }
        return IDM_OK;
    }
    FitArgs a;
    a.tile_start = h->tile_start;
    a.lead = h->lead;
    a.pos0 = h->d.pos0;
    a.vel0 = h->d.vel0;
    a.length = h->d.length;
    a.obs = obs;
    a.params = h->d.params;
    a.adam_m = h->d.adam_m;
    a.adam_v = h->d.adam_v;
    a.grad_params = h->d.grad_params;
    a.grad_state0 = h->d.grad_state0;
    a.n = h->n;
    a.steps = steps;
    a.iters = iters;
    a.opt_mask = h->d.opt_mask;
    a.k = consts_of(h->d);
    a.adam_table = h->adam_table;
    a.beta1 = ad.beta1;
    a.beta2 = ad.beta2;
    a.eps = ad.eps;
    for (int q = 0; q < 5; ++q) { a.lo[q] = ad.lo[q]; a.hi[q] = ad.hi[q]; }
    a.loss_partials = h->loss_partials;
    a.status = h->status;
    {
        TimedLaunch tl(h, IDM_K_FWD);
        CK(h, launch_fit(a, h->ntiles, h->delta4, kind, h->st));
    }
    {
        TimedLaunch tl(h, IDM_K_REDUCE);
        CK(h, launch_reduce(h->loss_partials, h->ntiles, 1, h->loss_scalar, nullptr, h->st));
    }
    h->launches += 2;
    h->steps = steps;
    h->stage = 0;
    if (loss_dev)
        CK(h, cudaMemcpyAsync(loss_dev, h->loss_scalar, sizeof(double), cudaMemcpyDeviceToDevice,
                              h->st));
    if (loss_host) {
        CK(h, cudaMemcpyAsync(&h->pinned[0], h->loss_scalar, sizeof(double),
                              cudaMemcpyDeviceToHost, h->st));
        int st2 = sync_status(h);
        *loss_host = h->pinned[0];
        if (st2 != IDM_OK) return st2;
    }
    return IDM_OK;
}

int idm_timing_enable(idm_handle* h, int enable) {
    if (!h) return IDM_EINVAL;
    OnDevice on_dev(h);
    h->timing = enable != 0;
    return IDM_OK;
}

int idm_timing_read(idm_handle* h, double* ms, int64_t* launches) {
    if (!h) return IDM_EINVAL;
    OnDevice on_dev(h);
    double acc[IDM_NKERNELS] = {0};
    int64_t cnt[IDM_NKERNELS] = {0};
    for (auto& r : *h->ev_rec) {
        CK(h, cudaEventSynchronize(r.second.second));
        float t = 0.f;
        CK(h, cudaEventElapsedTime(&t, r.second.first, r.second.second));
        acc[r.first] += t;
        cnt[r.first] += 1;
        h->ev_pool->push_back(r.second.first);
        h->ev_pool->push_back(r.second.second);
    }
    h->ev_rec->clear();
    for (int i = 0; i < IDM_NKERNELS; ++i) {
        if (ms) ms[i] = acc[i];
        if (launches) launches[i] = cnt[i];
    }
    return IDM_OK;
}

int idm_check(idm_handle* h) {
    if (!h) return IDM_EINVAL;
    OnDevice on_dev(h);
    CK(h, cudaGetLastError());
    return sync_status(h);
}

}  // extern "C"

namespace {
// idm_step_host without the final read: uploads, then forward -> loss -> backward -> Adam.
int step_host_enqueue(idm_handle* h, int32_t steps, const float* pos0_host, const float* vel0_host,
                      const float* obs_host, const uint8_t* mask_host, int32_t kind, int32_t iter,
                      int32_t total_iters, float lr0, float lr1) {
    if (!obs_host) return fail(h, IDM_EINVAL, "obs_host is NULL");
    if (!h->d.obs_stage || (mask_host && !h->d.mask_stage))
        return fail(h, IDM_EINVAL, "idm_step_host needs desc.obs_stage (and mask_stage)");
    if (steps < 1 || steps > h->d.max_steps)
        return fail(h, IDM_EINVAL, "steps=%d outside [1, max_steps=%d]", steps, h->d.max_steps);
    size_t nb = sizeof(float) * (size_t)h->n;
    size_t ob = sizeof(float) * (size_t)(steps + 1) * (size_t)h->n;
    if (pos0_host) CK(h, cudaMemcpyAsync(h->d.pos0, pos0_host, nb, cudaMemcpyHostToDevice, h->st));
    if (vel0_host) CK(h, cudaMemcpyAsync(h->d.vel0, vel0_host, nb, cudaMemcpyHostToDevice, h->st));
    // staging: alternate obs_stage / obs_stage2 when both exist (and no mask: one mask stage);
    // the upload waits for the last loss kernel that read its buffer, overlaps the forward
    const int sb = (h->d.obs_stage2 && !mask_host) ? h->stage_next : 0;
    h->stage_next = h->d.obs_stage2 ? sb ^ 1 : 0;
    float* stage = sb ? h->d.obs_stage2 : h->d.obs_stage;
    cudaEvent_t ev_done = sb ? h->ev_loss_done2 : h->ev_loss_done;
    CK(h, cudaStreamWaitEvent(h->copy_st, ev_done, 0));
    CK(h, cudaMemcpyAsync(stage, obs_host, ob, cudaMemcpyHostToDevice, h->copy_st));
    if (mask_host)
        CK(h, cudaMemcpyAsync(h->d.mask_stage, mask_host, (size_t)(steps + 1) * (size_t)h->n,
                              cudaMemcpyHostToDevice, h->copy_st));
    CK(h, cudaEventRecord(h->ev_obs, h->copy_st));
    int s = idm_forward(h, steps);
    if (s) return s;
    CK(h, cudaStreamWaitEvent(h->st, h->ev_obs, 0));
    s = idm_loss_grad(h, stage, mask_host ? h->d.mask_stage : nullptr, kind, nullptr, nullptr);
    if (s) return s;
    CK(h, cudaEventRecord(ev_done, h->st));
    s = idm_backward(h);
    if (s) return s;
    return idm_adam_step(h, iter, total_iters, lr0, lr1);
}
}  // namespace

extern "C" {

int idm_step_host(idm_handle* h, int32_t steps, const float* pos0_host, const float* vel0_host,
                  const float* obs_host, const uint8_t* mask_host, int32_t kind, int32_t iter,
                  int32_t total_iters, float lr0, float lr1, double* loss_host) {
    if (!h) return IDM_EINVAL;
    OnDevice on_dev(h);
    int s = step_host_enqueue(h, steps, pos0_host, vel0_host, obs_host, mask_host, kind, iter,
                              total_iters, lr0, lr1);
    if (s) return s;
    CK(h, cudaMemcpyAsync(&h->pinned[0], h->loss_scalar, sizeof(double), cudaMemcpyDeviceToHost,
                          h->st));
    s = sync_status(h);
    if (loss_host) *loss_host = h->pinned[0];
    return s;
}

int idm_step_host_async(idm_handle* h, int32_t steps, const float* pos0_host,
                        const float* vel0_host, const float* obs_host, const uint8_t* mask_host,
                        int32_t kind, int32_t iter, int32_t total_iters, float lr0, float lr1) {
    if (!h) return IDM_EINVAL;
    OnDevice on_dev(h);
    if (h->async_n >= 2)
        return fail(h, IDM_ESTATE, "two idm_step_host_async steps in flight: call "
                                   "idm_step_host_wait first");
    int s = step_host_enqueue(h, steps, pos0_host, vel0_host, obs_host, mask_host, kind, iter,
                              total_iters, lr0, lr1);
    if (s) return s;
    const int slot = (h->async_head + h->async_n) % 2;
    CK(h, cudaMemcpyAsync(&h->pinned[4 + slot], h->loss_scalar, sizeof(double),
                          cudaMemcpyDeviceToHost, h->st));
    CK(h, cudaMemcpyAsync(&h->pinned[6 + slot], h->status, sizeof(unsigned long long),
                          cudaMemcpyDeviceToHost, h->st));
    CK(h, cudaEventRecord(h->ev_step[slot], h->st));
    h->async_n++;
    return IDM_OK;
}

int idm_step_host_wait(idm_handle* h, double* loss_host) {
    if (!h) return IDM_EINVAL;
    OnDevice on_dev(h);
    if (h->async_n == 0) return fail(h, IDM_ESTATE, "no idm_step_host_async step in flight");
    const int slot = h->async_head;
    CK(h, cudaEventSynchronize(h->ev_step[slot]));
    h->async_head = (h->async_head + 1) % 2;
    h->async_n--;
    if (loss_host) *loss_host = h->pinned[4 + slot];
    unsigned long long st;
    std::memcpy(&st, &h->pinned[6 + slot], sizeof(st));
    if (st != ~0ull) {  // drain the pipeline, then report (and clear) the status as idm_check
        CK(h, cudaStreamSynchronize(h->st));
        h->async_n = 0;
        CK(h, cudaMemsetAsync(h->status, 0xff, sizeof(unsigned long long), h->st));
        CK(h, cudaStreamSynchronize(h->st));
        return consume_status(h, st);
    }
    return IDM_OK;
}

}  // extern "C"
