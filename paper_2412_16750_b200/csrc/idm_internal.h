// idm_internal.h -- kernel argument blocks and launchers shared by idm_kernels.cu and idm_capi.cu.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "idm_device.cuh"

namespace idm {

// status word: UINT64_MAX = OK; otherwise (code_or_step << 32 | index), smallest wins.
constexpr unsigned kBadInput = 0xFFFFFFF0u;  // invalid pos0/vel0/length at vehicle index
constexpr unsigned kBadParam = 0xFFFFFFF1u;  // invalid parameter at flat index
constexpr unsigned kBadDelta = 0xFFFFFFF2u;  // delta != 4 in a delta=4-specialised kernel

struct ValidateArgs {
    const float *pos0, *vel0, *length, *params;
    int64_t n, n_par;
    unsigned long long* status;
    unsigned* delta_not4;
};

struct FwdVariant {
    bool delta4;  // every delta == 4 (two squarings instead of ex2/lg2)
    bool kahan;   // compensated displacement
    bool rec_v;   // record speeds
    int loss;     // 0, or fused Eq. 4 (1 = L1, 2 = L2): read obs, write dL/dP (idm_fit_step)
};

struct FwdArgs {
    const int64_t* tile_start;
    const uint8_t* lead;
    const float *pos0, *vel0, *length, *params;
    int64_t n, n_par;
    float *traj, *vel_traj, *state_out;
    float *ckpt_s, *ckpt_v;
    int steps, ckpt_every;
    Consts k;
    unsigned long long* status;
    // fused loss (LOSS variant)
    const float* obs;
    float* grad_traj;
    int kind;
    double* loss_partials;  // [ntiles]
};

struct AdamArgs {
    float *x, *m, *v;
    const float* grad;
    int64_t n_par;
    uint32_t opt_mask;
    float step_size, sqrt_bc2, beta1, beta2, eps;
    float lo[5], hi[5];
};

struct BwdArgs {
    const int64_t* tile_start;
    const uint8_t* lead;
    const float* params;
    int64_t n, n_par;
    const float* grad_traj;
    const float *ckpt_s, *ckpt_v;
    float *grad_params, *grad_state0;
    double* shared_partials;  // [ntiles][6] (shared mode)
    int steps, ckpt_every;
    Consts k;
    unsigned long long* status;
    AdamArgs adam;  // fused Adam epilogue (ADAM variant)
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
size_t bwd_smem_bytes(int ckpt_every);
cudaError_t launch_bwd(const BwdArgs& a, int ntiles, bool delta4, bool shared, bool adam,
                       cudaStream_t st);
bool ckpt_supported(int k);
cudaError_t launch_loss(const LossArgs& a, int nblocks, cudaStream_t st);
cudaError_t launch_reduce(const double* partials, int64_t n, int width, double* out, float* out_f,
                          cudaStream_t st);
cudaError_t launch_adam(const AdamArgs& a, cudaStream_t st);

constexpr int kLossBlocks = 148 * 8;  // fixed => deterministic loss reduction

}  // namespace idm
