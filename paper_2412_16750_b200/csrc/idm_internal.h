// idm_internal.h -- kernel argument blocks and launchers shared by idm_kernels.cu and idm_capi.cu.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "idm_device.cuh"

namespace idm {

// status word: UINT64_MAX = OK; otherwise (code_or_step << 32 | index), smallest wins.
constexpr unsigned kBadInput = 0xFFFFFFF0u;  // invalid pos0/vel0/length at vehicle index
constexpr unsigned kBadParam = 0xFFFFFFF1u;  // invalid parameter at flat index

struct ValidateArgs {
    const float *pos0, *vel0, *length, *params;
    int64_t n, n_par;
    unsigned long long* status;
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
};

struct LossArgs {
    const float *traj, *obs;
    const uint8_t* mask;
    float* grad;
    int64_t n_elem;
    int kind;
    double* partials;
};

struct AdamArgs {
    float *x, *m, *v;
    const float* grad;
    int64_t n_par;
    uint32_t opt_mask;
    float step_size, sqrt_bc2, beta1, beta2, eps;
    float lo[5], hi[5];
};

cudaError_t launch_validate(const ValidateArgs& a, cudaStream_t st);
cudaError_t launch_fwd(const FwdArgs& a, int ntiles, bool kahan, cudaStream_t st);
cudaError_t bwd_configure(int ckpt_every);
size_t bwd_smem_bytes(int ckpt_every);
cudaError_t launch_bwd(const BwdArgs& a, int ntiles, bool shared, cudaStream_t st);
cudaError_t launch_loss(const LossArgs& a, int nblocks, cudaStream_t st);
cudaError_t launch_reduce(const double* partials, int64_t n, int width, double* out, float* out_f,
                          cudaStream_t st);
cudaError_t launch_adam(const AdamArgs& a, cudaStream_t st);

constexpr int kLossBlocks = 148 * 8;  // fixed => deterministic loss reduction

}  // namespace idm
