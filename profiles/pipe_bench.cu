// pipe_bench.cu -- issue / pipe throughput microbenchmark behind the ALU roofline denominators
// (DESIGN.md section 4 "Roofline denominators"; bench.py `roofline`).
//
// Measures, on the GPU it runs on, the sustained per-SM rate of the instruction classes the
// IDM kernels are made of: scalar FP32 FFMA, packed FFMA2 (two lanes' FMAs per instruction,
// sm_100), FMUL2 / FADD2, the MUFU ops ex2 / lg2 / rcp (XU pipe), and FMNMX / selects.
// Each thread runs 8 independent dependency chains (enough to hide the pipe latency at 32 warps
// per SM), so the rate is the pipe's throughput.  Reported per SM per clock, in warp-instructions
// and in lane-operations, with the SM clock taken from clock64() inside the kernel (cycles) --
// so the result is independent of the clock the GPU happens to run at.
//
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o pipe_bench profiles/pipe_bench.cu
//   ./pipe_bench > profiles/rNN_pipe_bench.txt
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

constexpr int kChains = 8;
constexpr int kIters = 4096;
constexpr int kThreads = 256;
constexpr int kBlocksPerSM = 4;  // 32 warps per SM

enum Op { FFMA = 0, FFMA2, FMUL2, FADD2, EX2, LG2, RCP, FMNMX, MIX_FWD };
const char* kNames[] = {"FFMA (scalar)", "FFMA2 (packed f32x2)", "FMUL2 (packed)", "FADD2 (packed)",
                        "MUFU.EX2", "MUFU.LG2", "MUFU.RCP (+FADD)", "FMNMX", "mix 4 FFMA2 : 1 MUFU"};
// lane operations per instruction (packed ops do 2 per lane)
const int kLaneOps[] = {1, 2, 2, 2, 1, 1, 1, 1, 1};

__device__ __forceinline__ float ex2(float x) {
    float y;
    asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ float lg2(float x) {
    float y;
    asm volatile("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ float rcp(float x) {
    float y;
    asm volatile("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

template <int OP>
__global__ void __launch_bounds__(kThreads) bench(float* out, long long* cycles, float seed) {
    float a[kChains];
    float2 b[kChains];
#pragma unroll
    for (int c = 0; c < kChains; ++c) {
        a[c] = seed * (threadIdx.x + c + 1);
        b[c] = make_float2(a[c], a[c] + 1.f);
    }
    const float2 m2 = make_float2(0.999f, 0.998f), k2 = make_float2(1e-3f, 2e-3f);
    __syncthreads();
    const long long t0 = clock64();
    for (int it = 0; it < kIters; ++it) {
#pragma unroll
        for (int c = 0; c < kChains; ++c) {
            if (OP == FFMA) a[c] = __fmaf_rn(a[c], 0.999f, 1e-3f);
            if (OP == FFMA2) b[c] = __ffma2_rn(b[c], m2, k2);
            if (OP == FMUL2) b[c] = __fmul2_rn(b[c], m2);
            if (OP == FADD2) b[c] = __fadd2_rn(b[c], k2);
            if (OP == EX2) a[c] = ex2(a[c]);
            if (OP == LG2) a[c] = lg2(a[c]);
            if (OP == RCP) a[c] = rcp(a[c]) + 0.5f;  // (+ FADD: rcp(rcp(x)) would fold)
            if (OP == FMNMX) a[c] = fmaxf(a[c], a[(c + 1) % kChains]);
            if (OP == MIX_FWD) {
                b[c] = __ffma2_rn(b[c], m2, k2);
                b[c] = __ffma2_rn(b[c], m2, k2);
                b[c] = __ffma2_rn(b[c], m2, k2);
                b[c] = __ffma2_rn(b[c], m2, k2);
                a[c] = ex2(a[c]);
            }
        }
    }
    const long long t1 = clock64();
    __syncthreads();
    float s = 0.f;
#pragma unroll
    for (int c = 0; c < kChains; ++c) s += a[c] + b[c].x + b[c].y;
    out[blockIdx.x * kThreads + threadIdx.x] = s;
    if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
}

template <int OP>
void run(int sms, float* out, long long* cyc, long long* hcyc) {
    const int blocks = sms * kBlocksPerSM;
    bench<OP><<<blocks, kThreads>>>(out, cyc, 1e-3f);  // warm-up
    bench<OP><<<blocks, kThreads>>>(out, cyc, 1e-3f);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
        fprintf(stderr, "%s\n", cudaGetErrorString(e));
        exit(1);
    }
    cudaMemcpy(hcyc, cyc, sizeof(long long) * blocks, cudaMemcpyDeviceToHost);
    long long mx = 0;
    double mean = 0;
    for (int i = 0; i < blocks; ++i) {
        mx = hcyc[i] > mx ? hcyc[i] : mx;
        mean += hcyc[i];
    }
    mean /= blocks;
    const int per_iter = OP == MIX_FWD ? 5 : 1;  // instructions per chain per iteration
    // warp-instructions per SM over the slowest block's cycles (all blocks are co-resident)
    const double winst = (double)kBlocksPerSM * (kThreads / 32) * kIters * kChains * per_iter;
    const double ipc = winst / (double)mx;
    const double lane = OP == MIX_FWD ? (4.0 * 2 + 1) / 5.0 : kLaneOps[OP];
    printf("%-24s %8.3f warp-instr/clk/SM  %8.1f lane-ops/clk/SM  (cycles max %lld, mean %.0f)\n",
           kNames[OP], ipc, ipc * 32 * lane, mx, mean);
}

int main() {
    cudaDeviceProp p;
    cudaGetDeviceProperties(&p, 0);
    const int sms = p.multiProcessorCount;
    printf("device %s, sm_%d%d, %d SMs; %d blocks x %d threads per SM, %d chains/thread\n", p.name,
           p.major, p.minor, sms, kBlocksPerSM, kThreads, kChains);
    float* out;
    long long *cyc, *hcyc;
    cudaMalloc(&out, sizeof(float) * sms * kBlocksPerSM * kThreads);
    cudaMalloc(&cyc, sizeof(long long) * sms * kBlocksPerSM);
    hcyc = (long long*)malloc(sizeof(long long) * sms * kBlocksPerSM);
    run<FFMA>(sms, out, cyc, hcyc);
    run<FFMA2>(sms, out, cyc, hcyc);
    run<FMUL2>(sms, out, cyc, hcyc);
    run<FADD2>(sms, out, cyc, hcyc);
    run<EX2>(sms, out, cyc, hcyc);
    run<LG2>(sms, out, cyc, hcyc);
    run<RCP>(sms, out, cyc, hcyc);
    run<FMNMX>(sms, out, cyc, hcyc);
    run<MIX_FWD>(sms, out, cyc, hcyc);
    return 0;
}
