// Measured ceiling of the max-norm inner loop on this GPU.
//
// The FP32 roofline of the sweeps is not in MEASURED_PEAKS.json (that file
// holds HBM copy and bf16 GEMM peaks).  This kernel runs the ideal inner
// loop of the sweeps -- candidates broadcast from shared memory, packed
// FADD2 differences folded by 3-input FMNMX with |.| modifiers, 4 reference
// points per thread, no compares -- so its pair-coordinate rate is the
// practical peak the sweeps are measured against (bench.py reports both it
// and the nominal 128 lanes x 2 ops x clock figure).
#include <cuda_runtime.h>

#include "common.cuh"
#include "profile.cuh"

namespace ente {

constexpr int kMbDim = 8;
constexpr int kMbCands = 256;

__global__ void __launch_bounds__(128) pce_microbench_kernel(int iters, float *out) {
    __shared__ float4 cand[kMbCands * 2];
    for (int i = threadIdx.x; i < kMbCands * 2; i += blockDim.x)
        cand[i] = make_float4(i * 0.5f, i * 0.25f, -i * 0.125f, i * 1.5f);
    __syncthreads();
    float2 ref[4][kMbDim / 2];
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int p = 0; p < kMbDim / 2; ++p)
            ref[r][p] = make_float2(-(float)(threadIdx.x + r + p), -(float)(blockIdx.x + p));
    float acc[4] = {0.f, 0.f, 0.f, 0.f};
    for (int it = 0; it < iters; ++it) {
#pragma unroll 4
        for (int j = 0; j < kMbCands; ++j) {
            const float4 a = cand[2 * j], b = cand[2 * j + 1];
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                const float2 d0 = __fadd2_rn(ref[r][0], make_float2(a.x, a.y));
                const float2 d1 = __fadd2_rn(ref[r][1], make_float2(a.z, a.w));
                const float2 d2 = __fadd2_rn(ref[r][2], make_float2(b.x, b.y));
                const float2 d3 = __fadd2_rn(ref[r][3], make_float2(b.z, b.w));
                float m = fmaxf(fmaxf(fabsf(d0.x), fabsf(d0.y)), fabsf(d1.x));
                m = fmaxf(fmaxf(m, fabsf(d1.y)), fabsf(d2.x));
                m = fmaxf(fmaxf(m, fabsf(d2.y)), fabsf(d3.x));
                m = fmaxf(m, fabsf(d3.y));
                acc[r] = fminf(acc[r], m);  // keeps the result live (one op per pair)
            }
        }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc[0] + acc[1] + acc[2] + acc[3];
}

}  // namespace ente

using namespace ente;

// Runs the microbenchmark on `stream` and returns pair-coordinate evaluations
// per second (synchronises).  blocks <= 0 picks 8 CTAs per SM.
extern "C" int ente_microbench_pce(int iters, int blocks, double *pce_per_s, void *stream) {
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    int dev = 0, sms = 148;
    ENTE_CUDA(cudaGetDevice(&dev));
    ENTE_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    if (blocks <= 0) blocks = sms * 8;
    float *out = nullptr;
    ENTE_CUDA(cudaMalloc(&out, sizeof(float) * blocks * 128));
    cudaEvent_t a, b;
    ENTE_CUDA(cudaEventCreate(&a));
    ENTE_CUDA(cudaEventCreate(&b));
    pce_microbench_kernel<<<blocks, 128, 0, st>>>(1, out);  // warm-up
    ENTE_CUDA(cudaEventRecord(a, st));
    ENTE_LAUNCH("microbench_pce", st, pce_microbench_kernel<<<blocks, 128, 0, st>>>(iters, out));
    ENTE_CUDA(cudaEventRecord(b, st));
    ENTE_CUDA(cudaEventSynchronize(b));
    float ms = 0.f;
    ENTE_CUDA(cudaEventElapsedTime(&ms, a, b));
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    ENTE_CUDA(cudaFree(out));
    const double pce = (double)blocks * 128 * 4 * kMbDim * (double)kMbCands * iters;
    *pce_per_s = pce / (ms * 1e-3);
    return ENTE_OK;
}
