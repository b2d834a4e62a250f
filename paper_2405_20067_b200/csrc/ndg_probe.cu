// FP32-pipe peak probe: the roofline denominator for the FP32-SIMT pair kernels (K5 / K7).
// MEASURED_PEAKS.json carries only HBM copy bandwidth and cuBLAS bf16; bench.py measures the
// sustained FFMA rate with this kernel on the same box, at the clocks of the timed run.
// 8 independent 3-register FFMA chains per thread (enough ILP to cover the 4-cycle latency),
// 4 x 148 CTAs x 256 threads; flops = 2 * 8 * iters per thread.
#include "ndg_common.cuh"

__global__ void __launch_bounds__(256) fp32_probe_kernel(float* out, int iters, float y, float z) {
    float a0 = threadIdx.x * 1e-3f, a1 = a0 + 1.f, a2 = a0 + 2.f, a3 = a0 + 3.f;
    float a4 = a0 + 4.f, a5 = a0 + 5.f, a6 = a0 + 6.f, a7 = a0 + 7.f;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < 16; ++u) {
            a0 = fmaf(a0, y, z); a1 = fmaf(a1, y, z); a2 = fmaf(a2, y, z); a3 = fmaf(a3, y, z);
            a4 = fmaf(a4, y, z); a5 = fmaf(a5, y, z); a6 = fmaf(a6, y, z); a7 = fmaf(a7, y, z);
        }
    }
    float s = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
    if (s == 1234.5f) out[threadIdx.x] = s;   // keeps the chains alive, never true in practice
}

extern "C" int ndg_fp32_probe(float* out, int blocks, int iters, void* stream) {
    NDG_REQUIRE(blocks >= 1 && iters >= 1, "blocks and iters must be positive");
    fp32_probe_kernel<<<blocks, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(out, iters, 0.999999f, 1e-7f);
    NDG_CHECK_LAUNCH();
    return NDG_OK;
}

extern "C" double ndg_fp32_probe_flops(int blocks, int iters) { return 2.0 * 8 * 16 * (double)iters * 256 * blocks; }
