// FP32-pipe peak probe: the roofline denominator for the FP32-SIMT pair kernels (K5 / K7).
// MEASURED_PEAKS.json carries only HBM copy bandwidth and cuBLAS bf16; bench.py measures the
// sustained FFMA rate with this kernel on the same box, at the clocks of the timed run.
// 8 independent packed FFMA2 chains per thread (16 FMAs per step; FFMA2 reaches the FMA pipe's
// limit with half the issue slots of scalar FFMA: 74.2 vs 72.5 TFLOP/s measured on B200), so the
// denominator is the pipe's true peak; flops = 2 * 16 * 16 * iters per thread.
#include "ndg_common.cuh"

__global__ void __launch_bounds__(256) fp32_probe_kernel(float* out, int iters, float y, float z) {
    float2 a[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) a[u] = make_float2(threadIdx.x * 1e-3f + u, u + 0.5f);
    const float2 yy = make_float2(y, y), zz = make_float2(z, z);
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < 16; ++u)
#pragma unroll
            for (int v = 0; v < 8; ++v) a[v] = __ffma2_rn(yy, a[v], zz);
    }
    float s = 0.f;
#pragma unroll
    for (int u = 0; u < 8; ++u) s += a[u].x + a[u].y;
    if (s == 1234.5f) out[threadIdx.x] = s;   // keeps the chains alive, never true in practice
}

extern "C" int ndg_fp32_probe(float* out, int blocks, int iters, void* stream) {
    NDG_REQUIRE(blocks >= 1 && iters >= 1, "blocks and iters must be positive");
    fp32_probe_kernel<<<blocks, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(out, iters, 0.999999f, 1e-7f);
    NDG_CHECK_LAUNCH();
    return NDG_OK;
}

extern "C" double ndg_fp32_probe_flops(int blocks, int iters) { return 2.0 * 16 * 16 * (double)iters * 256 * blocks; }
