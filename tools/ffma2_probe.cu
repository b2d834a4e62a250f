// Microbenchmark: FP32 FMA throughput of scalar FFMA vs packed FFMA2 (sm_100a) on one B200.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void __launch_bounds__(256) p1(float* out, int iters, float y, float z) {
    float a[8];
    for (int u = 0; u < 8; ++u) a[u] = threadIdx.x * 1e-3f + u;
    for (int i = 0; i < iters; ++i)
#pragma unroll
        for (int u = 0; u < 16; ++u)
#pragma unroll
            for (int v = 0; v < 8; ++v) a[v] = fmaf(a[v], y, z);
    float s = 0; for (int u = 0; u < 8; ++u) s += a[u];
    if (s == 1234.5f) out[threadIdx.x] = s;
}
__global__ void __launch_bounds__(256) p2(float* out, int iters, float y, float z) {
    float2 a[8];
    for (int u = 0; u < 8; ++u) a[u] = make_float2(threadIdx.x * 1e-3f + u, u + 0.5f);
    for (int i = 0; i < iters; ++i)
#pragma unroll
        for (int u = 0; u < 16; ++u)
#pragma unroll
            for (int v = 0; v < 8; ++v) a[v] = __ffma2_rn(make_float2(y, y), a[v], make_float2(z, z));
    float s = 0; for (int u = 0; u < 8; ++u) s += a[u].x + a[u].y;
    if (s == 1234.5f) out[threadIdx.x] = s;
}
int main() {
    float* out; cudaMalloc(&out, 1024);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    int blocks = 148 * 8, iters = 4096;
    for (int which = 0; which < 2; ++which) {
        float best = 1e9;
        for (int r = 0; r < 6; ++r) {
            cudaEventRecord(a);
            if (which == 0) p1<<<blocks, 256>>>(out, iters, 0.999999f, 1e-7f);
            else p2<<<blocks, 256>>>(out, iters, 0.999999f, 1e-7f);
            cudaEventRecord(b); cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b); if (r && ms < best) best = ms;
        }
        double fmas = (double)blocks * 256 * iters * 16 * 8 * (which ? 2 : 1);
        printf("%s: %.3f ms  %.1f TFLOP/s\n", which ? "FFMA2" : "FFMA ", best, 2 * fmas / best / 1e9);
    }
    return 0;
}
