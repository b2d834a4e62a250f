// mma.sync throughput probe (sm_100a): m16n8k8 tf32 (round 1: is the legacy warp-level MMA fast enough to
// carry the N >= 13 backward's S = Z^T W Z accumulation in registers?) and m16n8k16 f16 (round 2: it
// issues at the same 0.467 MMA/clk/SM with twice the K, which K7-MMA now uses).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mma_sync_probe tools/mma_sync_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void mma_tf32(float (&d)[4], const unsigned (&a)[4], const unsigned (&b)[2]) {
    asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
                 "{%0,%1,%2,%3};\n"
                 : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
                 : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}

__device__ __forceinline__ void mma_f16(float (&d)[4], const unsigned (&a)[4], const unsigned (&b)[2]) {
    asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
                 "{%0,%1,%2,%3};\n"
                 : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
                 : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}

// m16n8k16 f16 inputs, f32 accumulation: twice the K of the tf32 shape per instruction
template <int ACC>
__global__ void probe16(float* out, int iters) {
    float d[ACC][4] = {};
    unsigned a[4], b[2];
    for (int i = 0; i < 4; ++i) a[i] = 0x3c003c00u + threadIdx.x + i;
    for (int i = 0; i < 2; ++i) b[i] = 0x38003800u + i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int k = 0; k < ACC; ++k) mma_f16(d[k], a, b);
    }
    float s = 0.f;
    for (int k = 0; k < ACC; ++k) s += d[k][0] + d[k][1] + d[k][2] + d[k][3];
    if (s == 12345.f) out[threadIdx.x] = s;
}

template <int ACC>
void run16(int warps_per_sm, float* out) {
    const int blocks = 148, threads = 32 * warps_per_sm, iters = 20000;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    probe16<ACC><<<blocks, threads>>>(out, 100);
    cudaEventRecord(a);
    probe16<ACC><<<blocks, threads>>>(out, iters);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    const double mmas = (double)blocks * warps_per_sm * iters * ACC;
    const double flops = mmas * 2 * 16 * 8 * 16;
    printf("mma.sync m16n8k16 f16   warps/SM %2d  acc/warp %d : %.2f TFLOP/s  %.3f mma/clk/SM (1.965 GHz)\n",
           warps_per_sm, ACC, flops / ms / 1e9, mmas / (ms * 1e-3) / 148 / 1.965e9);
}

template <int ACC>
__global__ void probe(float* out, int iters) {
    float d[ACC][4] = {};
    unsigned a[4], b[2];
    for (int i = 0; i < 4; ++i) a[i] = __float_as_uint(1.0f + threadIdx.x * 1e-3f + i);
    for (int i = 0; i < 2; ++i) b[i] = __float_as_uint(0.5f + i);
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int k = 0; k < ACC; ++k) mma_tf32(d[k], a, b);
    }
    float s = 0.f;
    for (int k = 0; k < ACC; ++k) s += d[k][0] + d[k][1] + d[k][2] + d[k][3];
    if (s == 12345.f) out[threadIdx.x] = s;
}

// FFMA reference on the same launch shape
__global__ void ffma(float* out, int iters) {
    float x[8];
    for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-3f + i;
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int i = 0; i < 8; ++i) x[i] = fmaf(x[i], 0.999f, 0.001f);
    float s = 0.f;
    for (int i = 0; i < 8; ++i) s += x[i];
    if (s == 12345.f) out[threadIdx.x] = s;
}

template <int ACC>
void run(int warps_per_sm, float* out) {
    const int blocks = 148, threads = 32 * warps_per_sm, iters = 20000;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    probe<ACC><<<blocks, threads>>>(out, 100);
    cudaEventRecord(a);
    probe<ACC><<<blocks, threads>>>(out, iters);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    const double mmas = (double)blocks * warps_per_sm * iters * ACC;
    const double flops = mmas * 2 * 16 * 8 * 8;
    printf("mma.sync m16n8k8 tf32  warps/SM %2d  acc/warp %d : %.2f TFLOP/s  %.3f mma/clk/SM (1.965 GHz)\n",
           warps_per_sm, ACC, flops / ms / 1e9, mmas / (ms * 1e-3) / 148 / 1.965e9);
}

int main() {
    float* out;
    cudaMalloc(&out, 4096);
    run<1>(4, out);
    run<2>(4, out);
    run<4>(4, out);
    run<2>(8, out);
    run<4>(8, out);
    run<4>(16, out);
    run<8>(16, out);
    run16<2>(8, out);
    run16<4>(8, out);
    run16<4>(16, out);
    run16<8>(16, out);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    ffma<<<148, 512>>>(out, 100);
    cudaEventRecord(a);
    ffma<<<148, 512>>>(out, 20000);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("FFMA reference: %.2f TFLOP/s\n", 148.0 * 512 * 20000 * 8 * 2 / ms / 1e9);
    return 0;
}
