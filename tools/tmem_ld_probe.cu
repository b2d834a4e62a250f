// TMEM read throughput vs load shape, loads in flight per wait and warps per SM (sm_100a).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tmem_ld_probe tools/tmem_ld_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int X>
__device__ __forceinline__ void ldx(uint32_t taddr, uint32_t* r);
template <>
__device__ __forceinline__ void ldx<16>(uint32_t a, uint32_t* r) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                   "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
                 : "r"(a));
}
template <>
__device__ __forceinline__ void ldx<32>(uint32_t a, uint32_t* r) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
                 "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                   "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
                   "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
                   "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
                 : "r"(a));
}

// each warp: iters x (NL loads of X columns, then one wait); lane quarter = warp % 4
template <int X, int NL>
__global__ void ld_rate(int iters, float* out) {
    __shared__ uint32_t tbase;
    const int tid = threadIdx.x, warp = tid / 32;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tbase)),
                     "r"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t base = tbase + ((uint32_t)((warp % 4) * 32) << 16) + (uint32_t)(((warp / 4) * 128) % 384);
    float acc = 0.f;
    for (int i = 0; i < iters; ++i) {
        uint32_t r[X * NL];
#pragma unroll
        for (int l = 0; l < NL; ++l) ldx<X>(base + (uint32_t)((l * X) % 128), r + l * X);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int j = 0; j < X * NL; ++j) acc += __uint_as_float(r[j]);
    }
    if (acc == 12345.f) out[tid] = acc;
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase), "r"(512));
}

template <int X, int NL>
void run(int warps, float* out) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int iters = 4000;
    ld_rate<X, NL><<<148, warps * 32>>>(iters, out);
    cudaDeviceSynchronize();
    cudaEventRecord(a);
    ld_rate<X, NL><<<148, warps * 32>>>(iters, out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    double bytes = 4.0 * 32 * X * NL * (double)iters * warps * 148;
    printf("x%-2d NL=%d warps=%2d: %6.1f B/clk/SM (%s)\n", X, NL, warps, bytes / (ms * 1e-3) / 148 / 1.965e9,
           cudaGetErrorString(cudaGetLastError()));
}

int main() {
    float* out;
    cudaMalloc(&out, 1 << 16);
    for (int w : {4, 8, 12, 16}) {
        run<16, 1>(w, out);
        run<16, 4>(w, out);
        run<16, 7>(w, out);
        run<32, 1>(w, out);
        run<32, 2>(w, out);
        run<32, 4>(w, out);
    }
    return 0;
}
