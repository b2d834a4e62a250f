// tcgen05 probe (sm_100a): (1) correctness of a hand-encoded kind::tf32 MMA with K-major
// SWIZZLE_NONE smem descriptors and TMEM accumulators, (2) MMA throughput, (3) tcgen05.ld
// bandwidth. Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tc_probe tools/tc_probe.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// K-major, no swizzle: element (r, k) of an R x K fp32 tile at byte (r%8)*16 + (r/8)*SBO + (k/4)*LBO + (k%4)*4
// with LBO = 128 (adjacent K core matrices contiguous), SBO = (K/4)*128.
__host__ __device__ inline uint32_t kmaj_off(int r, int k, int K) {
    return (r % 8) * 16 + (r / 8) * ((K / 4) * 128) + (k / 4) * 128 + (k % 4) * 4;
}
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;                 // version = 1 (sm_100)
    return d;                               // base_offset 0, lbo_mode 0, layout SWIZZLE_NONE (0)
}
__host__ __device__ constexpr uint32_t idesc_tf32(int M, int N) {
    return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void mma_tf32(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc, int acc) {
    asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                 "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n"
                 :: "r"(d_tmem), "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" :: "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t c) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(smem_u32(bar)), "r"(c) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n"
                 :: "r"(smem_u32(bar)), "r"(parity) : "memory");
}
__device__ __forceinline__ void tmem_alloc(uint32_t* dst, uint32_t ncols) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" :: "r"(smem_u32(dst)), "r"(ncols) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" :: "r"(taddr), "r"(ncols) : "memory");
}
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, float* v) {
    uint32_t r[8];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    for (int i = 0; i < 8; ++i) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ void tmem_ld32_nowait(uint32_t taddr, uint32_t* r) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
                 "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                   "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
                   "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
                   "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
                 : "r"(taddr));
}

constexpr int M = 128, N = 64, K = 32;

// (1) D[m][n] = sum_k A[m][k] * B[n][k]   (A: M x K, B: N x K, both row-major in global)
__global__ void gemm_check(const float* A, const float* B, float* D) {
    extern __shared__ __align__(1024) uint8_t sm[];
    float* sA = (float*)sm;
    float* sB = (float*)(sm + M * K * 4);
    __shared__ uint64_t bar;
    __shared__ uint32_t tbase;
    int tid = threadIdx.x;
    for (int i = tid; i < M * K; i += blockDim.x) { int r = i / K, k = i % K; *(float*)((uint8_t*)sA + kmaj_off(r, k, K)) = A[i]; }
    for (int i = tid; i < N * K; i += blockDim.x) { int r = i / K, k = i % K; *(float*)((uint8_t*)sB + kmaj_off(r, k, K)) = B[i]; }
    if (tid < 32) tmem_alloc(&tbase, 64);
    if (tid == 0) { mbar_init(&bar, 1); asm volatile("fence.mbarrier_init.release.cluster;"); }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    uint32_t d = tbase;
    if (tid == 0) {
        const uint32_t sbo = (K / 4) * 128;
        for (int ks = 0; ks < K / 8; ++ks) {
            uint64_t a = make_desc(smem_u32(sA) + ks * 256, 128, sbo);
            uint64_t b = make_desc(smem_u32(sB) + ks * 256, 128, sbo);
            mma_tf32(d, a, b, idesc_tf32(M, N), ks > 0);
        }
        mma_commit(&bar);
    }
    mbar_wait(&bar, 0);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    int warp = tid / 32, lane = tid % 32;
    for (int c = 0; c < N; c += 8) {
        float v[8];
        tmem_ld8(d + ((uint32_t)(warp * 32) << 16) + c, v);
        for (int j = 0; j < 8; ++j) D[(warp * 32 + lane) * N + c + j] = v[j];
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (tid < 32) tmem_dealloc(tbase, 64);
}

// (2) MMA throughput: one thread issues `iters` x (M=128, N=NN, K=8) MMAs on resident operands.
template <int NN>
__global__ void mma_rate(int iters, float* out) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint64_t bar;
    __shared__ uint32_t tbase;
    int tid = threadIdx.x;
    for (int i = tid; i < (128 + NN) * 8; i += blockDim.x) ((float*)sm)[i] = 1e-3f * (i % 7);
    if (tid < 32) tmem_alloc(&tbase, NN);
    if (tid == 0) { mbar_init(&bar, 1); asm volatile("fence.mbarrier_init.release.cluster;"); }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (tid == 0) {
        uint64_t a = make_desc(smem_u32(sm), 128, 256);
        uint64_t b = make_desc(smem_u32(sm) + 128 * 8 * 4, 128, 256);
        for (int i = 0; i < iters; ++i) mma_tf32(tbase, a, b, idesc_tf32(128, NN), i > 0);
        mma_commit(&bar);
    }
    mbar_wait(&bar, 0);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    float v[8];
    tmem_ld8(tbase + ((uint32_t)((tid / 32) * 32) << 16), v);
    if (v[0] == 12345.f) out[tid] = v[1];
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (tid < 32) tmem_dealloc(tbase, NN);
}

// (3) tcgen05.ld bandwidth: 4 warps x iters x (32 lanes x 32 cols x 4 B) per CTA.
__global__ void ld_rate(int iters, float* out) {
    __shared__ uint32_t tbase;
    int tid = threadIdx.x;
    if (tid < 32) tmem_alloc(&tbase, 256);
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    uint32_t base = tbase + ((uint32_t)((tid / 32 % 4) * 32) << 16);
    float acc = 0.f;
    for (int i = 0; i < iters; ++i) {
        uint32_t r[32];
        tmem_ld32_nowait(base + (i & 7) * 32, r);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        for (int j = 0; j < 32; ++j) acc += __uint_as_float(r[j]);
    }
    if (acc == 12345.f) out[tid] = acc;
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (tid < 32) tmem_dealloc(tbase, 256);
}

static float tf32_trunc(float x) { uint32_t u; memcpy(&u, &x, 4); u &= 0xFFFFE000u; memcpy(&x, &u, 4); return x; }

int main() {
    // (1) correctness
    float *A, *B, *D;
    cudaMallocManaged(&A, M * K * 4); cudaMallocManaged(&B, N * K * 4); cudaMallocManaged(&D, M * N * 4);
    srand(1);
    for (int i = 0; i < M * K; ++i) A[i] = (rand() % 2001 - 1000) / 997.0f;
    for (int i = 0; i < N * K; ++i) B[i] = (rand() % 2001 - 1000) / 991.0f;
    size_t smem = (M + N) * K * 4;
    cudaFuncSetAttribute(gemm_check, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    gemm_check<<<1, 128, smem>>>(A, B, D);
    cudaError_t e = cudaDeviceSynchronize();
    printf("gemm_check: %s\n", cudaGetErrorString(e));
    double maxerr_tr = 0, maxerr_full = 0, maxref = 0;
    for (int m = 0; m < M; ++m)
        for (int n = 0; n < N; ++n) {
            double rt = 0, rf = 0;
            for (int k = 0; k < K; ++k) { rt += (double)tf32_trunc(A[m * K + k]) * tf32_trunc(B[n * K + k]); rf += (double)A[m * K + k] * B[n * K + k]; }
            maxerr_tr = fmax(maxerr_tr, fabs(D[m * N + n] - rt));
            maxerr_full = fmax(maxerr_full, fabs(D[m * N + n] - rf));
            maxref = fmax(maxref, fabs(rf));
        }
    printf("  max|D - ref(tf32 truncated)| = %.3e   max|D - ref(fp32)| = %.3e   max|ref| = %.3f\n", maxerr_tr, maxerr_full, maxref);
    // (2) MMA rate
    float* out; cudaMalloc(&out, 4096);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    auto run_mma = [&](auto kern, int NN) {
        size_t sm = (128 + NN) * 8 * 4;
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        int iters = 20000;
        kern<<<148, 128, sm>>>(iters, out);
        cudaDeviceSynchronize();
        cudaEventRecord(a);
        kern<<<148, 128, sm>>>(iters, out);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        double fl = 2.0 * 128 * NN * 8 * (double)iters * 148;
        printf("mma tf32 M=128 N=%d K=8: %.3f ms, %.1f TFLOP/s (%s)\n", NN, ms, fl / ms / 1e9, cudaGetErrorString(cudaGetLastError()));
    };
    run_mma(mma_rate<64>, 64);
    run_mma(mma_rate<128>, 128);
    run_mma(mma_rate<256>, 256);
    // (3) TMEM load rate
    for (int ctas : {148, 296}) {
        int iters = 20000;
        ld_rate<<<ctas, 128>>>(iters, out);
        cudaDeviceSynchronize();
        cudaEventRecord(a);
        ld_rate<<<ctas, 128>>>(iters, out);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        double bytes = 4.0 * 32 * 32 * 4 * (double)iters * ctas;
        printf("tcgen05.ld 32x32b.x32, %d CTAs x 4 warps: %.3f ms, %.1f TB/s total, %.1f B/clk/SM @1.965GHz (%s)\n",
               ctas, ms, bytes / ms / 1e9, bytes / (ms * 1e-3) / 148 / 1.965e9, cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
