// FP32-pipe peak probe: the roofline denominator for the FP32-SIMT pair kernels (K5 / K7).
// MEASURED_PEAKS.json carries only HBM copy bandwidth and cuBLAS bf16; bench.py measures the
// sustained FFMA rate with this kernel on the same box, at the clocks of the timed run.
// 8 independent packed FFMA2 chains per thread (16 FMAs per step; FFMA2 reaches the FMA pipe's
// limit with half the issue slots of scalar FFMA: 74.2 vs 72.5 TFLOP/s measured on B200), so the
// denominator is the pipe's true peak; flops = 2 * 16 * 16 * iters per thread.
#include "ndg_tc.cuh"

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

// TF32 tensor-core peak probe (tcgen05.mma kind::tf32, M=128, N=256, K=8, operands resident in smem):
// the roofline denominator for the tensor-core forward. One CTA per SM, one elected lane issues
// `iters` MMAs; flops = 2 * 128 * 256 * 8 * iters per CTA.
#include "ndg_tc.cuh"

__global__ void __launch_bounds__(128) tf32_probe_kernel(int iters, float* out) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ __align__(8) uint64_t bar;
    __shared__ uint32_t tbase;
    const int tid = threadIdx.x;
    for (int i = tid; i < (128 + 256) * 8; i += blockDim.x) reinterpret_cast<float*>(sm)[i] = 1e-3f * (i % 7);
    if (tid < 32) ndg::tc::alloc(&tbase, 256);
    if (tid == 0) {
        ndg::mbar_init(&bar, 1);
        ndg::fence_mbar_init();
    }
    ndg::fence_proxy_async();
    ndg::tc::fence_before();
    __syncthreads();
    ndg::tc::fence_after();
    if (tid == 0) {
        const uint32_t base = ndg::smem_u32(sm);
        const uint64_t a = ndg::tc::smem_desc(base, 128 * 16);
        const uint64_t b = ndg::tc::smem_desc(base + 128 * 8 * 4, 256 * 16);
        for (int i = 0; i < iters; ++i) ndg::tc::mma_tf32(tbase, a, b, ndg::tc::idesc_tf32(128, 256), i > 0);
        ndg::tc::commit(&bar);
    }
    ndg::mbar_wait(&bar, 0);
    ndg::tc::fence_after();
    float v[16];
    ndg::tc::ld16(tbase + ((uint32_t)((tid / 32) * 32) << 16), v);
    ndg::tc::wait_ld();
    if (v[0] == 12345.f) out[tid] = v[1];
    ndg::tc::fence_before();
    __syncthreads();
    if (tid < 32) ndg::tc::dealloc(tbase, 256);
}

extern "C" int ndg_tf32_probe(float* out, int blocks, int iters, void* stream) {
    NDG_REQUIRE(blocks >= 1 && iters >= 1, "blocks and iters must be positive");
    const int smem = (128 + 256) * 8 * 4;
    tf32_probe_kernel<<<blocks, 128, smem, reinterpret_cast<cudaStream_t>(stream)>>>(iters, out);
    NDG_CHECK_LAUNCH();
    return NDG_OK;
}

extern "C" double ndg_tf32_probe_flops(int blocks, int iters) { return 2.0 * 128 * 256 * 8 * (double)iters * blocks; }

// Warp-level tensor-core peak probe (mma.sync m16n8k16 f16 -> f32, the K7-MMA instruction): 512 threads
// per CTA, each warp running 8 independent accumulator chains -- the roofline denominator for K7-MMA.
// (m16n8k8 tf32 issues at the same 0.467 MMA/clk/SM with half the K: tools/mma_sync_probe.cu.)
__global__ void __launch_bounds__(512) hmma_probe_kernel(int iters, float* out) {
    float d[8][4] = {};
    uint32_t a[4], b[2];
    for (int i = 0; i < 4; ++i) a[i] = 0x3c003c00u + threadIdx.x + i;
    for (int i = 0; i < 2; ++i) b[i] = 0x38003800u + i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int k = 0; k < 8; ++k)
            asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
                         "{%8,%9}, {%0,%1,%2,%3};\n"
                         : "+f"(d[k][0]), "+f"(d[k][1]), "+f"(d[k][2]), "+f"(d[k][3])
                         : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
    }
    float s = 0.f;
    for (int k = 0; k < 8; ++k) s += d[k][0] + d[k][1] + d[k][2] + d[k][3];
    if (s == 12345.f) out[threadIdx.x] = s;
}

extern "C" int ndg_hmma_probe(float* out, int blocks, int iters, void* stream) {
    NDG_REQUIRE(blocks >= 1 && iters >= 1, "blocks and iters must be positive");
    hmma_probe_kernel<<<blocks, 512, 0, reinterpret_cast<cudaStream_t>(stream)>>>(iters, out);
    NDG_CHECK_LAUNCH();
    return NDG_OK;
}

extern "C" double ndg_hmma_probe_flops(int blocks, int iters) { return 2.0 * 16 * 8 * 16 * 8 * 16 * (double)iters * blocks; }
