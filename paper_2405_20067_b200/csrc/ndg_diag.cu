// Diagnostics off the training hot path (float64): brute_force_active as a
// per-(tile, Gaussian) bit-mask, the reference set the culling ablation (cmd_bench_cull,
// SPEC.md:531-539) counts false culls against.
//
// Grid (tiles x ceil(Gev / 128)); thread = evaluated Gaussian with its float64 factor in registers;
// the tile's queries are staged in shared memory (float32, widened per use). A Gaussian is active in
// a tile iff some query has |z|^2 <= max_s2 with L z = x - m solved by forward substitution in
// float64 (eval_gaussian >= epsilon  <=>  |z|^2 <= -2 ln epsilon). The early exit at the first hit
// keeps the brute force cheap for the kept Gaussians; the culled ones cost a full tile sweep.
#include "ndg_common.cuh"

using namespace ndg;

namespace {

constexpr int kDiagThreads = 128;

template <int N>
__global__ void __launch_bounds__(kDiagThreads)
    active_mask_kernel(int tile, const float* __restrict__ queries, const double* __restrict__ mean64,
                       const double* __restrict__ chol64, const uint8_t* __restrict__ eflags, int64_t Gev,
                       double max_s2, uint32_t* __restrict__ mask, int64_t W, int64_t* __restrict__ counts) {
    constexpr int P = n_chol(N);
    extern __shared__ float s_x[];                       // [tile][N]
    const int64_t t = blockIdx.x;
    const int64_t e = (int64_t)blockIdx.y * kDiagThreads + threadIdx.x;
    for (int i = threadIdx.x; i < tile * N; i += kDiagThreads) s_x[i] = queries[t * tile * N + i];
    __syncthreads();
    bool hit = false;
    if (e < Gev && (eflags[e] & 3) == 1) {               // live and not degenerate
        double L[P], m[N], inv[N];
#pragma unroll
        for (int k = 0; k < P; ++k) L[k] = chol64[e * P + k];
#pragma unroll
        for (int i = 0; i < N; ++i) {
            m[i] = mean64[e * N + i];
            inv[i] = 1.0 / L[tri(i, i)];
        }
        for (int q = 0; q < tile && !hit; ++q) {
            double z[N], s = 0.0;
#pragma unroll
            for (int i = 0; i < N; ++i) {
                double a = (double)s_x[q * N + i] - m[i];
#pragma unroll
                for (int k = 0; k < i; ++k) a -= L[tri(i, k)] * z[k];
                z[i] = a * inv[i];
                s += z[i] * z[i];
            }
            hit = s <= max_s2;
        }
    }
    const uint32_t bits = __ballot_sync(0xffffffffu, hit);
    const int64_t word = e >> 5;
    if ((threadIdx.x & 31) == 0 && word < W) {
        mask[t * W + word] = bits;
        if (bits) atomicAdd(reinterpret_cast<unsigned long long*>(counts + t), (unsigned long long)__popc(bits));
    }
}

template <int N>
int launch_active(int64_t T, int tile, const float* q, const double* mean64, const double* chol64,
                  const uint8_t* eflags, int64_t Gev, double max_s2, uint32_t* mask, int64_t* counts,
                  cudaStream_t st) {
    const int64_t W = (Gev + 31) / 32;
    const int64_t gb = (Gev + kDiagThreads - 1) / kDiagThreads;
    NDG_REQUIRE(T <= 0x7fffffffLL && gb <= 65535, "too many tiles / Gaussians for the brute-force grid");
    const size_t smem = sizeof(float) * (size_t)tile * N;
    NDG_REQUIRE(smem <= 48 * 1024, "tile too large for the brute-force query staging");
    active_mask_kernel<N><<<dim3((unsigned)T, (unsigned)gb), kDiagThreads, smem, st>>>(tile, q, mean64, chol64, eflags,
                                                                                      Gev, max_s2, mask, W, counts);
    NDG_CHECK_LAUNCH();
    return NDG_OK;
}

}  // namespace

extern "C" int ndg_active_mask(int n, int64_t B, int tile, const float* queries, const double* mean64,
                               const double* chol64, const uint8_t* eflags, int64_t Gev, double max_s2,
                               uint32_t* mask, int64_t* counts, void* stream) {
    NDG_REQUIRE(tile >= 1 && B % tile == 0, "batch must be a multiple of tile");
    if (B == 0 || Gev == 0) return NDG_OK;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    const int64_t T = B / tile;
    switch (n) {
#define NDG_CASE(NN) \
    case NN:         \
        return launch_active<NN>(T, tile, queries, mean64, chol64, eflags, Gev, max_s2, mask, counts, st);
        NDG_CASE(1) NDG_CASE(2) NDG_CASE(3) NDG_CASE(4) NDG_CASE(5) NDG_CASE(6) NDG_CASE(7) NDG_CASE(8)
        NDG_CASE(9) NDG_CASE(10) NDG_CASE(11) NDG_CASE(12) NDG_CASE(13) NDG_CASE(14) NDG_CASE(15) NDG_CASE(16)
#undef NDG_CASE
        default:
            return NDG_ERR_UNSUPPORTED_DIMS;
    }
}
