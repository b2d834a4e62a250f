// Device-side batch sampling and the shading-toy target.
//
// sample_batch draws B fresh uniform queries in [0,1)^N and sorts them by the first (position)
// dimension into contiguous tiles. The sorted first coordinates of B iid uniforms are
// the uniform order statistics, and those are exactly S_k / S_{B+1} with S_k = E_0 + ... + E_{k-1}
// the partial sums of B + 1 iid exponentials (the Renyi representation) -- so the sort becomes one
// prefix sum: no sort, no key-value shuffle. The spacings are summed in 32.32 fixed point (int64), so
// the prefix is exact whatever the summation order and the first coordinates are non-decreasing by
// construction (a float64 parallel scan could round a block boundary backwards); the quantum 2^-32
// of a mean-1 spacing is far below float32's resolution of the result. The other N - 1 coordinates are iid and need no
// ordering. Randomness is a counter-based Philox4x32-10 stream keyed by (seed, draw), so a batch is a
// pure function of (seed, draw index): checkpoints store two integers, every rank of a data-parallel
// fit draws the same global batch and writes only the rows of its own tiles.
//
//   ndg_sample_spacings  thread per exponential: E_i = -log(u) in fixed point, block sums
//   ndg_sample_scan      one CTA: exclusive prefix of the block sums and the total S_{B+1}
//   ndg_sample_write     block scan of its E_i -> x_0, Philox uniforms for dims 1..N-1, strided tiles
//   ndg_shading_target   thread per query: the shading-toy function (datasets.ShadingToyTarget)
#include "ndg_common.cuh"

using namespace ndg;

namespace {

constexpr int kSampleThreads = 1024;
constexpr int64_t kMaxSampleBatch = int64_t(1) << 24;    // (B + 1) * max E * 2^32 < 2^63

struct U4 {
    uint32_t x, y, z, w;
};

// Philox4x32-10 (Salmon et al., SC'11): counter (c0..c3), key (k0, k1)
__device__ __forceinline__ U4 philox(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3, uint32_t k0, uint32_t k1) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const uint32_t lo0 = 0xD2511F53u * c0, hi0 = __umulhi(0xD2511F53u, c0);
        const uint32_t lo1 = 0xCD9E8D57u * c2, hi1 = __umulhi(0xCD9E8D57u, c2);
        const uint32_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
        c0 = n0;
        c1 = lo1;
        c2 = n2;
        c3 = lo0;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    return U4{c0, c1, c2, c3};
}

// streams of the counter's third word: which random quantity a word feeds
constexpr uint32_t kStreamSpacing = 0, kStreamDims = 1;

__device__ __forceinline__ long long exp_variate(uint64_t seed, uint64_t draw, int64_t i) {
    const U4 r = philox((uint32_t)i, (uint32_t)((uint64_t)i >> 32), kStreamSpacing, (uint32_t)draw, (uint32_t)seed,
                        (uint32_t)(seed >> 32) ^ (uint32_t)(draw >> 32));
    // 53-bit uniform in (0, 1]
    const double u = ((double)(r.x >> 5) * 67108864.0 + (double)(r.y >> 6) + 1.0) * (1.0 / 9007199254740992.0);
    return __double2ll_rn(-log(u) * 4294967296.0);      // <= 36.8 * 2^32 < 2^38
}

__device__ __forceinline__ long long block_sum(long long v, long long* s) {
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = v;
    __syncthreads();
    long long t = 0;
    if (threadIdx.x < 32) {
        t = threadIdx.x < (blockDim.x >> 5) ? s[threadIdx.x] : 0;
        for (int o = 16; o; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    }
    return t;                                           // valid in thread 0 (and all of warp 0)
}

__global__ void __launch_bounds__(kSampleThreads) spacings_kernel(int64_t n_exp, uint64_t seed, uint64_t draw,
                                                                  long long* __restrict__ block_sums) {
    __shared__ long long s[32];
    const int64_t i = blockIdx.x * (int64_t)kSampleThreads + threadIdx.x;
    const long long e = i < n_exp ? exp_variate(seed, draw, i) : 0;
    const long long t = block_sum(e, s);
    if (threadIdx.x == 0) block_sums[blockIdx.x] = t;
}

// exclusive prefix of the block sums (block_sums[nb] = total), one CTA
__global__ void __launch_bounds__(kSampleThreads) scan_kernel(int64_t nb, long long* __restrict__ block_sums) {
    __shared__ long long s[kSampleThreads];
    __shared__ long long carry;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (int64_t base = 0; base < nb; base += kSampleThreads) {
        const int64_t i = base + threadIdx.x;
        const long long v = i < nb ? block_sums[i] : 0;
        s[threadIdx.x] = v;
        __syncthreads();
        for (int o = 1; o < kSampleThreads; o <<= 1) {
            const long long x = threadIdx.x >= o ? s[threadIdx.x - o] : 0;
            __syncthreads();
            s[threadIdx.x] += x;
            __syncthreads();
        }
        if (i < nb) block_sums[i] = carry + s[threadIdx.x] - v;
        __syncthreads();
        if (threadIdx.x == kSampleThreads - 1) carry += s[kSampleThreads - 1];
        __syncthreads();
    }
    if (threadIdx.x == 0) block_sums[nb] = carry;
}

// row k of the sorted batch: x_0 = (E_0 + ... + E_k) / S_{B+1}; rows of tiles owned by this rank only
__global__ void __launch_bounds__(kSampleThreads) write_kernel(int n, int64_t B, int tile, int rank, int world,
                                                               uint64_t seed, uint64_t draw,
                                                               const long long* __restrict__ block_sums,
                                                               float* __restrict__ queries) {
    __shared__ long long s[kSampleThreads];
    const int64_t k = blockIdx.x * (int64_t)kSampleThreads + threadIdx.x;
    const long long e = k < B ? exp_variate(seed, draw, k) : 0;
    s[threadIdx.x] = e;
    __syncthreads();
    for (int o = 1; o < kSampleThreads; o <<= 1) {       // inclusive block scan
        const long long x = threadIdx.x >= o ? s[threadIdx.x - o] : 0;
        __syncthreads();
        s[threadIdx.x] += x;
        __syncthreads();
    }
    if (k >= B) return;
    const int64_t t = k / tile;
    if (t % world != rank) return;
    const int64_t row = (t / world) * tile + (k - t * tile);        // local row among the rank's tiles
    const double total = (double)block_sums[(B + kSampleThreads) / kSampleThreads];   // S_{B+1}
    float x0 = (float)((double)(block_sums[blockIdx.x] + s[threadIdx.x]) / total);     // monotone in k
    x0 = fminf(x0, 0.99999994f);                       // [0, 1) after float32 rounding
    float* q = queries + row * n;
    q[0] = x0;
    for (int d = 1; d < n; d += 4) {
        const U4 r = philox((uint32_t)k, (uint32_t)((uint64_t)k >> 32), kStreamDims + 2u * (uint32_t)(d / 4),
                            (uint32_t)draw, (uint32_t)seed, (uint32_t)(seed >> 32) ^ (uint32_t)(draw >> 32));
        const uint32_t w[4] = {r.x, r.y, r.z, r.w};
#pragma unroll
        for (int j = 0; j < 4; ++j)
            if (d + j < n) q[d + j] = (float)(w[j] >> 8) * (1.0f / 16777216.0f);       // 24-bit uniform in [0,1)
    }
}

// shading_toy_target, the same function as datasets.ShadingToyTarget: position (3),
// view direction (3, mapped from [0,1] to [-1,1]), albedo (3), roughness (1); p = [freq[3], phase[3]]
__global__ void shading_kernel(int n, int64_t B, const float* __restrict__ queries, const float* __restrict__ p,
                               float* __restrict__ out) {
    const int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (b >= B) return;
    const float* q = queries + b * n;
    const float tau = 6.283185307179586f;
    const float px = q[0], py = q[1], pz = q[2];
    const float shade = 0.55f + 0.45f * (sinf(tau * p[0] * px + p[3]) * sinf(tau * p[1] * py + p[4]) *
                                         sinf(tau * p[2] * pz + p[5]));
    float alb[3] = {0.6f, 0.6f, 0.6f};
    if (n >= 9)
        for (int c = 0; c < 3; ++c) alb[c] = q[6 + c];
    const float rough = n >= 10 ? q[9] : 0.5f;
    float v[3];
    for (int c = 0; c < 3; ++c) v[c] = 3 + c < n ? 2.f * q[3 + c] - 1.f : 1.f;
    const float vn = fmaxf(sqrtf(v[0] * v[0] + v[1] * v[1] + v[2] * v[2]), 1e-6f);
    float rf[3] = {sinf(tau * px), cosf(tau * py), 0.5f + pz};
    const float rn = sqrtf(rf[0] * rf[0] + rf[1] * rf[1] + rf[2] * rf[2]);
    const float dot = fmaxf((v[0] * rf[0] + v[1] * rf[1] + v[2] * rf[2]) / (vn * rn), 0.f);
    const float lobe = powf(dot, 2.f + 40.f * (1.f - rough));
    for (int c = 0; c < 3; ++c) out[b * 3 + c] = alb[c] * shade * 0.6f + 0.4f * lobe;
}

}  // namespace

extern "C" int64_t ndg_sample_workspace(int64_t B) {
    return (int64_t)sizeof(long long) * ((B + kSampleThreads) / kSampleThreads + 2);
}

extern "C" int ndg_sample_batch(int n, int64_t B, int tile, int rank, int world, uint64_t seed, uint64_t draw,
                                int64_t* workspace, float* queries, void* stream) {
    if (!ndg_supported_dims(n)) return NDG_ERR_UNSUPPORTED_DIMS;
    NDG_REQUIRE(tile >= 1 && B % tile == 0 && world >= 1 && rank >= 0 && rank < world,
                "batch must be a multiple of the tile; 0 <= rank < world");
    NDG_REQUIRE(B <= kMaxSampleBatch, "one sampled batch holds at most 2^24 queries");
    if (B == 0) return NDG_OK;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    const int64_t n_exp = B + 1;                          // B + 1 spacings: S_{B+1} normalises
    const int64_t nb = (n_exp + kSampleThreads - 1) / kSampleThreads;
    long long* ws = reinterpret_cast<long long*>(workspace);
    spacings_kernel<<<(unsigned)nb, kSampleThreads, 0, st>>>(n_exp, seed, draw, ws);
    scan_kernel<<<1, kSampleThreads, 0, st>>>(nb, ws);
    write_kernel<<<(unsigned)((B + kSampleThreads - 1) / kSampleThreads), kSampleThreads, 0, st>>>(
        n, B, tile, rank, world, seed, draw, ws, queries);
    NDG_CHECK_LAUNCH();
    return NDG_OK;
}

extern "C" int ndg_shading_target(int n, int64_t B, const float* queries, const float* params, float* out,
                                  void* stream) {
    NDG_REQUIRE(n >= 4 && n <= 10, "the shading toy needs 4 <= N <= 10");
    if (B == 0) return NDG_OK;
    shading_kernel<<<(unsigned)((B + 255) / 256), 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(n, B, queries,
                                                                                                     params, out);
    NDG_CHECK_LAUNCH();
    return NDG_OK;
}
