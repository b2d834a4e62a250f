// K4p: binning with a bucket pre-filter (the north_star's "hash bucketing").
//
// cull_tile culls a Gaussian when ANY projection separates it from the tile, so a
// Gaussian can only survive a tile whose interval on r0 and r1 lies within thr of its m_r0, m_r1. The
// live Gaussians are bucketed on a 64 x 64 grid over (m_r0, m_r1) (counting sort, per-cell ranges in a
// permutation array, their (m_r, thr) gathered into cell order so the test reads them coalesced); a
// tile then visits only the cells whose (m_r0, m_r1) range can reach its [lo - thr_max, hi + thr_max]
// rectangle (one cell of slack each side against rounding at cell edges) and runs the SAME exact FP64
// test as K4a on them (all k vectors, strict >, equality kept). Every skipped Gaussian would have been
// culled by r0 or r1 alone, so the mask -- and the CSR K4c compacts from it -- is bit-identical to the
// dense kernel's. The pre-filter pays where tiles are tight and Gaussians narrow (G-buffer-like
// inference regime); with broad Gaussians or loose tiles nearly every cell is in
// range. So the plan kernel counts, with a summed-area table of the cell populations, how many tests the
// pre-filtered pass would run, and ON THE DEVICE selects it only below kPfFraction of the dense pass's
// T * Gev tests; the other path's kernels exit at once. No host round trip, same result either way.
#include "ndg_common.cuh"

using namespace ndg;

namespace {

constexpr int kNB = 64;                  // cells per axis
constexpr int kCells = kNB * kNB;
constexpr double kPfFraction = 0.35;     // pre-filtered tests / dense tests below which K4p runs

__device__ __forceinline__ unsigned long long ord(double x) {       // order-preserving double -> u64
    const unsigned long long u = (unsigned long long)__double_as_longlong(x);
    return (u & 0x8000000000000000ULL) ? ~u : (u | 0x8000000000000000ULL);
}
__device__ __forceinline__ double unord(unsigned long long k) {
    const unsigned long long u = (k & 0x8000000000000000ULL) ? (k & ~0x8000000000000000ULL) : ~k;
    return __longlong_as_double((long long)u);
}

// workspace layout (bytes): see ndg_cull_prefilter_workspace
struct Pf {
    unsigned long long* stats;   // [8]: min0, max0, min1, max1, tmax0, tmax1, (est, flag)
    int* hist;                   // [kCells]
    int* start;                  // [kCells + 1]
    int* cursor;                 // [kCells]
    int32_t* perm;               // [Gev]
    double* ms;                  // [k][Gev] m_r in cell order
    double* ts;                  // [k][Gev] thr in cell order
};

__host__ __device__ inline Pf pf_view(void* ws, int64_t Gev, int k) {
    char* p = reinterpret_cast<char*>(ws);
    Pf v;
    v.stats = reinterpret_cast<unsigned long long*>(p);
    p += 8 * sizeof(unsigned long long);
    v.hist = reinterpret_cast<int*>(p);
    p += kCells * sizeof(int);
    v.start = reinterpret_cast<int*>(p);
    p += (kCells + 4) * sizeof(int);
    v.cursor = reinterpret_cast<int*>(p);
    p += kCells * sizeof(int);
    v.perm = reinterpret_cast<int32_t*>(p);
    p += ((Gev * 4 + 15) / 16) * 16;
    v.ms = reinterpret_cast<double*>(p);
    p += (size_t)k * Gev * 8;
    v.ts = reinterpret_cast<double*>(p);
    return v;
}

__device__ __forceinline__ void cell_geom(const unsigned long long* st, double& mn0, double& d0, double& mn1,
                                          double& d1) {
    mn0 = unord(st[0]);
    mn1 = unord(st[2]);
    const double w0 = unord(st[1]) - mn0, w1 = unord(st[3]) - mn1;
    d0 = w0 > 0.0 ? w0 / kNB : 1.0;
    d1 = w1 > 0.0 ? w1 / kNB : 1.0;
}

__device__ __forceinline__ int cell_of(double m, double mn, double d) {
    const double c = floor((m - mn) / d);
    return c < 0.0 ? 0 : (c >= kNB ? kNB - 1 : (int)c);
}

// cell range a tile interval [lo, hi] widened by tmax can reach, one cell of slack each side
__device__ __forceinline__ void cell_range(double lo, double hi, double tmax, double mn, double d, int& a, int& b) {
    const double fa = floor((lo - tmax - mn) / d) - 1.0, fb = floor((hi + tmax - mn) / d) + 1.0;
    a = fa < 0.0 ? 0 : (fa >= kNB ? kNB : (int)fa);
    b = fb < 0.0 ? -1 : (fb >= kNB ? kNB - 1 : (int)fb);
}

__global__ void pf_init_kernel(unsigned long long* __restrict__ st, int* __restrict__ hist, int* __restrict__ cursor) {
    for (int i = threadIdx.x; i < kCells; i += blockDim.x) hist[i] = cursor[i] = 0;
    if (threadIdx.x < 8) st[threadIdx.x] = (threadIdx.x == 0 || threadIdx.x == 2) ? ~0ull : 0ull;
}

__global__ void pf_stats_kernel(int64_t Gev, const double* __restrict__ m_r, const double* __restrict__ thr,
                                unsigned long long* __restrict__ st) {
    unsigned long long v[6] = {~0ull, 0ull, ~0ull, 0ull, 0ull, 0ull};
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < Gev; e += (int64_t)gridDim.x * blockDim.x) {
        const double t0 = thr[e], t1 = thr[Gev + e];
        if (t0 < 0.0) continue;                              // never evaluated: always culled
        const unsigned long long a = ord(m_r[e]), b = ord(m_r[Gev + e]);
        v[0] = min(v[0], a);
        v[1] = max(v[1], a);
        v[2] = min(v[2], b);
        v[3] = max(v[3], b);
        v[4] = max(v[4], ord(t0));
        v[5] = max(v[5], ord(t1));
    }
#pragma unroll
    for (int o = 16; o; o >>= 1)
#pragma unroll
        for (int j = 0; j < 6; ++j) {
            const unsigned long long w = __shfl_xor_sync(0xffffffffu, v[j], o);
            v[j] = (j == 0 || j == 2) ? min(v[j], w) : max(v[j], w);
        }
    if ((threadIdx.x & 31) == 0) {
        atomicMin(st + 0, v[0]);
        atomicMax(st + 1, v[1]);
        atomicMin(st + 2, v[2]);
        atomicMax(st + 3, v[3]);
        atomicMax(st + 4, v[4]);
        atomicMax(st + 5, v[5]);
    }
}

__global__ void pf_hist_kernel(int64_t Gev, const double* __restrict__ m_r, const double* __restrict__ thr,
                               const unsigned long long* __restrict__ st, int* __restrict__ hist) {
    __shared__ int sh[kCells];
    for (int i = threadIdx.x; i < kCells; i += blockDim.x) sh[i] = 0;
    __syncthreads();
    double mn0, d0, mn1, d1;
    cell_geom(st, mn0, d0, mn1, d1);
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < Gev; e += (int64_t)gridDim.x * blockDim.x) {
        if (thr[e] < 0.0) continue;
        atomicAdd(&sh[cell_of(m_r[e], mn0, d0) * kNB + cell_of(m_r[Gev + e], mn1, d1)], 1);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < kCells; i += blockDim.x)
        if (sh[i]) atomicAdd(hist + i, sh[i]);
}

// one CTA of 1024: exclusive scan of the cell populations, summed-area table, the pre-filtered pass's
// test count over all tiles -> stats[6] (count), stats[7] (1 = run K4p, 0 = run the dense K4a)
__global__ void __launch_bounds__(1024) pf_plan_kernel(int64_t T, int k, const double* __restrict__ lo,
                                                       const double* __restrict__ hi, const int* __restrict__ hist,
                                                       int* __restrict__ start, unsigned long long* __restrict__ st,
                                                       int mode) {
    __shared__ int s_sat[(kNB + 1) * (kNB + 1)];
    __shared__ int s_part[1024];
    __shared__ unsigned long long s_sum[32];
    const int tid = threadIdx.x;
    // exclusive scan of hist (4 cells per thread)
    int v[4], a = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        v[j] = hist[tid * 4 + j];
        a += v[j];
    }
    s_part[tid] = a;
    __syncthreads();
    for (int o = 1; o < 1024; o <<= 1) {
        const int x = tid >= o ? s_part[tid - o] : 0;
        __syncthreads();
        s_part[tid] += x;
        __syncthreads();
    }
    int base = s_part[tid] - a;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        start[tid * 4 + j] = base;
        base += v[j];
    }
    if (tid == 1023) start[kCells] = s_part[1023];
    // summed-area table: s_sat[(r+1)(kNB+1) + (c+1)] = population of cells [0..r] x [0..c]
    for (int i = tid; i < (kNB + 1) * (kNB + 1); i += 1024) s_sat[i] = 0;
    __syncthreads();
    if (tid < kNB) {                                          // row prefix sums
        int acc = 0;
        for (int c = 0; c < kNB; ++c) {
            acc += hist[tid * kNB + c];
            s_sat[(tid + 1) * (kNB + 1) + c + 1] = acc;
        }
    }
    __syncthreads();
    if (tid < kNB) {                                          // column prefix sums
        for (int r = 1; r < kNB; ++r) s_sat[(r + 1) * (kNB + 1) + tid + 1] += s_sat[r * (kNB + 1) + tid + 1];
    }
    __syncthreads();
    const int live = s_part[1023];
    double mn0, d0, mn1, d1;
    cell_geom(st, mn0, d0, mn1, d1);
    const double tm0 = unord(st[4]), tm1 = unord(st[5]);
    unsigned long long tests = 0;
    for (int64_t t = tid; live > 0 && t < T; t += 1024) {
        int a0, b0, a1, b1;
        cell_range(lo[t * k], hi[t * k], tm0, mn0, d0, a0, b0);
        cell_range(lo[t * k + 1], hi[t * k + 1], tm1, mn1, d1, a1, b1);
        if (b0 < a0 || b1 < a1) continue;
        const int W1 = kNB + 1;
        tests += (unsigned long long)(s_sat[(b0 + 1) * W1 + b1 + 1] - s_sat[a0 * W1 + b1 + 1] - s_sat[(b0 + 1) * W1 + a1] +
                                      s_sat[a0 * W1 + a1]);
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) tests += __shfl_xor_sync(0xffffffffu, tests, o);
    if ((tid & 31) == 0) s_sum[tid >> 5] = tests;
    __syncthreads();
    if (tid == 0) {
        unsigned long long tot = 0;
        for (int w = 0; w < 32; ++w) tot += s_sum[w];
        st[6] = tot;
        const bool cheaper = live > 0 && (double)tot < kPfFraction * (double)live * (double)T;
        st[7] = live > 0 && (mode == 1 || (mode == 0 && cheaper)) ? 1ull : 0ull;
    }
}

__global__ void pf_scatter_kernel(int64_t Gev, int k, const double* __restrict__ m_r, const double* __restrict__ thr,
                                  const unsigned long long* __restrict__ st, const int* __restrict__ start,
                                  int* __restrict__ cursor, int32_t* __restrict__ perm, double* __restrict__ ms,
                                  double* __restrict__ ts) {
    if (st[7] == 0) return;
    double mn0, d0, mn1, d1;
    cell_geom(st, mn0, d0, mn1, d1);
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < Gev; e += (int64_t)gridDim.x * blockDim.x) {
        if (thr[e] < 0.0) continue;
        const int cell = cell_of(m_r[e], mn0, d0) * kNB + cell_of(m_r[Gev + e], mn1, d1);
        const int pos = start[cell] + atomicAdd(cursor + cell, 1);     // order inside a cell is irrelevant:
        NDG_DCHECK(cell >= 0 && cell < kCells && pos >= start[cell] && pos < start[cell + 1]);
        perm[pos] = (int32_t)e;                                        // the mask is order-free
        for (int ri = 0; ri < k; ++ri) {
            ms[ri * Gev + pos] = m_r[ri * Gev + e];
            ts[ri * Gev + pos] = thr[ri * Gev + e];
        }
    }
}

__global__ void pf_zero_kernel(int64_t words, const unsigned long long* __restrict__ st, uint32_t* __restrict__ mask) {
    if (st[7] == 0) return;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < words; i += (int64_t)gridDim.x * blockDim.x)
        mask[i] = 0u;
}

// CTA per tile: the exact K4a test (FP64, strict >, early exit) over the Gaussians of the reachable cells
__global__ void __launch_bounds__(256) pf_cull_kernel(int64_t T, int k, int64_t Gev, const double* __restrict__ lo,
                                                      const double* __restrict__ hi,
                                                      const unsigned long long* __restrict__ st,
                                                      const int* __restrict__ start, const int32_t* __restrict__ perm,
                                                      const double* __restrict__ ms, const double* __restrict__ ts,
                                                      uint32_t* __restrict__ mask, int64_t* __restrict__ counts) {
    if (st[7] == 0) return;
    extern __shared__ double s_b[];                    // [2][k] tile interval
    __shared__ int s_cnt[8];
    const int64_t t = blockIdx.x;
    for (int ri = threadIdx.x; ri < k; ri += blockDim.x) {
        s_b[ri] = lo[t * k + ri];
        s_b[k + ri] = hi[t * k + ri];
    }
    __syncthreads();
    double mn0, d0, mn1, d1;
    cell_geom(st, mn0, d0, mn1, d1);
    int a0, b0, a1, b1;
    cell_range(s_b[0], s_b[k], unord(st[4]), mn0, d0, a0, b0);
    cell_range(s_b[1], s_b[k + 1], unord(st[5]), mn1, d1, a1, b1);
    const int64_t W = (Gev + 31) / 32;
    int cnt = 0;
    if (b1 >= a1) {
        for (int r = a0; r <= b0; ++r) {
            const int j1 = start[r * kNB + b1 + 1];
            for (int j = start[r * kNB + a1] + threadIdx.x; j < j1; j += blockDim.x) {
                bool kept = true;
                for (int ri = 0; ri < k; ++ri) {
                    const double m = ms[ri * Gev + j], th = ts[ri * Gev + j];
                    if (__dsub_rn(s_b[ri], m) > th || __dsub_rn(m, s_b[k + ri]) > th) {
                        kept = false;
                        break;
                    }
                }
                if (kept) {
                    const int e = perm[j];
                    NDG_DCHECK(e >= 0 && e < Gev && j < start[kCells]);
                    atomicOr(mask + t * W + (e >> 5), 1u << (e & 31));
                    ++cnt;
                }
            }
        }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
    if ((threadIdx.x & 31) == 0) s_cnt[threadIdx.x >> 5] = cnt;
    __syncthreads();
    if (threadIdx.x == 0) {
        int c = 0;
        for (int w = 0; w < 8; ++w) c += s_cnt[w];
        counts[t] = c;
    }
}

}  // namespace

extern "C" int64_t ndg_cull_prefilter_workspace(int64_t Gev, int k) {
    return (int64_t)(8 * 8 + kCells * 4 + (kCells + 4) * 4 + kCells * 4 + ((Gev * 4 + 15) / 16) * 16 +
                     2 * (size_t)k * Gev * 8);
}

// Launches the plan and both paths; each path's kernels exit at once unless the plan selected it (the
// dense path is K4a with a skip word = stats[7]). The workspace needs no initialisation.
int cull_mask_launch(int64_t T, int k, int64_t Gev, const double* lo, const double* hi, const double* m_r,
                     const double* thr, uint32_t* mask, int64_t* counts, const unsigned long long* skip,
                     cudaStream_t stream);

extern "C" int ndg_cull_prefilter(int64_t T, int k, int64_t Gev, const double* lo, const double* hi, const double* m_r,
                                  const double* thr, int mode, void* workspace, uint32_t* mask, int64_t* counts,
                                  void* stream) {
    NDG_REQUIRE(mode >= 0 && mode <= 2, "mode: 0 = auto, 1 = pre-filter, 2 = dense");
    NDG_REQUIRE(k >= 2 && k <= 256, "the pre-filter buckets on two projection vectors (2 <= k <= 256)");
    NDG_REQUIRE(Gev < (1LL << 31), "the pre-filter permutation is int32");
    if (T == 0 || Gev == 0) return NDG_OK;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    Pf v = pf_view(workspace, Gev, k);
    const unsigned gg = (unsigned)imin64((Gev + 255) / 256, 148 * 8);
    pf_init_kernel<<<1, 1024, 0, st>>>(v.stats, v.hist, v.cursor);
    pf_stats_kernel<<<gg, 256, 0, st>>>(Gev, m_r, thr, v.stats);
    pf_hist_kernel<<<gg, 256, 0, st>>>(Gev, m_r, thr, v.stats, v.hist);
    pf_plan_kernel<<<1, 1024, 0, st>>>(T, k, lo, hi, v.hist, v.start, v.stats, mode);
    pf_scatter_kernel<<<gg, 256, 0, st>>>(Gev, k, m_r, thr, v.stats, v.start, v.cursor, v.perm, v.ms, v.ts);
    const int64_t words = T * ((Gev + 31) / 32);
    pf_zero_kernel<<<(unsigned)imin64((words + 255) / 256, 148 * 16), 256, 0, st>>>(words, v.stats, mask);
    pf_cull_kernel<<<(unsigned)T, 256, 2 * k * sizeof(double), st>>>(T, k, Gev, lo, hi, v.stats, v.start, v.perm, v.ms,
                                                                      v.ts, mask, counts);
    NDG_CHECK_LAUNCH();
    return cull_mask_launch(T, k, Gev, lo, hi, m_r, thr, mask, counts, v.stats + 7, st);
}
