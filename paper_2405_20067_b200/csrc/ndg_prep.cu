// libndg.so: prologue (K1), projected bounds (K2), tile bounds (K3), binning (K4a-c), loss
// finalisation, epilogue (K8) and Adam (K9). The FP32 pair kernels K5 / K7 live in ndg_forward.cu /
// ndg_backward.cu. Reference operations are cited per kernel (SPEC.md = /root/reference/SPEC.md).
//
// Bit-exactness of the culling path: every float64 sum below runs in the oracle's order with
// explicit __dmul_rn / __dadd_rn (no FMA contraction), so m_r, s_r, the tile bounds and therefore
// the candidate lists equal oracle/ndg_oracle.py's bit for bit given the same activated factors.
#include <climits>
#include <cstdio>
#include <cstring>

#include <algorithm>
#include <cstdlib>

#include "ndg_common.cuh"

using namespace ndg;

static thread_local char g_last_error[256] = "";

extern "C" void ndg_set_last_error(const char* msg) {
    std::strncpy(g_last_error, msg, sizeof(g_last_error) - 1);
    g_last_error[sizeof(g_last_error) - 1] = 0;
}

extern "C" const char* ndg_last_error(void) { return g_last_error; }
extern "C" int ndg_abi_version(void) { return NDG_ABI_VERSION; }
extern "C" int ndg_supported_dims(int n) { return n >= 1 && n <= NMAX; }
extern "C" int ndg_raw_floats(int n) { return raw_floats(n); }
extern "C" int ndg_record_floats(int n) { return rec_floats(n); }
extern "C" int ndg_query_floats(int n) { return qrec_floats(n); }
extern "C" int ndg_accum_doubles(int n) { return acc_doubles(n); }
extern "C" int ndg_num_stats(void) { return kNumStats; }
extern "C" int ndg_backward_chunk(void) { return kBwdChunk; }

static inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

__device__ __forceinline__ void record_key(int64_t* slot, int64_t key) {
    atomicMax(reinterpret_cast<unsigned long long*>(slot), (unsigned long long)(LLONG_MAX - key));
}

__device__ __forceinline__ double act_offdiag(double r) {   // 2 * sigmoid(r) - 1
    double s = __ddiv_rn(1.0, __dadd_rn(1.0, exp(-r)));
    return __dsub_rn(__dmul_rn(2.0, s), 1.0);
}

__device__ __forceinline__ double sigmoid64(double r) { return 1.0 / (1.0 + exp(-r)); }

// ---------------------------------------------------------------------------------------------
// K1 prologue: activate_cholesky, compose_child (Eq. 6-7),
// alpha / colour activation. One thread per evaluated Gaussian.
// ---------------------------------------------------------------------------------------------
__global__ void prologue_kernel(int n, int64_t G, int64_t Gev, int amp_mode, const float* __restrict__ params,
                                const float* __restrict__ child, const uint8_t* __restrict__ flags,
                                float* __restrict__ rec, double* __restrict__ mean64, double* __restrict__ chol64,
                                uint8_t* __restrict__ eflags, ndg_status* st) {
    int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (e >= Gev) return;
    const int P = n_chol(n), R = raw_floats(n), RS = rec_floats(n);
    const bool is_child = e >= G;
    const int64_t i = is_child ? e - G : e;
    const uint8_t f = flags ? flags[i] : 0;
    const bool frozen = f & 2, has_child = f & 1;
    const float* prow = params + i * R;
    bool live = !frozen && (!is_child || has_child);

    // non-finite raw parameters -> InvalidParameterError; parent rows always checked,
    // child rows only when the child is live.
    if (!is_child || has_child) {
        const float* row = is_child ? child + i * R : prow;
        for (int t = 0; t < R; ++t)
            if (!isfinite(row[t])) {
                record_key(&st->invalid_key, (is_child ? G * R : 0) + i * R + t);
                break;
            }
    }

    double L[n_chol(NMAX)], m[NMAX];
    for (int r = 0; r < n; ++r)
        for (int c = 0; c <= r; ++c) {
            double raw = (double)prow[n + tri(r, c)];
            L[tri(r, c)] = (r == c) ? exp(raw) : act_offdiag(raw);
        }
    for (int r = 0; r < n; ++r) m[r] = (double)prow[r];
    const float* arow = prow;
    if (is_child) {
        const float* crow = child + i * R;
        double U[n_chol(NMAX)], mc[NMAX], Lc[n_chol(NMAX)];
        for (int r = 0; r < n; ++r)
            for (int c = 0; c <= r; ++c) {
                double raw = (double)crow[n + tri(r, c)];
                U[tri(r, c)] = (r == c) ? exp(raw) : act_offdiag(raw);
            }
        for (int r = 0; r < n; ++r) {   // m_c = L m_u + m_p, ascending k
            double acc = __dmul_rn(L[tri(r, 0)], (double)crow[0]);
            for (int k = 1; k <= r; ++k) acc = __dadd_rn(acc, __dmul_rn(L[tri(r, k)], (double)crow[k]));
            mc[r] = __dadd_rn(acc, m[r]);
        }
        for (int r = 0; r < n; ++r)     // L U, ascending k
            for (int c = 0; c <= r; ++c) {
                double acc = __dmul_rn(L[tri(r, c)], U[tri(c, c)]);
                for (int k = c + 1; k <= r; ++k) acc = __dadd_rn(acc, __dmul_rn(L[tri(r, k)], U[tri(k, c)]));
                Lc[tri(r, c)] = acc;
            }
        for (int t = 0; t < P; ++t) L[t] = Lc[t];
        for (int r = 0; r < n; ++r) m[r] = mc[r];
        arow = crow;
    }
    bool degenerate = false;
    for (int t = 0; t < P; ++t) degenerate |= !isfinite(L[t]);
    for (int r = 0; r < n; ++r) degenerate |= L[tri(r, r)] < 1e-30;
    if (degenerate && live) atomicAdd(reinterpret_cast<unsigned long long*>(&st->n_degenerate), 1ull);
    live = live && !degenerate;

    for (int t = 0; t < P; ++t) chol64[e * P + t] = L[t];
    for (int r = 0; r < n; ++r) mean64[e * n + r] = m[r];
    eflags[e] = (uint8_t)((live ? 1 : 0) | (degenerate ? 2 : 0));

    float* out = rec + e * RS;
    if (!live) {
        for (int t = 0; t < RS; ++t) out[t] = 0.f;
        return;
    }
    double ampr = (double)arow[n + P + 3];
    double alpha = amp_mode == NDG_BRIGHTNESS ? exp(ampr) : sigmoid64(ampr);
    for (int t = 0; t < RS; ++t) out[t] = 0.f;   // also zeroes the row pads of nlu
    for (int r = 0; r < n; ++r) {
        double inv = 1.0 / L[tri(r, r)];
        const float nb = (float)(-kC * m[r] * inv);
        out[rec_nb2(n) + 2 * r] = nb;
        out[rec_nb2(n) + 2 * r + 1] = nb;
        out[rec_rho(n) + r] = (float)(kC * inv);
        for (int c = 0; c < r; ++c) out[rec_l(n, r, c)] = (float)(-L[tri(r, c)] * inv);
    }
    for (int ch = 0; ch < 3; ++ch) out[rec_a(n) + ch] = (float)(alpha * sigmoid64((double)arow[n + P + ch]));
}

extern "C" int ndg_prologue(int n, int64_t G, int64_t Gev, int amp_mode, const float* params, const float* child,
                            const uint8_t* flags, float* rec, double* mean64, double* chol64, uint8_t* eflags,
                            ndg_status* status, void* stream) {
    if (!ndg_supported_dims(n)) return NDG_ERR_UNSUPPORTED_DIMS;
    NDG_REQUIRE(G >= 0 && (Gev == G || Gev == 2 * G), "Gev must be G or 2G");
    NDG_REQUIRE(Gev == G || child != nullptr, "child rows required when Gev == 2G");
    if (Gev == 0) return NDG_OK;
    const int threads = spread_threads(Gev, 128);
    prologue_kernel<<<(unsigned)((Gev + threads - 1) / threads), threads, 0, as_stream(stream)>>>(
        n, G, Gev, amp_mode, params, child, flags, rec, mean64, chol64, eflags, status);
    NDG_CHECK_LAUNCH();
    return NDG_OK;
}

// ---------------------------------------------------------------------------------------------
// K2 projected bounds: project_components (Eq. 3-4). FP64, oracle order.
// ---------------------------------------------------------------------------------------------
__global__ void project_kernel(int n, int64_t Gev, const double* __restrict__ mean64,
                               const double* __restrict__ chol64, const uint8_t* __restrict__ eflags,
                               const double* __restrict__ dirs, int k, double mult, double* __restrict__ m_r,
                               double* __restrict__ s_r, double* __restrict__ thr, int kpb) {
    extern __shared__ double sdir[];
    for (int t = threadIdx.x; t < k * n; t += blockDim.x) sdir[t] = dirs[t];
    __syncthreads();
    int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (e >= Gev) return;
    const int P = n_chol(n);
    double m[NMAX], L[n_chol(NMAX)];
    for (int r = 0; r < n; ++r) m[r] = mean64[e * n + r];
    for (int t = 0; t < P; ++t) L[t] = chol64[e * P + t];
    const uint8_t f = eflags[e];
    const bool live = f & 1, degenerate = f & 2;
    const int r0 = blockIdx.y * kpb, r1 = min(k, r0 + kpb);   // this CTA's projections (blockIdx.y)
    for (int ri = r0; ri < r1; ++ri) {
        const double* r = sdir + ri * n;
        double acc = __dmul_rn(m[0], r[0]);
        for (int j = 1; j < n; ++j) acc = __dadd_rn(acc, __dmul_rn(m[j], r[j]));
        double ss = 0.0;
        for (int j = 0; j < n; ++j) {
            double u = __dmul_rn(L[tri(j, j)], r[j]);           // (L^T r)_j = sum_{i>=j} L_ij r_i
            for (int i = j + 1; i < n; ++i) u = __dadd_rn(u, __dmul_rn(L[tri(i, j)], r[i]));
            ss = (j == 0) ? __dmul_rn(u, u) : __dadd_rn(ss, __dmul_rn(u, u));
        }
        double s = degenerate ? 0.0 : __dsqrt_rn(ss);
        m_r[ri * Gev + e] = acc;
        s_r[ri * Gev + e] = s;
        thr[ri * Gev + e] = live ? __dmul_rn(mult, s) : -1.0;
    }
}

extern "C" int ndg_project(int n, int64_t Gev, const double* mean64, const double* chol64, const uint8_t* eflags,
                           const double* dirs, int k, double multiplier, double* m_r, double* s_r, double* thr,
                           void* stream) {
    if (!ndg_supported_dims(n)) return NDG_ERR_UNSUPPORTED_DIMS;
    NDG_REQUIRE(k >= 1 && k <= 256, "k must be in 1..256");
    if (Gev == 0) return NDG_OK;
    const int threads = spread_threads(Gev, 128);
    const int64_t gx = (Gev + threads - 1) / threads;
    // projections per CTA: all k, or fewer (blockIdx.y) when the Gaussians alone leave SMs idle
    const int kpb = (int)std::max<int64_t>(1, std::min<int64_t>(k, gx * k / (2 * 148)));
    project_kernel<<<dim3((unsigned)gx, (unsigned)((k + kpb - 1) / kpb)), threads, sizeof(double) * k * n,
                     as_stream(stream)>>>(n, Gev, mean64, chol64, eflags, dirs, k, multiplier, m_r, s_r, thr, kpb);
    NDG_CHECK_LAUNCH();
    return NDG_OK;
}

// ---------------------------------------------------------------------------------------------
// K3 tile bounds: TileBounds. One CTA per tile, one thread per query.
// ---------------------------------------------------------------------------------------------
__global__ void tile_bounds_kernel(int n, int tile, const float* __restrict__ q, const double* __restrict__ dirs,
                                   int k, double* __restrict__ lo, double* __restrict__ hi, int kpb) {
    __shared__ double s_lo[32], s_hi[32];
    const int64_t t = blockIdx.x;
    const int qi = threadIdx.x;
    const bool valid = qi < tile;
    float x[NMAX];
#pragma unroll
    for (int j = 0; j < NMAX; ++j) x[j] = (valid && j < n) ? q[(t * tile + qi) * n + j] : 0.f;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarps = blockDim.x >> 5;
    const int r0 = blockIdx.y * kpb, r1 = min(k, r0 + kpb);   // this CTA's projections (blockIdx.y)
    for (int ri = r0; ri < r1; ++ri) {
        const double* r = dirs + ri * n;
        double acc = __dmul_rn((double)x[0], r[0]);
#pragma unroll
        for (int j = 1; j < NMAX; ++j)
            if (j < n) acc = __dadd_rn(acc, __dmul_rn((double)x[j], r[j]));
        double mn = valid ? acc : INFINITY, mx = valid ? acc : -INFINITY;
#pragma unroll
        for (int o = 16; o; o >>= 1) {
            mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
            mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        }
        if (lane == 0) {
            s_lo[warp] = mn;
            s_hi[warp] = mx;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            for (int w = 1; w < nwarps; ++w) {
                mn = fmin(mn, s_lo[w]);
                mx = fmax(mx, s_hi[w]);
            }
            lo[t * k + ri] = mn;
            hi[t * k + ri] = mx;
        }
        __syncthreads();
    }
}

extern "C" int ndg_tile_bounds(int n, int64_t B, int tile, const float* queries, const double* dirs, int k,
                               double* lo, double* hi, void* stream) {
    if (!ndg_supported_dims(n)) return NDG_ERR_UNSUPPORTED_DIMS;
    NDG_REQUIRE(tile >= 1 && tile <= 1024 && B % tile == 0, "tile must be in 1..1024 and divide B");
    NDG_REQUIRE(k >= 1 && k <= 256, "k must be in 1..256");
    int64_t T = B / tile;
    if (T == 0) return NDG_OK;
    int threads = ((tile + 31) / 32) * 32;
    const int kpb = (int)std::max<int64_t>(1, std::min<int64_t>(k, T * k / (2 * 148)));   // split k when T is small
    tile_bounds_kernel<<<dim3((unsigned)T, (unsigned)((k + kpb - 1) / kpb)), threads, 0, as_stream(stream)>>>(
        n, tile, queries, dirs, k, lo, hi, kpb);
    NDG_CHECK_LAUNCH();
    return NDG_OK;
}

// ---------------------------------------------------------------------------------------------
// K1c centred records for very sharp mixtures (HotPath centres the FP32 kernels when the z-GEMM
// conditioning says rho x + nb2 would cancel): a copy of K1's records with the nb2 pair of row i
// replaced by (m_hi, m_lo), the float32 head and tail of the float64 mean, so the FP32 K5 / K7 evaluate
// z_i = rho_i ((x_i - m_hi) - m_lo) + sum_k l_ik z_k, exact near the Gaussian (Sterbenz).
// ---------------------------------------------------------------------------------------------
__global__ void centre_records_kernel(int n, int64_t Gev, const double* __restrict__ mean64,
                                      const float* __restrict__ rec, float* __restrict__ rec_c) {
    const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (e >= Gev) return;
    const int RS = rec_floats(n);
    for (int k = 0; k < RS; ++k) rec_c[e * RS + k] = rec[e * RS + k];
    for (int i = 0; i < n; ++i) {
        const double m = mean64[e * n + i];
        const float hi = (float)m;
        rec_c[e * RS + rec_nb2(n) + 2 * i] = hi;
        rec_c[e * RS + rec_nb2(n) + 2 * i + 1] = (float)(m - (double)hi);
    }
}

extern "C" int ndg_centre_records(int n, int64_t Gev, const double* mean64, const float* rec, float* rec_c,
                                  void* stream) {
    if (!ndg_supported_dims(n)) return NDG_ERR_UNSUPPORTED_DIMS;
    if (Gev == 0) return NDG_OK;
    centre_records_kernel<<<(unsigned)((Gev + 127) / 128), 128, 0, as_stream(stream)>>>(n, Gev, mean64, rec, rec_c);
    NDG_CHECK_LAUNCH();
    return NDG_OK;
}

// ---------------------------------------------------------------------------------------------
// K4a cull mask: cull_tile for all tiles. Thread = evaluated Gaussian, CTA =
// 256 Gaussians x TILES tiles; the tiles' intervals sit in shared memory and are broadcast, the
// Gaussian's (m_r, thr) live in registers for k <= 16 (read through L1 for larger k, which keeps the
// shared memory at 2 * 16 * k doubles for any k <= 256). Culled iff any
// vector has lo - m_r > thr or m_r - hi > thr (FP64; the same predicate as
// max(lo - m_r, m_r - hi, 0) > multiplier * s_r); thr < 0 = never evaluated. Warp ballot -> one mask
// word per 32 Gaussians; per-CTA popcount -> one atomic per tile.
// ---------------------------------------------------------------------------------------------
constexpr int kCullThreads = 256;
constexpr int kCullRegK = 16;          // k handled from registers
constexpr int kCullTilesReg = 64;      // tiles per CTA on the register path (amortises the (m_r, thr) loads)
constexpr int kCullTilesSmem = 16;

template <bool REG, bool FULL>
__global__ void __launch_bounds__(kCullThreads) cull_mask_kernel(int64_t T, int k, int64_t Gev,
                                                                  const double* __restrict__ lo,
                                                                  const double* __restrict__ hi,
                                                                  const double* __restrict__ m_r,
                                                                  const double* __restrict__ thr,
                                                                  uint32_t* __restrict__ mask,
                                                                  int64_t* __restrict__ counts,
                                                                  const unsigned long long* __restrict__ skip,
                                                                  int tpc_rt) {
    constexpr int TILES = REG ? kCullTilesReg : kCullTilesSmem;
    const int tpc = FULL ? TILES : tpc_rt;       // tiles per CTA (FULL: the compile-time maximum)
    if (skip && *skip) return;                     // the bucket pre-filter (ndg_cull_prefilter) took this step
    extern __shared__ double sm[];
    double* s_lo = sm;                             // [TILES][k]
    double* s_hi = s_lo + TILES * k;
    __shared__ int s_cnt[TILES][kCullThreads / 32];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t e = blockIdx.x * (int64_t)kCullThreads + tid;
    const int64_t t0 = blockIdx.y * (int64_t)tpc;
    const int ntile = (int)imin64(tpc, T - t0);
    for (int x = tid; x < ntile * k; x += kCullThreads) {
        s_lo[x] = lo[t0 * k + x];
        s_hi[x] = hi[t0 * k + x];
    }
    double mr_r[kCullRegK], th_r[kCullRegK];
    bool never;
    if constexpr (REG) {
#pragma unroll
        for (int ri = 0; ri < kCullRegK; ++ri) {
            mr_r[ri] = (ri < k && e < Gev) ? m_r[ri * Gev + e] : 0.0;
            th_r[ri] = (ri < k && e < Gev) ? thr[ri * Gev + e] : -1.0;
        }
        never = th_r[0] < 0.0;
    } else {
        never = (e < Gev ? thr[e] : -1.0) < 0.0;
    }
    __syncthreads();
    const int64_t W = (Gev + 31) / 32;
    for (int tt = 0; tt < ntile; ++tt) {
        bool kept = !never;
        if constexpr (REG) {
#ifdef NDG_CULL_EARLY_EXIT
#pragma unroll
            for (int ri = 0; ri < kCullRegK; ++ri) {
                if (ri < k && kept) {
                    const double l = s_lo[tt * k + ri], h = s_hi[tt * k + ri];
                    if (__dsub_rn(l, mr_r[ri]) > th_r[ri] || __dsub_rn(mr_r[ri], h) > th_r[ri]) kept = false;
                }
            }
#else
            // all k tests, branch-free: independent FP64 chains instead of a serial test-and-branch
#pragma unroll
            for (int ri = 0; ri < kCullRegK; ++ri) {
                if (ri < k) {
                    const double l = s_lo[tt * k + ri], h = s_hi[tt * k + ri];
                    kept &= !(__dsub_rn(l, mr_r[ri]) > th_r[ri]) & !(__dsub_rn(mr_r[ri], h) > th_r[ri]);
                }
            }
#endif
        } else {
            for (int ri = 0; ri < k && kept; ++ri) {          // kept is false for e >= Gev (never)
                const double mr = __ldg(m_r + ri * Gev + e), th = __ldg(thr + ri * Gev + e);
                const double l = s_lo[tt * k + ri], h = s_hi[tt * k + ri];
                if (__dsub_rn(l, mr) > th || __dsub_rn(mr, h) > th) kept = false;
            }
        }
        const uint32_t word = __ballot_sync(0xffffffffu, kept);
        if (lane == 0) {
            const int64_t wi = e >> 5;
            if (wi < W) mask[(t0 + tt) * W + wi] = word;
            s_cnt[tt][warp] = __popc(word);
        }
    }
    __syncthreads();
    if (tid < ntile) {
        int c = 0;
        for (int w = 0; w < kCullThreads / 32; ++w) c += s_cnt[tid][w];
        if (c) atomicAdd(reinterpret_cast<unsigned long long*>(&counts[t0 + tid]), (unsigned long long)c);
    }
}

int cull_mask_launch(int64_t T, int k, int64_t Gev, const double* lo, const double* hi, const double* m_r,
                     const double* thr, uint32_t* mask, int64_t* counts, const unsigned long long* skip,
                     cudaStream_t stream) {
    NDG_REQUIRE(k >= 1 && k <= 256, "k must be in 1..256 for the cull kernel");
    if (T == 0 || Gev == 0) return NDG_OK;
    const bool reg = k <= kCullRegK;
    const int tiles = reg ? kCullTilesReg : kCullTilesSmem;
    // tiles per CTA: up to `tiles` (amortises the per-Gaussian bound loads), fewer when that would leave
    // SMs idle (small configurations: cfg1's 16 Gaussian blocks x 64 tiles would run on 16 SMs)
    const int64_t gx = (Gev + kCullThreads - 1) / kCullThreads;
    const int tpc = (int)std::max<int64_t>(1, std::min<int64_t>(tiles, T * gx / (2 * 148)));
    dim3 grid((unsigned)gx, (unsigned)((T + tpc - 1) / tpc));
    NDG_REQUIRE(grid.y <= 65535, "too many tiles for one cull launch");
    const size_t smem = sizeof(double) * 2 * tiles * k;    // <= 64 KB at k = 256
    static DeviceOnce attr_set;
    if (attr_set.first()) {
        cudaFuncSetAttribute(cull_mask_kernel<false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
        cudaFuncSetAttribute(cull_mask_kernel<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
        cudaFuncSetAttribute(cull_mask_kernel<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
        cudaFuncSetAttribute(cull_mask_kernel<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
    }
    // the full-CTA case keeps the tile count a compile-time constant (the runtime bound costs 13%)
    const bool full = tpc == tiles;
    if (reg && full)
        cull_mask_kernel<true, true><<<grid, kCullThreads, smem, stream>>>(T, k, Gev, lo, hi, m_r, thr, mask, counts,
                                                                           skip, tpc);
    else if (reg)
        cull_mask_kernel<true, false><<<grid, kCullThreads, smem, stream>>>(T, k, Gev, lo, hi, m_r, thr, mask, counts,
                                                                            skip, tpc);
    else if (full)
        cull_mask_kernel<false, true><<<grid, kCullThreads, smem, stream>>>(T, k, Gev, lo, hi, m_r, thr, mask, counts,
                                                                            skip, tpc);
    else
        cull_mask_kernel<false, false><<<grid, kCullThreads, smem, stream>>>(T, k, Gev, lo, hi, m_r, thr, mask, counts,
                                                                             skip, tpc);
    NDG_CHECK_LAUNCH();
    return NDG_OK;
}

extern "C" int ndg_cull_mask(int64_t T, int k, int64_t Gev, const double* lo, const double* hi, const double* m_r,
                             const double* thr, uint32_t* mask, int64_t* counts, void* stream) {
    return cull_mask_launch(T, k, Gev, lo, hi, m_r, thr, mask, counts, nullptr, as_stream(stream));
}

// ---------------------------------------------------------------------------------------------
// K4b exclusive scan of the per-tile counts (single CTA, chunked Hillis-Steele in shared memory).
// ---------------------------------------------------------------------------------------------
__global__ void scan_counts_kernel(int64_t T, const int64_t* __restrict__ counts, int64_t* __restrict__ offsets,
                                   int64_t* __restrict__ chunk_offsets) {
    __shared__ int64_t s_a[1024], s_b[1024];
    __shared__ int64_t carry_a, carry_b;
    if (threadIdx.x == 0) carry_a = carry_b = 0;
    __syncthreads();
    for (int64_t base = 0; base < T; base += 1024) {
        const int64_t t = base + threadIdx.x;
        const int64_t c = t < T ? counts[t] : 0;
        s_a[threadIdx.x] = c;
        s_b[threadIdx.x] = (c + kBwdChunk - 1) / kBwdChunk;
        __syncthreads();
        for (int o = 1; o < 1024; o <<= 1) {
            int64_t va = threadIdx.x >= o ? s_a[threadIdx.x - o] : 0;
            int64_t vb = threadIdx.x >= o ? s_b[threadIdx.x - o] : 0;
            __syncthreads();
            s_a[threadIdx.x] += va;
            s_b[threadIdx.x] += vb;
            __syncthreads();
        }
        if (t < T) {   // inclusive -> offsets[t + 1]
            offsets[t + 1] = carry_a + s_a[threadIdx.x];
            chunk_offsets[t + 1] = carry_b + s_b[threadIdx.x];
        }
        __syncthreads();
        if (threadIdx.x == 1023) {
            carry_a += s_a[1023];
            carry_b += s_b[1023];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        offsets[0] = 0;
        chunk_offsets[0] = 0;
    }
}

extern "C" int ndg_scan_counts(int64_t T, const int64_t* counts, int64_t* offsets, int64_t* chunk_offsets,
                               void* stream) {
    scan_counts_kernel<<<1, 1024, 0, as_stream(stream)>>>(T, counts, offsets, chunk_offsets);
    NDG_CHECK_LAUNCH();
    return NDG_OK;
}

// ---------------------------------------------------------------------------------------------
// K7 work items in band order. One CTA per band of kBand tiles writes that band's items
// (t << 32 | c) into items[chunk_offsets[b0] .. chunk_offsets[b1]): the first cmin chunks (cmin = the
// fewest any tile of the band has) chunk-major -- all of the band's tiles on chunk 0, then on chunk 1 --
// so the CTAs in flight at one time share the same Gaussians' records and accumulators in L2 (dense
// regimes: every tile's list is almost the whole mixture), the remaining chunks tile-major after them.
// ---------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(256) work_items_kernel(int64_t T, const int64_t* __restrict__ chunk_off,
                                                         int64_t* __restrict__ items) {
    __shared__ int64_t s_ex[kBand + 1];
    __shared__ int64_t s_min;
    const int64_t b0 = (int64_t)blockIdx.x * kBand, b1 = imin64(b0 + kBand, T);
    const int nb = (int)(b1 - b0);
    if (threadIdx.x == 0) s_min = INT64_MAX;
    __syncthreads();
    int64_t mn = INT64_MAX;
    for (int i = threadIdx.x; i < nb; i += blockDim.x) mn = min(mn, chunk_off[b0 + i + 1] - chunk_off[b0 + i]);
    atomicMin(reinterpret_cast<unsigned long long*>(&s_min), (unsigned long long)mn);
    __syncthreads();
    const int64_t cmin = s_min;
    if (threadIdx.x == 0) {                       // exclusive prefix of the extra chunks per tile
        int64_t a = 0;
        for (int i = 0; i < nb; ++i) {
            s_ex[i] = a;
            a += chunk_off[b0 + i + 1] - chunk_off[b0 + i] - cmin;
        }
        s_ex[nb] = a;
    }
    __syncthreads();
    const int64_t base = chunk_off[b0], head = cmin * nb, total = head + s_ex[nb];
    for (int64_t i = threadIdx.x; i < total; i += blockDim.x) {
        int64_t t, c;
        if (i < head) {
            c = i / nb;
            t = b0 + i % nb;
        } else {
            const int64_t j = i - head;
            int lo = 0, hi = nb;                  // s_ex[lo] <= j < s_ex[lo + 1]
            while (hi - lo > 1) {
                const int mid = (lo + hi) >> 1;
                if (s_ex[mid] <= j) lo = mid;
                else hi = mid;
            }
            t = b0 + lo;
            c = cmin + (j - s_ex[lo]);
        }
        NDG_DCHECK(t >= b0 && t < b1 && c >= 0 && c < chunk_off[t + 1] - chunk_off[t] && base + i < chunk_off[b1]);
        items[base + i] = (t << 32) | c;
    }
}

extern "C" int ndg_work_items(int64_t T, const int64_t* chunk_offsets, int64_t* items, void* stream) {
    if (T <= 0) return NDG_OK;
    work_items_kernel<<<(unsigned)((T + kBand - 1) / kBand), 256, 0, as_stream(stream)>>>(T, chunk_offsets, items);
    NDG_CHECK_LAUNCH();
    return NDG_OK;
}

// ---------------------------------------------------------------------------------------------
// Bounds of the deterministic backward reduction (ndg_common.cuh): H = max_q sum_c |dpred_c|,
// Dmax = max_q,c |dpred_c|, Lmax = max_q ell over the step's query records, Amax = max |a_c| over live
// Gaussians -- as float bit patterns (uint32 atomicMax of non-negative values; `bounds` zeroed by the
// caller). Order-independent, so the scales every K7 launch derives from them are deterministic.
// Non-finite inputs are left out: the partials they enter are themselves non-finite and flag only
// their own Gaussians (-> NonFiniteGradientError naming the component).
// ---------------------------------------------------------------------------------------------
__global__ void bwd_bounds_kernel(int n, int64_t B, const float* __restrict__ qrec, int64_t Gev,
                                  const float* __restrict__ rec, const uint8_t* __restrict__ eflags,
                                  uint32_t* __restrict__ bounds) {
    const int QS = qrec_floats(n), RS = rec_floats(n), A0 = rec_a(n);
    uint32_t h = 0, d = 0, l = 0, am = 0;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < B; q += stride) {
        const float* r = qrec + q * QS + n;
        const float a0 = fabsf(r[0]), a1 = fabsf(r[1]), a2 = fabsf(r[2]);
        if (!isfinite(a0 + a1 + a2 + r[3])) continue;   // a non-finite query flags only the pairs it enters
        h = max(h, __float_as_uint(a0 + a1 + a2));
        d = max(d, max(__float_as_uint(a0), max(__float_as_uint(a1), __float_as_uint(a2))));
        l = max(l, __float_as_uint(fabsf(r[3])));
    }
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < Gev; e += stride) {
        if ((eflags[e] & 3) != 1) continue;       // live, not degenerate
        const float* r = rec + e * RS + A0;
        if (!isfinite(r[0] + r[1] + r[2])) continue;
        am = max(am, max(__float_as_uint(fabsf(r[0])), max(__float_as_uint(fabsf(r[1])), __float_as_uint(fabsf(r[2])))));
    }
    h = __reduce_max_sync(0xffffffffu, h);
    d = __reduce_max_sync(0xffffffffu, d);
    l = __reduce_max_sync(0xffffffffu, l);
    am = __reduce_max_sync(0xffffffffu, am);
    if ((threadIdx.x & 31) == 0) {
        if (h) atomicMax(bounds + 0, h);
        if (d) atomicMax(bounds + 1, d);
        if (l) atomicMax(bounds + 2, l);
        if (am) atomicMax(bounds + 3, am);
    }
}

extern "C" int ndg_bwd_bounds(int n, int64_t B, const float* qrec, int64_t Gev, const float* rec,
                              const uint8_t* eflags, uint32_t* bounds, void* stream) {
    if (!ndg_supported_dims(n)) return NDG_ERR_UNSUPPORTED_DIMS;
    bwd_bounds_kernel<<<148 * 4, 256, 0, as_stream(stream)>>>(n, B, qrec, Gev, rec, eflags, bounds);
    NDG_CHECK_LAUNCH();
    return NDG_OK;
}

// ---------------------------------------------------------------------------------------------
// Fixed point -> float64 accumulators, in place over the hi words (acc = [2][Gev][A] int64 -> the
// first Gev * A words become float64). A flagged Gaussian gets NaN in every slot (its flag slot's
// output is NaN too, so a thread reading the flag after it was overwritten still sees nonzero bits).
// ---------------------------------------------------------------------------------------------
__global__ void acc_dequant_kernel(int n, int64_t Gev, int64_t B, const uint32_t* __restrict__ bounds,
                                   long long* __restrict__ acc) {
    const int A = acc_doubles(n), F = acc_flag(n), T0 = acc_tail(n);
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= Gev * A) return;
    const int j = (int)(i % A);
    const int64_t e = i / A;
    const FxScales fx = fx_scales(bounds, B);
    const long long hi = acc[i], lo = acc[Gev * A + i];
    const bool bad = acc[e * A + F] != 0;
    double v;
    if (bad) {
        v = __longlong_as_double(0x7ff8000000000000LL);
    } else if (j == F) {
        v = 0.0;
    } else if (j == T0 + 5) {
        v = (double)hi;                                  // pairs: exact count
    } else {
        const double sc = (j < F || j == T0 + 4) ? fx.h : (j < T0 + 3 ? fx.g : fx.l);
        v = (double)hi / sc + (double)lo / (sc * kFxLo);
    }
    reinterpret_cast<double*>(acc)[i] = v;
}

extern "C" int ndg_acc_dequant(int n, int64_t Gev, int64_t B, const uint32_t* bounds, int64_t* acc, void* stream) {
    if (!ndg_supported_dims(n)) return NDG_ERR_UNSUPPORTED_DIMS;
    const int64_t total = Gev * acc_doubles(n);
    if (total == 0) return NDG_OK;
    acc_dequant_kernel<<<(unsigned)((total + 255) / 256), 256, 0, as_stream(stream)>>>(
        n, Gev, B, bounds, reinterpret_cast<long long*>(acc));
    NDG_CHECK_LAUNCH();
    return NDG_OK;
}

// ---------------------------------------------------------------------------------------------
// K4c compaction: CTA per tile; block prefix scan of per-word popcounts, then each thread writes
// the ascending indices of its word's set bits.
// ---------------------------------------------------------------------------------------------
constexpr int kCompactThreads = 256;

__global__ void __launch_bounds__(kCompactThreads) compact_kernel(int64_t Gev, const uint32_t* __restrict__ mask,
                                                                   const int64_t* __restrict__ offsets,
                                                                   int32_t* __restrict__ idx) {
    __shared__ int s_warp[kCompactThreads / 32];
    __shared__ int64_t s_base;
    const int64_t t = blockIdx.x;
    const int64_t W = (Gev + 31) / 32;
    const uint32_t* row = mask + t * W;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) s_base = offsets[t];
    __syncthreads();
    for (int64_t w0 = 0; w0 < W; w0 += kCompactThreads) {
        const int64_t wi = w0 + tid;
        uint32_t word = wi < W ? row[wi] : 0u;
        int c = __popc(word), incl = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            int v = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += v;
        }
        if (lane == 31) s_warp[warp] = incl;
        __syncthreads();
        int before = 0, total = 0;
        for (int w = 0; w < kCompactThreads / 32; ++w) {
            if (w < warp) before += s_warp[w];
            total += s_warp[w];
        }
        const int64_t pos = s_base + before + incl - c;
        // warp-cooperative expansion: word `src` of the warp is written by all lanes (lane l writes the
        // index of bit l), so dense words become one coalesced 128-B store instead of 32 strided ones
        for (int src = 0; src < 32; ++src) {
            const uint32_t wd = __shfl_sync(0xffffffffu, word, src);
            if (wd == 0u) continue;                               // warp-uniform
            const int64_t p = __shfl_sync(0xffffffffu, pos, src);
            if ((wd >> lane) & 1u) {
                const int64_t at = p + __popc(wd & ((1u << lane) - 1u));
                NDG_DCHECK(at >= offsets[t] && at < offsets[t + 1] && (w0 + warp * 32 + src) * 32 + lane < Gev);
                idx[at] = (int32_t)((w0 + warp * 32 + src) * 32 + lane);
            }
        }
        __syncthreads();
        if (tid == 0) s_base += total;
        __syncthreads();
    }
}

extern "C" int ndg_cull_compact(int64_t T, int64_t Gev, const uint32_t* mask, const int64_t* offsets, int32_t* idx,
                                void* stream) {
    if (T == 0 || Gev == 0) return NDG_OK;
    compact_kernel<<<(unsigned)T, kCompactThreads, 0, as_stream(stream)>>>(Gev, mask, offsets, idx);
    NDG_CHECK_LAUNCH();
    return NDG_OK;
}

// ---------------------------------------------------------------------------------------------
// Loss finalisation: fixed-order float64 sum of the per-tile partials (deterministic).
// ---------------------------------------------------------------------------------------------
__global__ void loss_finalize_kernel(int64_t T, const double* __restrict__ part, double* __restrict__ loss) {
    __shared__ double s[256];
    double acc = 0.0;
    for (int64_t t = threadIdx.x; t < T; t += 256) acc += part[t];
    s[threadIdx.x] = acc;
    __syncthreads();
    for (int o = 128; o; o >>= 1) {
        if (threadIdx.x < o) s[threadIdx.x] += s[threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x == 0) *loss = s[0];
}

// ---------------------------------------------------------------------------------------------
// Standalone loss_rel_l2 for the module-level API (the training step fuses it into
// K5): per 256-query block a float64 partial (fixed-order tree), then ndg_loss_finalize. dpred (may be
// NULL) = 2 (p - t) / (p^2 + eps) / (3 n_total), the gradient with the denominator detached (:291).
// ---------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(256) loss_rel_l2_kernel(int64_t B, const float* __restrict__ pred,
                                                          const float* __restrict__ target, double eps, int64_t n_total,
                                                          float* __restrict__ dpred, double* __restrict__ part) {
    __shared__ double s[256];
    const int64_t b = blockIdx.x * 256LL + threadIdx.x;
    double l = 0.0;
    if (b < B) {
        const double inv = 1.0 / (3.0 * (double)n_total);
        for (int c = 0; c < 3; ++c) {
            const double p = pred[b * 3 + c], d = p - (double)target[b * 3 + c], den = p * p + eps;
            l += d * d / den;
            if (dpred) dpred[b * 3 + c] = (float)(2.0 * d / den * inv);
        }
        l *= inv;
    }
    s[threadIdx.x] = l;
    __syncthreads();
    for (int o = 128; o; o >>= 1) {
        if (threadIdx.x < o) s[threadIdx.x] += s[threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x == 0) part[blockIdx.x] = s[0];
}

extern "C" int ndg_loss_rel_l2(int64_t B, const float* pred, const float* target, double eps, int64_t n_total,
                               float* dpred, double* loss_partial, void* stream) {
    NDG_REQUIRE(eps > 0.0 && n_total >= 1, "eps > 0 and n_total >= 1 required (SPEC.md:255)");
    if (B == 0) return NDG_OK;
    loss_rel_l2_kernel<<<(unsigned)((B + 255) / 256), 256, 0, as_stream(stream)>>>(B, pred, target, eps, n_total,
                                                                                    dpred, loss_partial);
    NDG_CHECK_LAUNCH();
    return NDG_OK;
}

extern "C" int ndg_loss_finalize(int64_t T, const double* loss_partial, double* loss, void* stream) {
    loss_finalize_kernel<<<1, 256, 0, as_stream(stream)>>>(T, loss_partial, loss);
    NDG_CHECK_LAUNCH();
    return NDG_OK;
}

// ---------------------------------------------------------------------------------------------
// K8 epilogue: tail of backward. Thread per component; float64.
//   per evaluated Gaussian: S = -S'/C^2, t = -t'/C; G_L = -tril(L^-T S), dm = -L^-T t
//   parent: d mean_raw = dm; d chol_raw = G_L * (L_ii | (1 - L_ij^2)/2)
//   child (L_c = L U, m_c = L m_u + m_p): dU = tril(L^T G_Lc), dm_u = L^T dm_c,
//          parent += tril(G_Lc U^T) + tril(dm_c m_u^T) on L and dm_c on the mean.
//   colour / amplitude: d color_raw = gA * alpha * c (1 - c); d amp_raw = (gA . c) * alpha'.
// ---------------------------------------------------------------------------------------------

// One thread per component (large G: enough components to fill the GPU; see epilogue_kernel). Templated on
// N with the solve done in place (S -> X -> G_L in one N x N array), so its float64 scratch is 2 N^2 + P + 2N
// doubles instead of 4 x 16^2 + 136 + 32 (the local-memory traffic that made it DRAM-bound: 1 GB at 100k
// components). Same operations in the same order as before, so the same bits.
template <int N>
__global__ void epilogue_thread_kernel(int64_t G, int64_t Gev, int amp_mode, const float* __restrict__ params,
                                       const float* __restrict__ child, const uint8_t* __restrict__ flags,
                                       const uint8_t* __restrict__ eflags, const double* __restrict__ chol64,
                                       const double* __restrict__ accum, float* __restrict__ gp,
                                       float* __restrict__ gc, float* __restrict__ stats, ndg_status* st) {
    constexpr int n = N;
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= G) return;
    constexpr int P = n_chol(N), R = raw_floats(N), A = acc_doubles(N);
    double GLp[N * N], dmp[N];
    double X[N * N];                     // S, then X = L^-T S in place, then G_L = -tril(X) in place
    for (int t = 0; t < n * n; ++t) GLp[t] = 0.0;
    for (int r = 0; r < n; ++r) dmp[r] = 0.0;
    float* op = gp + i * R;
    float* oc = gc ? gc + i * R : nullptr;
    for (int t = 0; t < R; ++t) op[t] = 0.f;
    if (oc)
        for (int t = 0; t < R; ++t) oc[t] = 0.f;
    const double* Lp = chol64 + i * P;
    const double invC = 1.0 / kC, invC2 = invC * invC;
    const int nev = (Gev == 2 * G) ? 2 : 1;
    for (int which = 0; which < nev; ++which) {
        const int64_t e = which ? G + i : i;
        const double* acc = accum + e * A;
        float* so = stats + e * kNumStats;
        if (!(eflags[e] & 1)) {
            so[0] = so[1] = so[2] = 0.f;
            continue;
        }
        so[0] = (float)acc[acc_tail(n) + 3];
        so[1] = (float)(acc[acc_tail(n) + 4] * invC);
        so[2] = (float)acc[acc_tail(n) + 5];
        const double* Le = chol64 + e * P;
        for (int r = 0; r < n; ++r)
            for (int c = 0; c <= r; ++c) X[r * n + c] = X[c * n + r] = -acc[tri(r, c)] * invC2;
        for (int c = 0; c < n; ++c)                      // X = L^-T S, column c, rows n-1 .. 0, in place
            for (int r = n - 1; r >= 0; --r) {
                double a = X[r * n + c];
                for (int k = r + 1; k < n; ++k) a -= Le[tri(k, r)] * X[k * n + c];
                X[r * n + c] = a / Le[tri(r, r)];
            }
        double* GL = X;
        for (int r = 0; r < n; ++r)
            for (int c = 0; c < n; ++c) GL[r * n + c] = c <= r ? -X[r * n + c] : 0.0;
        double dm[N];
        for (int r = n - 1; r >= 0; --r) {   // dm = -L^-T t (single-column back substitution)
            double a = -acc[P + r] * invC;
            for (int k = r + 1; k < n; ++k) a -= Le[tri(k, r)] * dm[k];
            dm[r] = a / Le[tri(r, r)];
        }
        for (int r = 0; r < n; ++r) dm[r] = -dm[r];
        const float* row = which ? child + i * R : params + i * R;
        float* out = which ? oc : op;
        const double ar = (double)row[n + P + 3];
        const double alpha = amp_mode == NDG_BRIGHTNESS ? exp(ar) : sigmoid64(ar);
        double dalpha = 0.0;
        for (int ch = 0; ch < 3; ++ch) {
            const double cc = sigmoid64((double)row[n + P + ch]);
            const double gA = acc[acc_tail(n) + ch];
            out[n + P + ch] = (float)(gA * alpha * cc * (1.0 - cc));
            dalpha += gA * cc;
        }
        out[n + P + 3] = (float)(dalpha * (amp_mode == NDG_BRIGHTNESS ? alpha : alpha * (1.0 - alpha)));
        if (!which) {
            for (int t = 0; t < n * n; ++t) GLp[t] += GL[t];
            for (int r = 0; r < n; ++r) dmp[r] += dm[r];
        } else {
            const float* crow = child + i * R;
            double U[P];
            for (int r = 0; r < n; ++r)
                for (int c = 0; c <= r; ++c) {
                    const double raw = (double)crow[n + tri(r, c)];
                    U[tri(r, c)] = (r == c) ? exp(raw) : act_offdiag(raw);
                }
            for (int r = 0; r < n; ++r)
                for (int c = 0; c <= r; ++c) {
                    double s1 = 0.0, s2 = 0.0;
                    for (int k = 0; k <= c; ++k) s1 += GL[r * n + k] * U[tri(c, k)];   // (G U^T)_rc
                    for (int k = r; k < n; ++k) s2 += Lp[tri(k, r)] * GL[k * n + c];  // (L^T G)_rc
                    GLp[r * n + c] += s1 + dm[r] * (double)crow[c];
                    const double d = s2 * (r == c ? U[tri(r, r)] : (1.0 - U[tri(r, c)] * U[tri(r, c)]) * 0.5);
                    out[n + tri(r, c)] = (float)d;
                }
            for (int r = 0; r < n; ++r) {
                double s = 0.0;
                for (int k = r; k < n; ++k) s += Lp[tri(k, r)] * dm[k];
                out[r] = (float)s;
                dmp[r] += dm[r];
            }
        }
    }
    for (int r = 0; r < n; ++r) op[r] = (float)dmp[r];
    for (int r = 0; r < n; ++r)
        for (int c = 0; c <= r; ++c) {
            const double l = Lp[tri(r, c)];
            op[n + tri(r, c)] = (float)(GLp[r * n + c] * (r == c ? l : (1.0 - l * l) * 0.5));
        }
    // non-finite gradient -> NonFiniteGradientError
    for (int which = 0; which < nev; ++which) {
        const float* out = which ? oc : op;
        for (int t = 0; t < R; ++t)
            if (!isfinite(out[t])) {
                record_key(&st->nonfinite_key, (which ? G * R : 0) + i * R + t);
                break;
            }
    }
}

// Warp per component, for small G (cfg1: 4096 components are 128 one-thread-per-component warps): lane c
// runs column c of X = L^-T S (back substitution), and the P-entry and n-entry loops of the chain rule are
// spread over the lanes; the matrices live in the warp's slice of shared memory. Every value is computed in
// the same order as in epilogue_thread_kernel, so the two give the same bits. At 100k components the warp
// form is issue-bound on its lane-serial parts (436 vs 348 us), so large G keeps one thread per component.
constexpr int kEpiWarps = 8;
constexpr int64_t kEpiWarpMaxG = 16384;   // the warp form up to here (cfg1 4096: 37 -> ~20 us), threads beyond

__host__ __device__ constexpr int epi_doubles(int n) { return 3 * n_chol(n) + 2 * n * n + 2 * n; }   // per warp

__device__ __forceinline__ void tri_rc(int t, int& r, int& c) {   // packed lower index -> (row, col)
    r = (int)((sqrtf(8.f * t + 1.f) - 1.f) * 0.5f);
    r += (r + 1) * (r + 2) / 2 <= t;
    r -= r * (r + 1) / 2 > t;
    c = t - r * (r + 1) / 2;
}

__global__ void __launch_bounds__(kEpiWarps * 32) epilogue_kernel(
    int n, int64_t G, int64_t Gev, int amp_mode, const float* __restrict__ params, const float* __restrict__ child,
    const uint8_t* __restrict__ flags, const uint8_t* __restrict__ eflags, const double* __restrict__ chol64,
    const double* __restrict__ accum, float* __restrict__ gp, float* __restrict__ gc, float* __restrict__ stats,
    ndg_status* st) {
    extern __shared__ double esm[];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int P = n_chol(n), R = raw_floats(n), A = acc_doubles(n), nn = n * n;
    double* sLp = esm + wib * epi_doubles(n);   // the parent's L (packed)
    double* sL = sLp + P;                       // L of the evaluated Gaussian e (packed)
    double* sU = sL + P;                        // the child's activated U (packed)
    double* sGL = sU + P;                       // X = L^-T S, then G_L = -tril(X) of e (dense n x n)
    double* sGLp = sGL + nn;                    // accumulated parent G_L (dense)
    double* sdm = sGLp + nn;                    // dm of e
    double* sdmp = sdm + n;                     // accumulated parent dm
    const int64_t i = blockIdx.x * (int64_t)kEpiWarps + wib;
    if (i >= G) return;                         // warp-uniform
    const double invC = 1.0 / kC, invC2 = invC * invC;
    float* op = gp + i * R;
    float* oc = gc ? gc + i * R : nullptr;
    for (int t = lane; t < R; t += 32) {
        op[t] = 0.f;
        if (oc) oc[t] = 0.f;
    }
    for (int t = lane; t < P; t += 32) sLp[t] = chol64[i * P + t];
    for (int t = lane; t < nn; t += 32) sGLp[t] = 0.0;
    for (int t = lane; t < n; t += 32) sdmp[t] = 0.0;
    const int nev = (Gev == 2 * G) ? 2 : 1;
    for (int which = 0; which < nev; ++which) {
        const int64_t e = which ? G + i : i;
        const double* acc = accum + e * A;
        float* so = stats + e * kNumStats;
        if (!(eflags[e] & 1)) {                 // warp-uniform
            if (lane == 0) so[0] = so[1] = so[2] = 0.f;
            continue;
        }
        if (lane == 0) {
            so[0] = (float)acc[acc_tail(n) + 3];
            so[1] = (float)(acc[acc_tail(n) + 4] * invC);
            so[2] = (float)acc[acc_tail(n) + 5];
        }
        for (int t = lane; t < P; t += 32) sL[t] = chol64[e * P + t];
        __syncwarp();
        if (lane < n) {                         // X[:, c] = L^-T S[:, c], S = -sym(S') / C^2
            const int c = lane;
            for (int r = n - 1; r >= 0; --r) {
                double a = -acc[r >= c ? tri(r, c) : tri(c, r)] * invC2;
                for (int k = r + 1; k < n; ++k) a -= sL[tri(k, r)] * sGL[k * n + c];
                sGL[r * n + c] = a / sL[tri(r, r)];
            }
        }
        __syncwarp();
        for (int t = lane; t < nn; t += 32) {
            const int r = t / n, c = t - (t / n) * n;
            sGL[t] = c <= r ? -sGL[t] : 0.0;
        }
        if (lane == 0) {                        // dm = -L^-T t (single-column back substitution)
            for (int r = n - 1; r >= 0; --r) {
                double a = -acc[P + r] * invC;
                for (int k = r + 1; k < n; ++k) a -= sL[tri(k, r)] * sdm[k];
                sdm[r] = a / sL[tri(r, r)];
            }
            for (int r = 0; r < n; ++r) sdm[r] = -sdm[r];
        }
        const float* row = which ? child + i * R : params + i * R;
        float* out = which ? oc : op;
        if (lane == 0) {                        // colour and amplitude
            const double ar = (double)row[n + P + 3];
            const double alpha = amp_mode == NDG_BRIGHTNESS ? exp(ar) : sigmoid64(ar);
            double dalpha = 0.0;
            for (int ch = 0; ch < 3; ++ch) {
                const double cc = sigmoid64((double)row[n + P + ch]);
                const double gA = acc[acc_tail(n) + ch];
                out[n + P + ch] = (float)(gA * alpha * cc * (1.0 - cc));
                dalpha += gA * cc;
            }
            out[n + P + 3] = (float)(dalpha * (amp_mode == NDG_BRIGHTNESS ? alpha : alpha * (1.0 - alpha)));
        }
        __syncwarp();
        if (!which) {
            for (int t = lane; t < nn; t += 32) sGLp[t] += sGL[t];
            for (int r = lane; r < n; r += 32) sdmp[r] += sdm[r];
        } else {
            const float* crow = child + i * R;
            for (int t = lane; t < P; t += 32) {
                int r, c;
                tri_rc(t, r, c);
                const double raw = (double)crow[n + t];
                sU[t] = (r == c) ? exp(raw) : act_offdiag(raw);
            }
            __syncwarp();
            for (int t = lane; t < P; t += 32) {
                int r, c;
                tri_rc(t, r, c);
                double s1 = 0.0, s2 = 0.0;
                for (int k = 0; k <= c; ++k) s1 += sGL[r * n + k] * sU[tri(c, k)];     // (G U^T)_rc
                for (int k = r; k < n; ++k) s2 += sLp[tri(k, r)] * sGL[k * n + c];    // (L^T G)_rc
                sGLp[r * n + c] += s1 + sdm[r] * (double)crow[c];
                const double d = s2 * (r == c ? sU[tri(r, r)] : (1.0 - sU[tri(r, c)] * sU[tri(r, c)]) * 0.5);
                out[n + t] = (float)d;
            }
            for (int r = lane; r < n; r += 32) {
                double s = 0.0;
                for (int k = r; k < n; ++k) s += sLp[tri(k, r)] * sdm[k];
                out[r] = (float)s;
                sdmp[r] += sdm[r];
            }
        }
        __syncwarp();
    }
    for (int r = lane; r < n; r += 32) op[r] = (float)sdmp[r];
    for (int t = lane; t < P; t += 32) {
        int r, c;
        tri_rc(t, r, c);
        const double l = sLp[t];
        op[n + t] = (float)(sGLp[r * n + c] * (r == c ? l : (1.0 - l * l) * 0.5));
    }
    __syncwarp();
    // non-finite gradient -> NonFiniteGradientError: the lowest offending entry of each row
    for (int which = 0; which < nev; ++which) {
        const float* out = which ? oc : op;
        for (int base = 0; base < R; base += 32) {
            const int t = base + lane;
            const unsigned m = __ballot_sync(0xffffffffu, t < R && !isfinite(out[t]));
            if (m) {
                if (lane == 0) record_key(&st->nonfinite_key, (which ? G * R : 0) + i * R + base + __ffs(m) - 1);
                break;
            }
        }
    }
}

extern "C" int ndg_epilogue(int n, int64_t G, int64_t Gev, int amp_mode, const float* params, const float* child,
                            const uint8_t* flags, const uint8_t* eflags, const double* chol64, const double* accum,
                            float* grad_params, float* grad_child, float* stats, ndg_status* status, void* stream) {
    if (!ndg_supported_dims(n)) return NDG_ERR_UNSUPPORTED_DIMS;
    NDG_REQUIRE(Gev == G || Gev == 2 * G, "Gev must be G or 2G");
    NDG_REQUIRE(Gev == G || (child && grad_child), "child rows and child gradients required when Gev == 2G");
    if (G == 0) return NDG_OK;
    // NDG_EPILOGUE_WARP_MAX overrides the crossover (tests pin the two forms against each other)
    static const int64_t warp_max = [] {
        const char* v = getenv("NDG_EPILOGUE_WARP_MAX");
        return v ? (int64_t)atoll(v) : kEpiWarpMaxG;
    }();
    if (G > warp_max) {
        const int threads = 64;
        const unsigned grid = (unsigned)((G + threads - 1) / threads);
        float* gch = Gev == 2 * G ? grad_child : nullptr;
        switch (n) {
#define NDG_CASE(NN)                                                                                      \
    case NN:                                                                                              \
        epilogue_thread_kernel<NN><<<grid, threads, 0, as_stream(stream)>>>(G, Gev, amp_mode, params, child, \
                                                                           flags, eflags, chol64, accum,  \
                                                                           grad_params, gch, stats, status); \
        break;
            NDG_CASE(1) NDG_CASE(2) NDG_CASE(3) NDG_CASE(4) NDG_CASE(5) NDG_CASE(6) NDG_CASE(7) NDG_CASE(8)
            NDG_CASE(9) NDG_CASE(10) NDG_CASE(11) NDG_CASE(12) NDG_CASE(13) NDG_CASE(14) NDG_CASE(15) NDG_CASE(16)
#undef NDG_CASE
        }
        NDG_CHECK_LAUNCH();
        return NDG_OK;
    }
    const size_t smem = sizeof(double) * kEpiWarps * epi_doubles(n);
    static DeviceOnce attr;
    if (attr.first())
        cudaFuncSetAttribute(epilogue_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
    epilogue_kernel<<<(unsigned)((G + kEpiWarps - 1) / kEpiWarps), kEpiWarps * 32, smem, as_stream(stream)>>>(
        n, G, Gev, amp_mode, params, child, flags, eflags, chol64, accum, grad_params,
        Gev == 2 * G ? grad_child : nullptr, stats, status);
    NDG_CHECK_LAUNCH();
    return NDG_OK;
}

// ---------------------------------------------------------------------------------------------
// K9 Adam with per-block learning rates.
// ---------------------------------------------------------------------------------------------
__global__ void adam_kernel(int n, int64_t rows, float* __restrict__ p, const float* __restrict__ g,
                            float* __restrict__ m1, float* __restrict__ m2, const uint8_t* __restrict__ row_mask,
                            const uint8_t* __restrict__ flags, uint32_t require, uint32_t forbid,
                            float c1, float c2, float lr_mean, float lr_chol, float lr_color, float lr_amp, float b1,
                            float b2, float eps) {
    const int R = raw_floats(n), P = n_chol(n);
    const int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (x >= rows * R) return;
    const int64_t row = x / R;
    const int col = (int)(x - row * R);
    if (row_mask && !row_mask[row]) return;
    if (flags && ((flags[row] & require) != require || (flags[row] & forbid))) return;
    const float lr = col < n ? lr_mean : (col < n + P ? lr_chol : (col < n + P + 3 ? lr_color : lr_amp));
    const float gv = g[x];
    const float a = __fadd_rn(__fmul_rn(b1, m1[x]), __fmul_rn(1.f - b1, gv));
    const float b = __fadd_rn(__fmul_rn(b2, m2[x]), __fmul_rn(__fmul_rn(1.f - b2, gv), gv));
    m1[x] = a;
    m2[x] = b;
    p[x] = __fsub_rn(p[x], __fdiv_rn(__fmul_rn(lr, __fdiv_rn(a, c1)), __fadd_rn(__fsqrt_rn(__fdiv_rn(b, c2)), eps)));
}

namespace {
int adam_launch(int n, int64_t rows, float* params, const float* grad, float* m1, float* m2, const uint8_t* row_mask,
                const uint8_t* flags, uint32_t require, uint32_t forbid, int step, float lr_mean, float lr_chol,
                float lr_color, float lr_amp, float beta1, float beta2, float eps, void* stream) {
    if (!ndg_supported_dims(n)) return NDG_ERR_UNSUPPORTED_DIMS;
    NDG_REQUIRE(step >= 1, "adam step counter starts at 1");
    const int64_t total = rows * raw_floats(n);
    if (total == 0) return NDG_OK;
    const float c1 = (float)(1.0 - pow((double)beta1, step));
    const float c2 = (float)(1.0 - pow((double)beta2, step));
    int threads = 256;
    adam_kernel<<<(unsigned)((total + threads - 1) / threads), threads, 0, as_stream(stream)>>>(
        n, rows, params, grad, m1, m2, row_mask, flags, require, forbid, c1, c2, lr_mean, lr_chol, lr_color, lr_amp,
        beta1, beta2, eps);
    NDG_CHECK_LAUNCH();
    return NDG_OK;
}
}  // namespace

extern "C" int ndg_adam(int n, int64_t rows, float* params, const float* grad, float* m1, float* m2,
                        const uint8_t* row_mask, int step, float lr_mean, float lr_chol, float lr_color, float lr_amp,
                        float beta1, float beta2, float eps, void* stream) {
    return adam_launch(n, rows, params, grad, m1, m2, row_mask, nullptr, 0, 0, step, lr_mean, lr_chol, lr_color,
                       lr_amp, beta1, beta2, eps, stream);
}

// The same update with the row selection read straight from the mixture's flags (no mask tensor to build per
// step): row r is updated iff (flags[r] & require) == require and (flags[r] & forbid) == 0.
extern "C" int ndg_adam_flags(int n, int64_t rows, float* params, const float* grad, float* m1, float* m2,
                              const uint8_t* flags, int require, int forbid, int step, float lr_mean, float lr_chol,
                              float lr_color, float lr_amp, float beta1, float beta2, float eps, void* stream) {
    NDG_REQUIRE(flags != nullptr && require >= 0 && require <= 255 && forbid >= 0 && forbid <= 255,
                "flags pointer and 8-bit require / forbid masks");
    return adam_launch(n, rows, params, grad, m1, m2, nullptr, flags, (uint32_t)require, (uint32_t)forbid, step,
                       lr_mean, lr_chol, lr_color, lr_amp, beta1, beta2, eps, stream);
}
