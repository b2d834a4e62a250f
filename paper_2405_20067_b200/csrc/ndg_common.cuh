// Shared definitions of the libndg.so kernels (sm_100a). See include/ndg.h for the ABI and
// DESIGN.md for the data layout in HBM and the roofline of each kernel.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/ndg.h"

namespace ndg {

constexpr int NMAX = 16;
#ifndef NDG_BWD_CHUNK
#define NDG_BWD_CHUNK 128
#endif
constexpr int kBwdChunk = NDG_BWD_CHUNK;  // candidates per backward work item (one per thread)
constexpr int kNumStats = 3;

__host__ __device__ constexpr int n_chol(int n) { return n * (n + 1) / 2; }
__host__ __device__ constexpr int n_strict(int n) { return n * (n - 1) / 2; }
__host__ __device__ constexpr int pad4(int x) { return (x + 3) & ~3; }
__host__ __device__ constexpr int tri(int i, int j) { return i * (i + 1) / 2 + j; }
__host__ __device__ constexpr int tri_s(int i, int j) { return i * (i - 1) / 2 + j; }    // strict lower
__host__ __device__ constexpr int64_t imin64(int64_t a, int64_t b) { return a < b ? a : b; }
__host__ __device__ constexpr int raw_floats(int n) { return n + n_chol(n) + 4; }

// Evaluation record (float32), one per evaluated Gaussian, 16-byte multiple so a record is one
// cp.async.bulk and a run of LDS.128 broadcasts. Laid out for packed FP32x2 (FFMA2) use:
//   nb2[2N]  = (nb_i, nb_i), nb_i = -C * m_i / L_ii   (duplicated: the addend operand of FFMA2 is a pair)
//   rho[N]   = C / L_ii                                (C = sqrt(0.5 * log2 e): folds the -1/2 and ln->log2)
//   nlu[..]  = -L_ij / L_ii, strict lower, row i padded to an even length so (j, j+1) pairs are
//              8-byte aligned (the backward's packed row dot products); the pad entries are 0
//   a[3]     = alpha * sigmoid(color)                  (premultiplied colour)
// so z~_i = fma(rho_i, x_i, nb_i) + sum_j nlu_ij z~_j equals C * z_i of L z = x - m
// and g = exp2(-|z~|^2) = exp(-|z|^2 / 2).
__host__ __device__ constexpr int pad2(int x) { return (x + 1) & ~1; }
__host__ __device__ constexpr int rec_nb2(int) { return 0; }
__host__ __device__ constexpr int rec_rho(int n) { return 2 * n; }
__host__ __device__ constexpr int rec_lu(int n) { return pad2(3 * n); }
__host__ __device__ constexpr int lu_row_start(int i) {   // sum_{r<i} 2*ceil(r/2)
    int s = 0;
    for (int r = 0; r < i; ++r) s += 2 * ((r + 1) / 2);
    return s;
}
__host__ __device__ constexpr int lu_floats(int n) { return lu_row_start(n); }
__host__ __device__ constexpr int rec_l(int n, int i, int j) { return rec_lu(n) + lu_row_start(i) + j; }
__host__ __device__ constexpr int rec_a(int n) { return rec_lu(n) + lu_floats(n); }
__host__ __device__ constexpr int rec_floats(int n) { return pad4(rec_a(n) + 3); }

// Tensor-core (tcgen05) record: N rows x tc_k(N) floats (Ahat_e, see ndg_forward_tc.cu); one MMA
// column block of 128 holds tc_chunk(N) Gaussians.
__host__ __device__ constexpr int tc_k(int n) { return ((n + 1 + 7) / 8) * 8; }
__host__ __device__ constexpr int tc_chunk(int n) { return 128 / n < 32 ? 128 / n : 32; }   // <= one per producer lane
__host__ __device__ constexpr int tc_rec_floats(int n) { return n * tc_k(n) + 4; }   // rows | a[3] | pad

// Backward query record (float32): x[N] | dpred[3] | ell, produced by the fused forward+loss.
__host__ __device__ constexpr int qrec_floats(int n) { return pad4(n + 4); }

// Accumulators per evaluated Gaussian: S'[P] | t'[N] | flag | gA[3] | loss_share | proxy | pairs, in the
// scaled z~ units with coefficient +g*h (the epilogue applies -1/C^2, -1/C, 1/C). The backward adds
// into them as two int64 fixed-point words per slot (see "deterministic reduction" below);
// ndg_acc_dequant turns them into float64 in place for the K8 epilogue. `flag` is nonzero when a
// partial was non-finite or outside its bound (the epilogue then sees NaN -> NonFiniteGradientError).
__host__ __device__ constexpr int acc_flag(int n) { return n_chol(n) + n; }
__host__ __device__ constexpr int acc_tail(int n) { return n_chol(n) + n + 1; }
__host__ __device__ constexpr int acc_doubles(int n) { return acc_tail(n) + 3 + kNumStats; }

// Threads per CTA for a thread-per-item kernel: the largest power of two <= max_threads that still gives
// every SM two CTAs, at least 32 -- small configurations (cfg1: 4096 Gaussians) then spread over ~128
// SMs instead of running 128-thread CTAs on 32 of them.
__host__ __device__ constexpr int spread_threads(int64_t items, int max_threads) {
    int t = max_threads;
    while (t > 32 && (items + t - 1) / t < 2 * 148) t >>= 1;
    return t;
}

// Backward work items in band order (ndg_work_items): bands of kBand tiles run chunk-major.
constexpr int kBand = 512;

constexpr double kC = 0.84932180028801907;      // sqrt(0.5 * log2(e))

}  // namespace ndg

// ---------------------------------------------------------------------------------------------
// Deterministic cross-tile reduction of the backward.
//
// Every per-(tile, candidate) float32 partial v of accumulator slot j is added to TWO int64 words,
//   hi[j] += rint(x),  lo[j] += rint((x - rint(x)) * 2^40),   x = v * s_c,
// with s_c = 2^(62 - e_c) a power of two from an a-priori bound U_c = 2^e_c (rounded up) on the sum of
// |v| over every partial of the slot's class c. Integer addition is associative, so the two sums --
// and the float64 value hi / s_c + lo / (s_c 2^40) that ndg_acc_dequant makes of them -- are the same
// whatever order the tiles finish in: gradients and checkpoints are bitwise reproducible. The
// quantum is U_c * 2^-102, far below the float32 rounding of the per-tile partials themselves.
// Bounds per pair (exact arithmetic, x2 margin for float32 rounding; at most B pairs per Gaussian):
//   h-class (S', t', proxy): g z~_i z~_j <= max x 2^-x = 0.531, g |z~_i| and g sqrt(s~) <= 0.515, so
//             |term| <= 0.54 |h| with |h| = |dpred . a| <= H * Amax;
//   gA:       g |dpred_c| <= Dmax;     loss share: g ell <= Lmax;     pairs: exact integer counts.
// H, Dmax, Lmax (over the step's finite queries) and Amax (over live Gaussians) come from
// ndg_bwd_bounds as float bit patterns (uint32 atomicMax of non-negative floats); a non-finite query
// makes only the partials it enters non-finite, and those set their Gaussian's flag.
// ---------------------------------------------------------------------------------------------
namespace ndg {

struct FxScales {
    double h, g, l;
};

__device__ __forceinline__ double fx_scale_for(double U) {
    if (U == 0.0) return 1.0;                      // the class is identically zero
    if (!(U > 0.0) || isinf(U)) return __longlong_as_double(0x7ff8000000000000LL);   // NaN: flag everything
    int ex;
    frexp(U, &ex);                                 // U = m 2^ex, m in [0.5, 1): U <= 2^ex
    int s = 62 - ex;
    s = s > 960 ? 960 : (s < -960 ? -960 : s);
    return ldexp(1.0, s);
}

__device__ __forceinline__ FxScales fx_scales(const uint32_t* __restrict__ bnd, int64_t B) {
    const double H = __uint_as_float(bnd[0]), D = __uint_as_float(bnd[1]), Lm = __uint_as_float(bnd[2]),
                 Am = __uint_as_float(bnd[3]);
    const double nb = 2.0 * (double)B;
    return FxScales{fx_scale_for(nb * 0.54 * H * Am), fx_scale_for(nb * D), fx_scale_for(nb * Lm)};
}

constexpr double kFxLo = 1099511627776.0;          // 2^40: the lo word's extra resolution

__device__ __forceinline__ void fx_add(unsigned long long* hi, unsigned long long* lo, unsigned long long* flag,
                                       float v, double sc) {
    if (v == 0.f) return;
    const double x = (double)v * sc;
    if (!(fabs(x) < 4611686018427387904.0)) {      // non-finite, or past 2^62: never silently wrong
        atomicOr(flag, 1ull);
        return;
    }
    const double xh = rint(x);
    const long long qh = (long long)xh;
    if (qh) atomicAdd(hi, (unsigned long long)qh);
    const long long ql = __double2ll_rn((x - xh) * kFxLo);
    if (ql) atomicAdd(lo, (unsigned long long)ql);
}

}  // namespace ndg

// Kernel attributes (e.g. the dynamic shared-memory opt-in) are per device: a launcher sets them the
// first time it runs on each device of the process, thread-safely.
#include <atomic>
namespace ndg {
struct DeviceOnce {
    std::atomic<unsigned long long> mask{0};
    bool first() {
        int d = 0;
        cudaGetDevice(&d);
        const unsigned long long bit = 1ull << (d & 63);
        return !(mask.fetch_or(bit) & bit);
    }
};
}  // namespace ndg

// Bounds-checked build (make exp EXP="-DNDG_CHECKED" TAG=checked): device-side invariant checks on the
// indices the kernels derive (candidate indices against Gev, CSR positions against the tile's range,
// work items against the tile count, pre-filter cells and permutation slots); a failed check prints
// the kernel, the condition and the block, and traps. Compiled out of the default build.
#ifdef NDG_CHECKED
#include <cstdio>
#define NDG_DCHECK(cond)                                                                            \
    do {                                                                                            \
        if (!(cond)) {                                                                              \
            printf("NDG_CHECKED %s:%d: %s failed (block %d, thread %d)\n", __FILE__, __LINE__, #cond, \
                   (int)blockIdx.x, (int)threadIdx.x);                                              \
            __trap();                                                                               \
        }                                                                                           \
    } while (0)
#else
#define NDG_DCHECK(cond) \
    do {                 \
    } while (0)
#endif

// error string (per-thread) defined in ndg_prep.cu
extern "C" void ndg_set_last_error(const char* msg);

#define NDG_CHECK_LAUNCH()                                                  \
    do {                                                                    \
        cudaError_t e_ = cudaGetLastError();                                \
        if (e_ != cudaSuccess) {                                            \
            ndg_set_last_error(cudaGetErrorString(e_));                     \
            return NDG_ERR_CUDA;                                            \
        }                                                                   \
    } while (0)

#define NDG_REQUIRE(cond, msg)                                              \
    do {                                                                    \
        if (!(cond)) {                                                      \
            ndg_set_last_error(msg);                                        \
            return NDG_ERR_BAD_ARGUMENT;                                    \
        }                                                                   \
    } while (0)

// ---------------------------------------------------------------------------------------------
// PTX helpers: mbarrier + 1-D bulk copy (TMA engine), fast exp2 / sqrt.
// ---------------------------------------------------------------------------------------------
namespace ndg {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    // try_wait with a suspend-time hint: the waiting warp sleeps in hardware until the phase
    // completes (or the hint expires) instead of re-polling shared memory in a tight loop.
    uint32_t addr = smem_u32(bar);
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
#ifdef NDG_MBAR_NOHINT
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
#else
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n"
#endif
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(addr),
        "r"(parity), "r"(0x989680)
        : "memory");
}

// 1-D bulk copy global -> shared through the TMA engine, completing bytes on `bar`.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ float ex2_neg(float s) {   // 2^(-s), MUFU.EX2 (ftz)
    float r;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(-s));
    return r;
}

__device__ __forceinline__ float sqrt_approx(float s) {
    float r;
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(s));
    return r;
}

}  // namespace ndg
