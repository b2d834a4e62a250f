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

// ------------------------------------------------------------------------------------------------
// gradcheck support (cmd_gradcheck): the rel-L2 loss of M raw-parameter variants in
// float64, culling off. CTA = variant: its threads activate the variant's evaluated Gaussians exactly
// as K1 does (diagonal exp, off-diagonal 2 sigmoid - 1, child composition m_c = L m_u + m_p, L U,
// alpha * sigmoid(colour)) into shared memory, then sweep the queries (forward substitution in
// float64) and reduce sum_q,ch (p - t)^2 * inv_den[q, ch] / (3B). inv_den = 1 / (pbar^2 + eps) is the
// detached denominator held at the base prediction (oracle pin 4); with inv_den == NULL the kernel
// instead writes variant 0's prediction to pred_out (the base pass).
// ------------------------------------------------------------------------------------------------
__device__ __forceinline__ double gc_offdiag(double r) { return 2.0 / (1.0 + exp(-r)) - 1.0; }
__device__ __forceinline__ double gc_sigmoid(double r) { return 1.0 / (1.0 + exp(-r)); }

template <int N>
__global__ void loss_f64_kernel(int G, int amp_mode, const double* __restrict__ params, const double* __restrict__ child,
                                const uint8_t* __restrict__ flags, int64_t B, const float* __restrict__ queries,
                                const float* __restrict__ targets, const double* __restrict__ inv_den,
                                double* __restrict__ pred_out, double* __restrict__ loss_out) {
    constexpr int P = n_chol(N), R = raw_floats(N), W = P + N + 3;   // per evaluated Gaussian: L | m | a
    extern __shared__ double s_g[];                                     // [2G][W]
    __shared__ double s_red[256];
    const int m = blockIdx.x, tid = threadIdx.x;
    const double* pv = params + (int64_t)m * G * R;
    const double* cv = child + (int64_t)m * G * R;
    for (int e = tid; e < 2 * G; e += blockDim.x) {
        const bool is_child = e >= G;
        const int i = is_child ? e - G : e;
        const uint8_t f = flags[i];
        double* out = s_g + e * W;
        const bool live = !(f & 2) && (!is_child || (f & 1));
        double L[P], mu[N];
        for (int r = 0; r < N; ++r)
            for (int c = 0; c <= r; ++c) {
                const double raw = pv[i * R + N + tri(r, c)];
                L[tri(r, c)] = r == c ? exp(raw) : gc_offdiag(raw);
            }
        for (int r = 0; r < N; ++r) mu[r] = pv[i * R + r];
        const double* arow = pv + i * R;
        if (is_child) {
            double U[P], Lc[P], mc[N];
            const double* crow = cv + i * R;
            for (int r = 0; r < N; ++r)
                for (int c = 0; c <= r; ++c) {
                    const double raw = crow[N + tri(r, c)];
                    U[tri(r, c)] = r == c ? exp(raw) : gc_offdiag(raw);
                }
            for (int r = 0; r < N; ++r) {
                double acc = mu[r];
                for (int k = 0; k <= r; ++k) acc += L[tri(r, k)] * crow[k];
                mc[r] = acc;
            }
            for (int r = 0; r < N; ++r)
                for (int c = 0; c <= r; ++c) {
                    double acc = 0.0;
                    for (int k = c; k <= r; ++k) acc += L[tri(r, k)] * U[tri(k, c)];
                    Lc[tri(r, c)] = acc;
                }
            for (int t = 0; t < P; ++t) L[t] = Lc[t];
            for (int r = 0; r < N; ++r) mu[r] = mc[r];
            arow = crow;
        }
        const double ampr = arow[N + P + 3];
        const double alpha = amp_mode == NDG_BRIGHTNESS ? exp(ampr) : gc_sigmoid(ampr);
        for (int t = 0; t < P; ++t) out[t] = L[t];
        for (int r = 0; r < N; ++r) out[P + r] = mu[r];
        for (int ch = 0; ch < 3; ++ch) out[P + N + ch] = live ? alpha * gc_sigmoid(arow[N + P + ch]) : 0.0;
    }
    __syncthreads();
    double acc = 0.0;
    for (int64_t q = tid; q < B; q += blockDim.x) {
        double x[N], p[3] = {0.0, 0.0, 0.0};
        for (int d = 0; d < N; ++d) x[d] = (double)queries[q * N + d];
        for (int e = 0; e < 2 * G; ++e) {
            const double* ge = s_g + e * W;
            if (ge[P + N] == 0.0 && ge[P + N + 1] == 0.0 && ge[P + N + 2] == 0.0) continue;
            double z[N], s2 = 0.0;
            for (int r = 0; r < N; ++r) {
                double a = x[r] - ge[P + r];
                for (int k = 0; k < r; ++k) a -= ge[tri(r, k)] * z[k];
                z[r] = a / ge[tri(r, r)];
                s2 += z[r] * z[r];
            }
            const double g = exp(-0.5 * s2);
            for (int ch = 0; ch < 3; ++ch) p[ch] += g * ge[P + N + ch];
        }
        if (inv_den) {
            for (int ch = 0; ch < 3; ++ch) {
                const double d = p[ch] - (double)targets[q * 3 + ch];
                acc += d * d * inv_den[q * 3 + ch];
            }
        } else if (m == 0 && pred_out) {
            for (int ch = 0; ch < 3; ++ch) pred_out[q * 3 + ch] = p[ch];
        }
    }
    s_red[tid] = acc;
    __syncthreads();
    for (int o = blockDim.x / 2; o; o >>= 1) {
        if (tid < o) s_red[tid] += s_red[tid + o];
        __syncthreads();
    }
    if (tid == 0) loss_out[m] = s_red[0] / (3.0 * (double)B);
}

template <int N>
int launch_loss_f64(int G, int amp_mode, int M, const double* params, const double* child, const uint8_t* flags,
                    int64_t B, const float* q, const float* t, const double* inv_den, double* pred_out, double* loss,
                    cudaStream_t st) {
    constexpr int W = n_chol(N) + N + 3;
    const size_t smem = sizeof(double) * 2 * (size_t)G * W;
    NDG_REQUIRE(smem <= 160 * 1024, "too many components for the float64 gradcheck evaluator");
    static DeviceOnce attr;
    if (attr.first()) cudaFuncSetAttribute(loss_f64_kernel<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
    loss_f64_kernel<N><<<M, 256, smem, st>>>(G, amp_mode, params, child, flags, B, q, t, inv_den, pred_out, loss);
    NDG_CHECK_LAUNCH();
    return NDG_OK;
}

// ---------------------------------------------------------------------------------------------
// Float64 finite differences of the loss, one coordinate per CTA (finite_diff_grad),
// evaluated so that rounding does not swamp small coordinates: a perturbation of raw row r changes only
// the evaluated Gaussians that read r (the parent and its live child for a parent row, the child for a
// child row), so with p_s = pbar + delta_s, delta_s = c_s - c_0 (their contributions at step s minus at
// the base) and d = pbar - t, every stencil sum sum_s w_s (p_s - t)^2 with sum_s w_s = 0 equals
// sum_s w_s (2 d delta_s + delta_s^2): the O(1) terms cancel exactly instead of in floating point.
// Stencil: central, 4 points (-2h, -h, h, 2h; weights 1, -8, 8, -1 over 12h) or 2 points (-h, h).
// The denominator is held at the base prediction, as in ndg_loss_f64.
// ---------------------------------------------------------------------------------------------
template <int N>
__device__ void fd_activate(int amp_mode, const double* prow, const double* crow, bool is_child, double* out) {
    constexpr int P = n_chol(N);
    double L[P], mu[N];
    for (int r = 0; r < N; ++r)
        for (int c = 0; c <= r; ++c) {
            const double raw = prow[N + tri(r, c)];
            L[tri(r, c)] = r == c ? exp(raw) : gc_offdiag(raw);
        }
    for (int r = 0; r < N; ++r) mu[r] = prow[r];
    const double* arow = prow;
    if (is_child) {
        double U[P], Lc[P], mc[N];
        for (int r = 0; r < N; ++r)
            for (int c = 0; c <= r; ++c) {
                const double raw = crow[N + tri(r, c)];
                U[tri(r, c)] = r == c ? exp(raw) : gc_offdiag(raw);
            }
        for (int r = 0; r < N; ++r) {
            double acc = mu[r];
            for (int k = 0; k <= r; ++k) acc += L[tri(r, k)] * crow[k];
            mc[r] = acc;
        }
        for (int r = 0; r < N; ++r)
            for (int c = 0; c <= r; ++c) {
                double acc = 0.0;
                for (int k = c; k <= r; ++k) acc += L[tri(r, k)] * U[tri(k, c)];
                Lc[tri(r, c)] = acc;
            }
        for (int t = 0; t < P; ++t) L[t] = Lc[t];
        for (int r = 0; r < N; ++r) mu[r] = mc[r];
        arow = crow;
    }
    const double ampr = arow[N + P + 3];
    const double alpha = amp_mode == NDG_BRIGHTNESS ? exp(ampr) : gc_sigmoid(ampr);
    for (int t = 0; t < P; ++t) out[t] = L[t];
    for (int r = 0; r < N; ++r) out[P + r] = mu[r];
    for (int ch = 0; ch < 3; ++ch) out[P + N + ch] = alpha * gc_sigmoid(arow[N + P + ch]);
}

template <int N>
__global__ void __launch_bounds__(256) fd_f64_kernel(int G, int amp_mode, const double* __restrict__ params,
                                                     const double* __restrict__ child, const uint8_t* __restrict__ flags,
                                                     int64_t B, const float* __restrict__ queries,
                                                     const float* __restrict__ targets, const double* __restrict__ pbar,
                                                     const double* __restrict__ inv_den, const int* __restrict__ coords,
                                                     double h, int points, double* __restrict__ fd_out) {
    constexpr int P = n_chol(N), R = raw_floats(N), W = P + N + 3;
    constexpr int MAXS = 5;                       // base + up to 4 stencil points
    __shared__ double s_g[MAXS][2][W];            // [step][parent | child][L | m | a]
    __shared__ double s_red[256];
    __shared__ int s_live[2];
    const int tid = threadIdx.x;
    const int row = coords[2 * blockIdx.x], col = coords[2 * blockIdx.x + 1];
    const bool crow_pert = row >= G;
    const int i = crow_pert ? row - G : row;
    const int nst = points == 4 ? 5 : 3;
    const double off4[5] = {0.0, -2.0, -1.0, 1.0, 2.0}, off2[3] = {0.0, -1.0, 1.0};
    if (tid == 0) {
        s_live[0] = !crow_pert && !(flags[i] & 2);
        s_live[1] = (flags[i] & 1) && !(flags[i] & 2);
    }
    if (tid < 2 * nst) {
        const int st = tid >> 1, which = tid & 1;   // which: 0 parent Gaussian, 1 child Gaussian
        double prow[R], crow[R];
        for (int t = 0; t < R; ++t) {
            prow[t] = params[i * R + t];
            crow[t] = child[i * R + t];
        }
        const double d = (points == 4 ? off4[st] : off2[st]) * h;
        if (crow_pert) crow[col] += d;
        else prow[col] += d;
        fd_activate<N>(amp_mode, prow, crow, which == 1, s_g[st][which]);
    }
    __syncthreads();
    const double w4[5] = {0.0, 1.0, -8.0, 8.0, -1.0}, w2[3] = {0.0, -1.0, 1.0};
    double acc = 0.0;
    for (int64_t q = tid; q < B; q += blockDim.x) {
        double x[N], c[MAXS][3];
        for (int dd = 0; dd < N; ++dd) x[dd] = (double)queries[q * N + dd];
        for (int st = 0; st < nst; ++st) {
            c[st][0] = c[st][1] = c[st][2] = 0.0;
            for (int which = 0; which < 2; ++which) {
                if (!s_live[which]) continue;
                const double* ge = s_g[st][which];
                double z[N], s2 = 0.0;
                for (int r = 0; r < N; ++r) {
                    double a = x[r] - ge[P + r];
                    for (int k = 0; k < r; ++k) a -= ge[tri(r, k)] * z[k];
                    z[r] = a / ge[tri(r, r)];
                    s2 += z[r] * z[r];
                }
                const double g = exp(-0.5 * s2);
                for (int ch = 0; ch < 3; ++ch) c[st][ch] += g * ge[P + N + ch];
            }
        }
        for (int ch = 0; ch < 3; ++ch) {
            const double d0 = pbar[q * 3 + ch] - (double)targets[q * 3 + ch];
            double sum = 0.0;
            for (int st = 1; st < nst; ++st) {
                const double del = c[st][ch] - c[0][ch];
                sum += (points == 4 ? w4[st] : w2[st]) * (2.0 * d0 * del + del * del);
            }
            acc += sum * inv_den[q * 3 + ch];
        }
    }
    s_red[tid] = acc;
    __syncthreads();
    for (int o = blockDim.x / 2; o; o >>= 1) {
        if (tid < o) s_red[tid] += s_red[tid + o];
        __syncthreads();
    }
    if (tid == 0) fd_out[blockIdx.x] = s_red[0] / (3.0 * (double)B) / ((points == 4 ? 12.0 : 2.0) * h);
}

// ---------------------------------------------------------------------------------------------
// NonFiniteGradientError.batch_index (errors.py:26-33): the lowest query index whose
// pair with evaluated Gaussian e (or e2, its child; -1 = none) -- on a tile where it is a candidate
// (cull mask bit) -- yields a non-finite backward term in K7's own float32 arithmetic (z~ from the
// evaluation record, g, w = g dpred . a, w s~, dpred, ell). Run only on the error path.
// ---------------------------------------------------------------------------------------------
template <int N>
__global__ void nonfinite_query_kernel(int64_t B, int tile, const float* __restrict__ qrec,
                                       const float* __restrict__ rec, const uint32_t* __restrict__ mask, int64_t W,
                                       int64_t e1, int64_t e2, unsigned long long* __restrict__ out) {
    constexpr int RS = rec_floats(N), QS = qrec_floats(N), A0 = rec_a(N);
    const int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (b >= B) return;
    const int64_t t = b / tile;
    const float* xq = qrec + b * QS;
    for (int which = 0; which < 2; ++which) {
        const int64_t e = which ? e2 : e1;
        if (e < 0 || !((mask[t * W + (e >> 5)] >> (e & 31)) & 1u)) continue;
        const float* r = rec + e * RS;
        float z[N], s = 0.f;
        for (int i = 0; i < N; ++i) {
            float acc = fmaf(r[rec_rho(N) + i], xq[i], r[rec_nb2(N) + 2 * i]);
            for (int k = 0; k < i; ++k) acc = fmaf(r[rec_l(N, i, k)], z[k], acc);
            z[i] = acc;
            s = fmaf(acc, acc, s);
        }
        const float g = exp2f(-s);
        const float w = g * (xq[N] * r[A0] + xq[N + 1] * r[A0 + 1] + xq[N + 2] * r[A0 + 2]);
        bool bad = !isfinite(s) || !isfinite(w) || !isfinite(w * s) || !isfinite(xq[N + 3]);
        for (int c = 0; c < 3; ++c) bad |= !isfinite(xq[N + c]);
        if (bad) atomicMin(out, (unsigned long long)b);
    }
}

// ---------------------------------------------------------------------------------------------
// Float64 backward pair loop (gradcheck's analytic side; not on the training path):
// thread per evaluated Gaussian over every query (culling off), same sufficient statistics and z~
// scaling as K7 (S' = sum w z~ z~^T, t' = sum w z~, gA, loss share, proxy, pairs with z~ = C z,
// g = 2^-|z~|^2, w = g dpred . a) but all in float64, written (not added) to accum[Gev][A] for the
// K8 epilogue. So the analytic gradient can be held to SPEC.md:572's per-coordinate bar.
// ---------------------------------------------------------------------------------------------
template <int N>
__global__ void backward_f64_kernel(int64_t G, int64_t Gev, int amp_mode, const float* __restrict__ params,
                                    const float* __restrict__ child, const double* __restrict__ mean64,
                                    const double* __restrict__ chol64, const uint8_t* __restrict__ eflags, int64_t B,
                                    const float* __restrict__ queries, const double* __restrict__ dpred,
                                    const double* __restrict__ ell, double* __restrict__ accum) {
    constexpr int P = n_chol(N), A = acc_doubles(N), T0 = acc_tail(N), R = raw_floats(N);
    const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (e >= Gev) return;
    double* acc = accum + e * A;
    for (int j = 0; j < A; ++j) acc[j] = 0.0;
    if ((eflags[e] & 3) != 1) return;
    const float* row = e < G ? params + e * R : child + (e - G) * R;
    const double ampr = (double)row[N + P + 3];
    const double alpha = amp_mode == NDG_BRIGHTNESS ? exp(ampr) : gc_sigmoid(ampr);
    double a[3], L[P], m[N];
    for (int ch = 0; ch < 3; ++ch) a[ch] = alpha * gc_sigmoid((double)row[N + P + ch]);
    for (int t = 0; t < P; ++t) L[t] = chol64[e * P + t];
    for (int r = 0; r < N; ++r) m[r] = mean64[e * N + r];
    for (int64_t q = 0; q < B; ++q) {
        double z[N], s = 0.0;
        for (int r = 0; r < N; ++r) {
            double v = (double)queries[q * N + r] - m[r];
            for (int k = 0; k < r; ++k) v -= L[tri(r, k)] * z[k];
            z[r] = v / L[tri(r, r)];
        }
        for (int r = 0; r < N; ++r) {
            z[r] *= kC;
            s += z[r] * z[r];
        }
        const double g = exp2(-s);
        const double* dp = dpred + q * 3;
        const double w = g * (dp[0] * a[0] + dp[1] * a[1] + dp[2] * a[2]);
        for (int i = 0; i < N; ++i) {
            for (int j = 0; j <= i; ++j) acc[tri(i, j)] += w * z[i] * z[j];
            acc[P + i] += w * z[i];
        }
        for (int ch = 0; ch < 3; ++ch) acc[T0 + ch] += g * dp[ch];
        if (ell) acc[T0 + 3] += g * ell[q];
        acc[T0 + 4] += fabs(w) * sqrt(s);
        acc[T0 + 5] += 1.0;
    }
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

extern "C" int ndg_loss_f64(int n, int G, int amp_mode, int M, const double* params, const double* child,
                            const uint8_t* flags, int64_t B, const float* queries, const float* targets,
                            const double* inv_den, double* pred_out, double* loss, void* stream) {
    NDG_REQUIRE(G >= 1 && M >= 1 && B >= 1, "need at least one component, variant and query");
    NDG_REQUIRE(inv_den || pred_out, "the base pass (inv_den == NULL) needs pred_out");
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    switch (n) {
#define NDG_CASE(NN) \
    case NN:         \
        return launch_loss_f64<NN>(G, amp_mode, M, params, child, flags, B, queries, targets, inv_den, pred_out, loss, st);
        NDG_CASE(1) NDG_CASE(2) NDG_CASE(3) NDG_CASE(4) NDG_CASE(5) NDG_CASE(6) NDG_CASE(7) NDG_CASE(8)
        NDG_CASE(9) NDG_CASE(10) NDG_CASE(11) NDG_CASE(12) NDG_CASE(13) NDG_CASE(14) NDG_CASE(15) NDG_CASE(16)
#undef NDG_CASE
        default:
            return NDG_ERR_UNSUPPORTED_DIMS;
    }
}

extern "C" int ndg_backward_f64(int n, int64_t G, int64_t Gev, int amp_mode, const float* params, const float* child,
                                const double* mean64, const double* chol64, const uint8_t* eflags, int64_t B,
                                const float* queries, const double* dpred, const double* ell, double* accum,
                                void* stream) {
    NDG_REQUIRE(Gev == G || Gev == 2 * G, "Gev must be G or 2G");
    if (Gev == 0) return NDG_OK;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    const unsigned grid = (unsigned)((Gev + 63) / 64);
    switch (n) {
#define NDG_CASE(NN)                                                                                            \
    case NN:                                                                                                    \
        backward_f64_kernel<NN><<<grid, 64, 0, st>>>(G, Gev, amp_mode, params, child, mean64, chol64, eflags, B, \
                                                     queries, dpred, ell, accum);                               \
        break;
        NDG_CASE(1) NDG_CASE(2) NDG_CASE(3) NDG_CASE(4) NDG_CASE(5) NDG_CASE(6) NDG_CASE(7) NDG_CASE(8)
        NDG_CASE(9) NDG_CASE(10) NDG_CASE(11) NDG_CASE(12) NDG_CASE(13) NDG_CASE(14) NDG_CASE(15) NDG_CASE(16)
#undef NDG_CASE
        default:
            return NDG_ERR_UNSUPPORTED_DIMS;
    }
    NDG_CHECK_LAUNCH();
    return NDG_OK;
}

extern "C" int ndg_fd_f64(int n, int G, int amp_mode, const double* params, const double* child, const uint8_t* flags,
                          int64_t B, const float* queries, const float* targets, const double* pred_base,
                          const double* inv_den, int M, const int* coords, double h, int points, double* fd,
                          void* stream) {
    NDG_REQUIRE(G >= 1 && B >= 1 && M >= 0 && h > 0.0 && (points == 2 || points == 4),
                "need components, queries, h > 0 and a 2- or 4-point stencil");
    if (M == 0) return NDG_OK;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    switch (n) {
#define NDG_CASE(NN)                                                                                             \
    case NN:                                                                                                     \
        fd_f64_kernel<NN><<<M, 256, 0, st>>>(G, amp_mode, params, child, flags, B, queries, targets, pred_base, \
                                             inv_den, coords, h, points, fd);                                   \
        break;
        NDG_CASE(1) NDG_CASE(2) NDG_CASE(3) NDG_CASE(4) NDG_CASE(5) NDG_CASE(6) NDG_CASE(7) NDG_CASE(8)
        NDG_CASE(9) NDG_CASE(10) NDG_CASE(11) NDG_CASE(12) NDG_CASE(13) NDG_CASE(14) NDG_CASE(15) NDG_CASE(16)
#undef NDG_CASE
        default:
            return NDG_ERR_UNSUPPORTED_DIMS;
    }
    NDG_CHECK_LAUNCH();
    return NDG_OK;
}

extern "C" int ndg_nonfinite_query(int n, int64_t B, int tile, const float* qrec, const float* rec, const uint32_t* mask,
                                   int64_t Gev, int64_t e1, int64_t e2, int64_t* out, void* stream) {
    NDG_REQUIRE(tile >= 1 && B % tile == 0, "batch must be a multiple of tile");
    if (B == 0) return NDG_OK;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    const int64_t W = (Gev + 31) / 32;
    const unsigned grid = (unsigned)((B + 255) / 256);
    auto* o = reinterpret_cast<unsigned long long*>(out);
    switch (n) {
#define NDG_CASE(NN)                                                                                     \
    case NN:                                                                                             \
        nonfinite_query_kernel<NN><<<grid, 256, 0, st>>>(B, tile, qrec, rec, mask, W, e1, e2, o);     \
        break;
        NDG_CASE(1) NDG_CASE(2) NDG_CASE(3) NDG_CASE(4) NDG_CASE(5) NDG_CASE(6) NDG_CASE(7) NDG_CASE(8)
        NDG_CASE(9) NDG_CASE(10) NDG_CASE(11) NDG_CASE(12) NDG_CASE(13) NDG_CASE(14) NDG_CASE(15) NDG_CASE(16)
#undef NDG_CASE
        default:
            return NDG_ERR_UNSUPPORTED_DIMS;
    }
    NDG_CHECK_LAUNCH();
    return NDG_OK;
}
