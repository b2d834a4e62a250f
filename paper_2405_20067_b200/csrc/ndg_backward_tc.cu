// K7 backward on the 5th-gen tensor cores (tcgen05, kind::tf32, 3xTF32) + K7b moments -> z-space.
//
// Replaces the pair loop of `backward`. Per pair (query q, candidate e) the
// backward needs z~ = Ahat_e xhat_q (xhat = [x - 1/2; 1], Ahat as in K5), g = 2^-|z~|^2,
// w = g * (dpred_q . a_e), and the per-Gaussian sums over the tile's queries
//     S' = sum w z~ z~^T,  t' = sum w z~,  gA = sum g dpred,  loss share = sum g ell,
//     proxy = sum |w| |z~|.
// Both big contractions run on the tensor cores:
//   z-GEMM      D1[q, (e,i)] = sum_k xhat_q[k] Ahat_e[i][k]          (exactly K5's GEMM)
//   moments     D2[f, e]     = sum_q phi_f(xhat_q) W[e, q]           (W = w, phi = xhat xhat^T packed)
// so S' = Ahat M Ahat^T and t' = Ahat M[:, N] with M = the (N+1)x(N+1) moment matrix (precision:
// tools/tc_precision_study.py "B1h", <= 1e-5 block-relative down to sigma 0.02). The per-pair FP32
// work left is |z~|^2, ex2, w, the hi/lo split of w and five scalar products (gA, loss share, proxy)
// reduced across the warp by a transpose-reduce (31 shuffles per 32 values).
//
// One CTA = one tile half (128 queries = MMA M of the z-GEMM = K of the moments GEMM), 16 warps:
//   0      TMA producer: one cp.async.bulk per candidate record into the staging ring
//   1      TMEM allocator + MMA issuer (z-GEMM per chunk; moments GEMM per super-chunk)
//   2,3    splitters: staging -> hi/lo K-major B planes of the z-GEMM + colours
//   4..11  epilogue: warp (q4, gh) reads its lane quarter's z~ for half gh of the chunk's Gaussians,
//          writes w (hi/lo) into the K-major moments B operand, reduces the scalar sums
//   12..15 drain: read D2 (lane = feature) after each moments GEMM, float64 atomics into accum
// TMEM: D1 2 x 128 | D2 2 x NG | A1 (xhat hi/lo) 2K columns. Shared memory: Phi (A operand of the
// moments GEMM, hi/lo, written once per CTA), W (single buffer, hi/lo), z-GEMM B ring, staging ring.
#include "ndg_tc.cuh"

using namespace ndg;

namespace {

constexpr int kBtSplit = 2;
constexpr int kBtEpi0 = 2 + kBtSplit;     // first epilogue warp
constexpr int kBtDrain0 = kBtEpi0 + 8;    // first drain warp
constexpr int kBtWarps = kBtDrain0 + 4;
constexpr int kBtThreads = kBtWarps * 32;
constexpr int kBtStages = 2;              // z-GEMM B-operand ring
constexpr int kBtARing = 8;               // colour ring
constexpr int kPlaneB = 128 * 16;         // z-GEMM B plane: 128 rows x 16 B
constexpr int kQ = 128;                   // queries per CTA
constexpr int kQP = kQ / 4;               // K planes of the moments GEMM
constexpr int kD1S = 128;                 // TMEM column stride of a D1 buffer

template <int N>
struct BtCfg {
    static constexpr int K = tc_k(N), P = K / 4, KS = K / 8;
    static constexpr int CH = (64 / N < 16 ? 64 / N : 16);        // Gaussians per epilogue warp per chunk
    static constexpr int C = 2 * CH;                               // Gaussians per chunk (<= 32 producer lanes)
    static constexpr int HALF = ((CH * N + 15) / 16) * 16;         // D1 columns of one Gaussian half
    static constexpr int NCOL = 2 * HALF;                          // z-GEMM N
    static constexpr int U = (64 / C > 1 ? 64 / C : 1);            // chunks per super-chunk
    static constexpr int NG = ((U * C + 15) / 16) * 16;            // moments GEMM N
    static constexpr int F = (N + 1) * (N + 2) / 2;                // moment features (= acc_tail(N))
    static constexpr int FP = ((F + 7) / 8) * 8;
    static constexpr int LBO_F = FP * 16 + 16;                     // +16 B: conflict-free column writes
    static constexpr int LBO_W = NG * 16 + 16;
    static constexpr int RT = tc_rec_floats(N);
    static constexpr size_t kPhi = (size_t)kQP * LBO_F + 128 * 16; // + slack: the MMA reads 128 rows/plane
    static constexpr size_t kW = (size_t)kQP * LBO_W;
    static constexpr size_t kBring = (size_t)kBtStages * 2 * P * kPlaneB;
    static constexpr size_t kFixed = 2 * kPhi + 2 * kW + kBring + (size_t)kBtARing * C * 16;
    static constexpr size_t kSlot = (size_t)C * RT * 4;
    static constexpr size_t kBudget = 225 * 1024;
    static constexpr int STG = (kFixed + 4 * kSlot <= kBudget) ? 4 : (kFixed + 2 * kSlot <= kBudget ? 2 : 0);
    static constexpr int D2_0 = 2 * kD1S;
    static constexpr int A1_0 = D2_0 + 2 * NG;
    static constexpr bool kOk = STG >= 2 && F < 128 && A1_0 + 2 * K <= 512 && NCOL <= kD1S;
};

template <int N>
constexpr size_t bt_smem_bytes() {
    using C_ = BtCfg<N>;
    return C_::kFixed + (size_t)C_::STG * C_::kSlot;
}

// Sum over the warp of v[lane]: halve the live set at each of the 5 shuffle steps.
__device__ __forceinline__ float transpose_reduce32(float (&v)[32], int lane) {
#pragma unroll
    for (int w = 16; w >= 1; w >>= 1) {
        const bool up = lane & w;
#pragma unroll
        for (int k = 0; k < w; ++k) {
            const float send = up ? v[k] : v[k + w];
            const float keep = up ? v[k + w] : v[k];
            v[k] = keep + __shfl_xor_sync(0xffffffffu, send, w);
        }
    }
    return v[0];
}

template <int N>
__global__ void __launch_bounds__(kBtThreads, 1)
    backward_tc_kernel(int tile, int halves, const float* __restrict__ qrec, const float* __restrict__ rec_tc,
                       const int64_t* __restrict__ offsets, const int32_t* __restrict__ idx,
                       double* __restrict__ accum) {
    using Cfg = BtCfg<N>;
    constexpr int K = Cfg::K, P = Cfg::P, KS = Cfg::KS, CH = Cfg::CH, C = Cfg::C, HALF = Cfg::HALF;
    constexpr int U = Cfg::U, NG = Cfg::NG, F = Cfg::F, LBO_F = Cfg::LBO_F, LBO_W = Cfg::LBO_W;
    constexpr int RT = Cfg::RT, STG = Cfg::STG, QS = qrec_floats(N), A = acc_doubles(N), TAIL = acc_tail(N);
    constexpr uint32_t IDESC1 = tc::idesc_tf32(128, Cfg::NCOL);
    constexpr uint32_t IDESC2 = tc::idesc_tf32(128, NG);

    extern __shared__ __align__(1024) uint8_t smem[];
    uint8_t* sPhi = smem;                                   // [hi,lo][kPhi]
    uint8_t* sW = sPhi + 2 * Cfg::kPhi;                     // [hi,lo][kW]
    uint8_t* sB = sW + 2 * Cfg::kW;                         // [stages][hi,lo][P][kPlaneB]
    float* sAval = reinterpret_cast<float*>(sB + Cfg::kBring);   // [kBtARing][C][4]
    float* sStage = sAval + kBtARing * C * 4;               // [STG][C][RT]
    __shared__ __align__(8) uint64_t sfull[STG], sempty[STG], full_bar[kBtStages], empty_bar[kBtStages];
    __shared__ __align__(8) uint64_t aempty_bar[kBtARing], tfull_bar[2], tempty_bar[2];
    __shared__ __align__(8) uint64_t wfull_bar, wempty_bar, d2full_bar[2], d2empty_bar[2];
    __shared__ uint32_t s_tbase;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t t = blockIdx.x / halves;
    const int q0 = (int)(blockIdx.x % halves) * kQ;
    const int nq = min(kQ, tile - q0);
    const int64_t beg = offsets[t], end = offsets[t + 1];
    const int64_t cnt = end - beg;
    if (cnt == 0) return;
    const int nchunks = (int)((cnt + C - 1) / C);
    const int nsuper = (nchunks + U - 1) / U;

    if (tid == 0) {
        for (int s = 0; s < STG; ++s) {
            mbar_init(&sfull[s], 1);
            mbar_init(&sempty[s], kBtSplit);
        }
        for (int s = 0; s < kBtStages; ++s) {
            mbar_init(&full_bar[s], kBtSplit);
            mbar_init(&empty_bar[s], 1);
        }
        for (int s = 0; s < kBtARing; ++s) mbar_init(&aempty_bar[s], 8);
        for (int b = 0; b < 2; ++b) {
            mbar_init(&tfull_bar[b], 1);
            mbar_init(&tempty_bar[b], 8);
            mbar_init(&d2full_bar[b], 1);
            mbar_init(&d2empty_bar[b], 4);
        }
        mbar_init(&wfull_bar, 8);
        mbar_init(&wempty_bar, 1);
        fence_mbar_init();
    }
    if (warp == 1) tc::alloc(&s_tbase, 512);
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t tbase = s_tbase;

    // per-query state of the epilogue threads (both Gaussian halves of a lane quarter hold it)
    const int q4 = warp & 3, gh = (warp - kBtEpi0) >> 2;
    const int r = q4 * 32 + lane;                            // query row within the CTA (= TMEM lane)
    float dp0 = 0.f, dp1 = 0.f, dp2 = 0.f, ell = 0.f;
    if (warp >= kBtEpi0 && warp < kBtDrain0) {
        float xh[N + 1];
#pragma unroll
        for (int d = 0; d <= N; ++d) xh[d] = 0.f;
        if (r < nq) {
            const float* qr = qrec + ((int64_t)t * tile + q0 + r) * QS;
#pragma unroll
            for (int d = 0; d < N; ++d) xh[d] = qr[d] - 0.5f;
            xh[N] = 1.f;
            dp0 = qr[N];
            dp1 = qr[N + 1];
            dp2 = qr[N + 2];
            ell = qr[N + 3];
        }
        if (gh == 0) {   // A operand of the z-GEMM: xhat hi / lo at TMEM columns A1_0 + [0, K) / [K, 2K)
            float hi[K], lo[K];
#pragma unroll
            for (int k = 0; k < K; ++k) hi[k] = lo[k] = 0.f;
#pragma unroll
            for (int d = 0; d <= N; ++d) tc::split_tf32(xh[d], hi[d], lo[d]);
            const uint32_t ta = tbase + ((uint32_t)(q4 * 32) << 16) + (uint32_t)Cfg::A1_0;
#pragma unroll
            for (int k0 = 0; k0 < K; k0 += 8) {
                tc::st8(ta + k0, hi + k0);
                tc::st8(ta + K + k0, lo + k0);
            }
            tc::wait_st();
        }
        // A operand of the moments GEMM: phi_f(xhat_r) for f = tri(i, j), j <= i <= N, column r
        constexpr int FH = (F + 1) / 2;
        uint8_t* col = sPhi + (r >> 2) * LBO_F + (r & 3) * 4;
#pragma unroll
        for (int i = 0; i <= N; ++i)
#pragma unroll
            for (int j = 0; j <= i; ++j) {
                const int f = i * (i + 1) / 2 + j;
                if ((f < FH) == (gh == 0)) {
                    float h, l;
                    tc::split_tf32(xh[i] * xh[j], h, l);
                    *reinterpret_cast<float*>(col + f * 16) = h;
                    *reinterpret_cast<float*>(col + Cfg::kPhi + f * 16) = l;
                }
            }
        fence_proxy_async();
    }
    tc::fence_before();
    __syncthreads();
    tc::fence_after();

    if (warp == 0) {
        // ------------------------------ TMA producer -------------------------------------------
        auto load_idx = [&](int c) -> int64_t {
            const int64_t pos = beg + (int64_t)c * C + lane;
            return (lane < C && c < nchunks && pos < end) ? (int64_t)__ldg(idx + pos) : 0;
        };
        int64_t e0 = load_idx(0), e1 = load_idx(1);
        for (int c = 0; c < nchunks; ++c) {
            const int64_t e2 = load_idx(c + 2);
            const int sl = c % STG;
            if (c >= STG) mbar_wait(&sempty[sl], (uint32_t)((c / STG) - 1) & 1);
            const int n_in = (int)imin64(C, end - beg - (int64_t)c * C);
            if (lane == 0) mbar_arrive_expect_tx(&sfull[sl], (uint32_t)(n_in * RT * 4));
            __syncwarp();
            if (lane < n_in) bulk_g2s(sStage + (sl * C + lane) * RT, rec_tc + e0 * RT, RT * 4, &sfull[sl]);
            e0 = e1;
            e1 = e2;
        }
    } else if (warp == 1) {
        // ------------------------------ MMA issuer ---------------------------------------------
        if (lane == 0) {
            const uint32_t b_base = smem_u32(sB), phi = smem_u32(sPhi), wb = smem_u32(sW);
            const uint32_t a1hi = tbase + (uint32_t)Cfg::A1_0, a1lo = a1hi + K;
            auto moments = [&](int S) {
                const int b2 = S & 1;
                if (S >= 2) mbar_wait(&d2empty_bar[b2], (uint32_t)((S >> 1) - 1) & 1);
                mbar_wait(&wfull_bar, (uint32_t)S & 1);
                tc::fence_after();
                const uint32_t d = tbase + (uint32_t)(Cfg::D2_0 + b2 * NG);
#pragma unroll 1
                for (int ks = 0; ks < kQ / 8; ++ks) {
                    const uint64_t ahi = tc::smem_desc(phi + 2 * ks * LBO_F, LBO_F);
                    const uint64_t alo = tc::smem_desc(phi + (uint32_t)Cfg::kPhi + 2 * ks * LBO_F, LBO_F);
                    const uint64_t bhi = tc::smem_desc(wb + 2 * ks * LBO_W, LBO_W);
                    const uint64_t blo = tc::smem_desc(wb + (uint32_t)Cfg::kW + 2 * ks * LBO_W, LBO_W);
                    tc::mma_tf32(d, ahi, bhi, IDESC2, ks > 0 ? 1u : 0u);
                    tc::mma_tf32(d, ahi, blo, IDESC2, 1u);
                    tc::mma_tf32(d, alo, bhi, IDESC2, 1u);
                }
                tc::commit(&wempty_bar);          // W may be rewritten
                tc::commit(&d2full_bar[b2]);      // moments of super-chunk S are in D2 buffer b2
            };
            int pend = -1;
            for (int c = 0; c < nchunks; ++c) {
                const int s = c % kBtStages, b = c & 1;
                mbar_wait(&full_bar[s], (uint32_t)(c / kBtStages) & 1);
                if (c >= 2) mbar_wait(&tempty_bar[b], (uint32_t)((c >> 1) - 1) & 1);
                tc::fence_after();
                const uint32_t d = tbase + (uint32_t)(b * kD1S);
#pragma unroll
                for (int ks = 0; ks < KS; ++ks) {
                    const uint64_t bhi = tc::smem_desc(b_base + ((s * 2 + 0) * P + 2 * ks) * kPlaneB, kPlaneB);
                    const uint64_t blo = tc::smem_desc(b_base + ((s * 2 + 1) * P + 2 * ks) * kPlaneB, kPlaneB);
                    tc::mma_tf32_ta(d, a1hi + 8 * ks, bhi, IDESC1, ks > 0 ? 1u : 0u);
                    tc::mma_tf32_ta(d, a1hi + 8 * ks, blo, IDESC1, 1u);
                    tc::mma_tf32_ta(d, a1lo + 8 * ks, bhi, IDESC1, 1u);
                }
                tc::commit(&empty_bar[s]);
                tc::commit(&tfull_bar[b]);
                // the previous super-chunk's moments go in right behind the next z-GEMM, so the tensor
                // pipe has work while the epilogue finishes writing W
                if (pend >= 0) {
                    moments(pend);
                    pend = -1;
                }
                if (c % U == U - 1 || c == nchunks - 1) pend = c / U;
            }
            if (pend >= 0) moments(pend);
        }
        __syncwarp();
    } else if (warp < kBtEpi0) {
        // ------------------------------ splitters ----------------------------------------------
        constexpr int NSL = kBtSplit * 32;
        const int pl = (warp - 2) * 32 + lane;
        for (int c = 0; c < nchunks; ++c) {
            const int sl = c % STG, s = c % kBtStages, as = c % kBtARing;
            const int n_in = (int)imin64(C, end - beg - (int64_t)c * C);
            mbar_wait(&sfull[sl], (uint32_t)(c / STG) & 1);
            if (c >= kBtStages) mbar_wait(&empty_bar[s], (uint32_t)((c / kBtStages) - 1) & 1);
            if (c >= kBtARing) mbar_wait(&aempty_bar[as], (uint32_t)((c / kBtARing) - 1) & 1);
            const float* stg = sStage + sl * C * RT;
            uint8_t* bhi = sB + (s * 2 + 0) * P * kPlaneB;
            uint8_t* blo = sB + (s * 2 + 1) * P * kPlaneB;
#pragma unroll 2
            for (int u = pl; u < n_in * N * P; u += NSL) {       // unit = (gaussian g, plane p, row i)
                const int g = u / (N * P), rem = u - g * (N * P);
                const int p = rem / N, i = rem - p * N;
                const float4 v = *reinterpret_cast<const float4*>(stg + g * RT + rem * 4);
                float4 hi, lo;
                tc::split_tf32(v.x, hi.x, lo.x);
                tc::split_tf32(v.y, hi.y, lo.y);
                tc::split_tf32(v.z, hi.z, lo.z);
                tc::split_tf32(v.w, hi.w, lo.w);
                const int row = (g / CH) * HALF + (g % CH) * N + i;   // D1 column of (g, i)
                *reinterpret_cast<float4*>(bhi + p * kPlaneB + row * 16) = hi;
                *reinterpret_cast<float4*>(blo + p * kPlaneB + row * 16) = lo;
            }
            for (int u = pl; u < n_in; u += NSL)
                *reinterpret_cast<float4*>(sAval + (as * C + u) * 4) =
                    *reinterpret_cast<const float4*>(stg + u * RT + N * K);
            fence_proxy_async();
            __syncwarp();
            if (lane == 0) {
                mbar_arrive(&full_bar[s]);
                mbar_arrive(&sempty[sl]);
            }
        }
    } else if (warp < kBtDrain0) {
        // ------------------------------ epilogue -----------------------------------------------
        uint8_t* wcol = sW + (r >> 2) * LBO_W + (r & 3) * 4;
        for (int c = 0; c < nchunks; ++c) {
            const int as = c % kBtARing, b = c & 1, S = c / U, u = c - S * U;
            const int n_in = (int)imin64(C, end - beg - (int64_t)c * C);
            mbar_wait(&tfull_bar[b], (uint32_t)(c >> 1) & 1);
            tc::fence_after();
            float v[HALF];
            const uint32_t ta = tbase + ((uint32_t)(q4 * 32) << 16) + (uint32_t)(b * kD1S + gh * HALF);
#pragma unroll
            for (int j = 0; j < HALF / 16; ++j) tc::ld16(ta + 16 * j, v + 16 * j);
            tc::wait_ld();
            tc::fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&tempty_bar[b]);
            float wv[CH], gv[CH], pv[CH];
#pragma unroll
            for (int jj = 0; jj < CH; ++jj) {
                const int g = gh * CH + jj;
                float s;
                if constexpr ((N & 1) == 0) {
                    float2 acc = make_float2(0.f, 0.f);
#pragma unroll
                    for (int i = 0; i < N; i += 2) {
                        const float2 zz = make_float2(v[jj * N + i], v[jj * N + i + 1]);
                        acc = __ffma2_rn(zz, zz, acc);
                    }
                    s = acc.x + acc.y;
                } else {
                    s = 0.f;
#pragma unroll
                    for (int i = 0; i < N; ++i) s = fmaf(v[jj * N + i], v[jj * N + i], s);
                }
                const float ge = (g < n_in) ? ex2_neg(s) : 0.f;
                const float4 av = *reinterpret_cast<const float4*>(sAval + (as * C + (g < n_in ? g : 0)) * 4);
                const float w = ge * fmaf(dp2, av.z, fmaf(dp1, av.y, dp0 * av.x));
                wv[jj] = w;
                gv[jj] = ge;
                pv[jj] = (g < n_in) ? fabsf(w) * sqrt_approx(s) : 0.f;
            }
            // W rows u*C + g, column r (single buffer: wait until the previous moments GEMM has read it)
            if (u == 0 && S >= 1) mbar_wait(&wempty_bar, (uint32_t)(S - 1) & 1);
#pragma unroll
            for (int jj = 0; jj < CH; ++jj) {
                float h, l;
                tc::split_tf32(wv[jj], h, l);
                const int row = u * C + gh * CH + jj;
                *reinterpret_cast<float*>(wcol + row * 16) = h;
                *reinterpret_cast<float*>(wcol + Cfg::kW + row * 16) = l;
            }
            fence_proxy_async();
            // scalar sums over the warp's 32 queries: slots (jj, k) = 5 jj + k, 6 Gaussians per pass
#pragma unroll
            for (int g0 = 0; g0 < CH; g0 += 6) {
                float red[32];
#pragma unroll
                for (int k = 0; k < 32; ++k) {
                    const int jj = g0 + k / 5, comp = k % 5;
                    float x = 0.f;
                    if (k < 30 && jj < CH) {
                        x = comp == 0 ? gv[jj] * dp0 : comp == 1 ? gv[jj] * dp1 : comp == 2 ? gv[jj] * dp2
                          : comp == 3 ? gv[jj] * ell : pv[jj];
                    }
                    red[k] = x;
                }
                const float tot = transpose_reduce32(red, lane);
                const int jj = g0 + lane / 5, comp = lane % 5, g = gh * CH + jj;
                if (lane < 30 && jj < CH && g < n_in) {
                    const int64_t e = idx[beg + (int64_t)c * C + g];
                    atomicAdd(accum + e * A + TAIL + comp, (double)tot);
                }
            }
            __syncwarp();
            if (lane == 0) {
                mbar_arrive(&aempty_bar[as]);
                if (u == U - 1 || c == nchunks - 1) mbar_arrive(&wfull_bar);
            }
        }
    } else {
        // ------------------------------ drain --------------------------------------------------
        const int dq = warp - kBtDrain0, f = dq * 32 + lane;   // TMEM lane = moment feature
        for (int S = 0; S < nsuper; ++S) {
            const int b2 = S & 1;
            mbar_wait(&d2full_bar[b2], (uint32_t)(S >> 1) & 1);
            tc::fence_after();
            float v[NG];
            const uint32_t ta = tbase + ((uint32_t)(dq * 32) << 16) + (uint32_t)(Cfg::D2_0 + b2 * NG);
#pragma unroll
            for (int j = 0; j < NG / 16; ++j) tc::ld16(ta + 16 * j, v + 16 * j);
            tc::wait_ld();
            tc::fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&d2empty_bar[b2]);
            const int64_t first = beg + (int64_t)S * U * C;
            const int count = (int)imin64(U * C, end - first);
            if (f <= F) {
#pragma unroll
                for (int uu = 0; uu < NG; ++uu) {
                    if (uu < count) {
                        const int64_t e = idx[first + uu];
                        if (f < F) atomicAdd(accum + e * A + f, (double)v[uu]);
                        else atomicAdd(accum + e * A + TAIL + 5, (double)nq);
                    }
                }
            }
        }
    }
    tc::fence_before();
    __syncthreads();
    if (warp == 1) {
        tc::fence_after();
        tc::dealloc(tbase, 512);
    }
}

template <int N>
int launch_backward_tc(int64_t B, int tile, const float* qrec, const float* rec_tc, const int64_t* off,
                       const int32_t* idx, double* accum, cudaStream_t st) {
    if constexpr (!BtCfg<N>::kOk) {
        return NDG_ERR_UNSUPPORTED_DIMS;
    } else {
        const int64_t T = B / tile;
        const int halves = (tile + kQ - 1) / kQ;
        const size_t smem = bt_smem_bytes<N>();
        static DeviceOnce attr;
        if (attr.first()) {
            cudaFuncSetAttribute(backward_tc_kernel<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        }
        NDG_REQUIRE(T * halves <= 0x7fffffffLL, "too many tiles");
        backward_tc_kernel<N><<<(unsigned)(T * halves), kBtThreads, smem, st>>>(tile, halves, qrec, rec_tc, off, idx,
                                                                               accum);
        NDG_CHECK_LAUNCH();
        return NDG_OK;
    }
}

// K7b: M (x-space moments, float64) -> S' = Ahat M Ahat^T, t' = Ahat M[:, N] in place, per evaluated
// Gaussian, with Ahat = C [L^-1 | L^-1 (1/2 - m)] recomputed in float64 from K1's factor.
template <int N>
__global__ void moments_to_zspace_kernel(int64_t Gev, const double* __restrict__ mean64,
                                         const double* __restrict__ chol64, const uint8_t* __restrict__ eflags,
                                         double* __restrict__ accum) {
    const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (e >= Gev || !(eflags[e] & 1)) return;
    constexpr int P = n_chol(N), F = (N + 1) * (N + 2) / 2;
    double* acc = accum + e * acc_doubles(N);
    double L[P], W[P], Ah[N][N + 1], M[F];
    for (int k = 0; k < P; ++k) L[k] = chol64[e * P + k];
    for (int k = 0; k < F; ++k) M[k] = acc[k];
    for (int j = 0; j < N; ++j)
        for (int i = j; i < N; ++i) {
            double a = (i == j) ? 1.0 : 0.0;
            for (int k = j; k < i; ++k) a -= L[tri(i, k)] * W[tri(k, j)];
            W[tri(i, j)] = a / L[tri(i, i)];
        }
    for (int i = 0; i < N; ++i) {
        double bias = 0.0;
        for (int j = 0; j < N; ++j) {
            const double w = j <= i ? kC * W[tri(i, j)] : 0.0;
            Ah[i][j] = w;
            bias += w * (0.5 - mean64[e * N + j]);
        }
        Ah[i][N] = bias;
    }
    auto m = [&](int a, int b) -> double { return a >= b ? M[tri(a, b)] : M[tri(b, a)]; };
    for (int i = 0; i < N; ++i) {
        double T[N + 1];
        for (int b = 0; b <= N; ++b) {
            double s = 0.0;
            for (int a = 0; a <= N; ++a) s += Ah[i][a] * m(a, b);
            T[b] = s;
        }
        for (int j = 0; j <= i; ++j) {
            double s = 0.0;
            for (int b = 0; b <= N; ++b) s += T[b] * Ah[j][b];
            acc[tri(i, j)] = s;
        }
        acc[P + i] = T[N];
    }
    acc[P + N] = 0.0;
}

template <int N>
int launch_m2z(int64_t Gev, const double* mean64, const double* chol64, const uint8_t* eflags, double* accum,
               cudaStream_t st) {
    moments_to_zspace_kernel<N><<<(unsigned)((Gev + 127) / 128), 128, 0, st>>>(Gev, mean64, chol64, eflags, accum);
    NDG_CHECK_LAUNCH();
    return NDG_OK;
}

}  // namespace

extern "C" int ndg_backward_tc_supported(int n) {
    switch (n) {
#define NDG_CASE(NN) \
    case NN:         \
        return BtCfg<NN>::kOk ? 1 : 0;
        NDG_CASE(1) NDG_CASE(2) NDG_CASE(3) NDG_CASE(4) NDG_CASE(5) NDG_CASE(6) NDG_CASE(7) NDG_CASE(8)
        NDG_CASE(9) NDG_CASE(10) NDG_CASE(11) NDG_CASE(12) NDG_CASE(13) NDG_CASE(14) NDG_CASE(15) NDG_CASE(16)
#undef NDG_CASE
        default:
            return 0;
    }
}

extern "C" int ndg_backward_tc(int n, int64_t B, int tile, const float* qrec, const float* rec_tc,
                               const int64_t* offsets, const int32_t* idx, double* accum, void* stream) {
    NDG_REQUIRE(tile >= 1 && tile <= 1024 && B % tile == 0, "tensor-core backward needs tile in 1..1024 dividing B");
    if (B == 0) return NDG_OK;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    switch (n) {
#define NDG_CASE(NN) \
    case NN:         \
        return launch_backward_tc<NN>(B, tile, qrec, rec_tc, offsets, idx, accum, st);
        NDG_CASE(1) NDG_CASE(2) NDG_CASE(3) NDG_CASE(4) NDG_CASE(5) NDG_CASE(6) NDG_CASE(7) NDG_CASE(8)
        NDG_CASE(9) NDG_CASE(10) NDG_CASE(11) NDG_CASE(12) NDG_CASE(13) NDG_CASE(14) NDG_CASE(15) NDG_CASE(16)
#undef NDG_CASE
        default:
            return NDG_ERR_UNSUPPORTED_DIMS;
    }
}

extern "C" int ndg_moments_to_zspace(int n, int64_t Gev, const double* mean64, const double* chol64,
                                     const uint8_t* eflags, double* accum, void* stream) {
    if (Gev == 0) return NDG_OK;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    switch (n) {
#define NDG_CASE(NN) \
    case NN:         \
        return launch_m2z<NN>(Gev, mean64, chol64, eflags, accum, st);
        NDG_CASE(1) NDG_CASE(2) NDG_CASE(3) NDG_CASE(4) NDG_CASE(5) NDG_CASE(6) NDG_CASE(7) NDG_CASE(8)
        NDG_CASE(9) NDG_CASE(10) NDG_CASE(11) NDG_CASE(12) NDG_CASE(13) NDG_CASE(14) NDG_CASE(15) NDG_CASE(16)
#undef NDG_CASE
        default:
            return NDG_ERR_UNSUPPORTED_DIMS;
    }
}
