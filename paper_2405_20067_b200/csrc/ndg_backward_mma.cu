// K7-MMA: the fused backward for large N on warp-level tensor cores (sm_100a, mma.sync m16n8k16 f16
// operands split hi / lo, fp32 accumulation).
//
// Same contract as the FP32 K7 (ndg_backward.cu): per (tile, candidate) it adds
//   S' += (w z~) z~^T (lower),  t' += w z~,  gA += g dpred,  loss_share += g ell,  proxy += |w| sqrt(s~)
// to the fixed-point accumulators (deterministic, ndg_common.cuh), with w = g h, h = dpred . a,
// g = 2^-s~, s~ = |z~|^2, in the scaled z~ units of the FP32 K7, so the K8 epilogue is shared.
//
// Why a second kernel: the FP32 K7 keeps one Gaussian per thread with its record (P + 2N + 3 floats)
// AND its accumulators (P + N + 5) in registers. Past N = 12 that no longer fits in 255 registers;
// at N = 16 the pair loop reloads ~100 spilled floats per query from local memory and the kernel
// runs at a third of the FP32 peak. Here a warp owns two Gaussians and a 16 x 8 (dims x queries)
// block of z~ is one MMA:
//   MMA1  Z^T (16 x 8)   = Ahat (16 x 16) . Xhat^T (16 x 8),  C initialised to the bias column
//   MMA2  S'  (16 x 16) += (s V)^T (16 dims x 16 queries) . V (16 queries x 8 dims) per column block,
//         V = sqrt|w| Z, s = sign w
// The C fragments of MMA1 for two 8-query n-tiles (lane (gid, tig): dims gid, gid+8 of queries 2tig,
// 2tig+1) ARE the A fragment (rows = dims, k = the 16 queries) and the B fragments MMA2 needs, so z~
// never leaves the registers. With V = V_h + V_l, S' = sum s V_h V_h^T + M + M^T (M = sum s V_h V_l^T)
// takes two MMAs per column block where the plain split product u z^T takes three (same products
// kept, same lo.lo dropped); M^T is formed once per (tile, Gaussian) in shared memory. The per-tile
// Xhat fragments (hi | lo, x - 1/2 as in K5) are built once per work item in shared memory and read
// as LDS.128.
//
// Ahat / bias / colour come from the K5 tensor-core record (rec_tc, ndg_tc_records): row i of Ahat is
// kC L^-1 (lower), column n the bias for xhat = x - 1/2, so z~ is the K5 z~ up to accumulation
// order. Its error grows like the z-GEMM's (RMS of B_e, engine.py guards it).
//
// Round 1 ran this on m16n8k8 tf32 (8.5 MMAs per Gaussian and 8 queries, 231 ms on the N = 16 A/B
// workload); m16n8k16 f16 issues at the same rate with twice the K (tools/mma_sync_probe.cu), which
// with the lane ownership below gives 10 MMAs per Gaussian and 16 queries and 176 ms, and a smaller
// error against the FP32 K7 (8.3e-7 vs 2.8e-6: the operand scaling keeps the splits exact).
#include <cuda_fp16.h>

#include "ndg_common.cuh"
#include "ndg_tc.cuh"

using namespace ndg;

namespace {

#ifndef NDG_MMA_MINB
#define NDG_MMA_MINB 4
#endif
constexpr int kThreads = 128;   // 4 warps; work item = (tile, chunk of kBwdChunk candidates)
constexpr int kGpw = 2;         // Gaussians per warp: the lanes own the two Gaussians' per-query scalars between them

// ---- mma.sync m16n8k16 f16 -> f32 --------------------------------------------------------------------
// All 16 input dims in ONE k-step, and 16 queries per S' update. Per Gaussian and 16 queries: MMA1
// 2 n-tiles x 3 products (hi.hi, hi.lo, lo.hi) = 6, MMA2 2 column blocks x 2 (v_h v_h, v_h v_l) = 4:
// 10 MMAs where the tf32 form issued 17.
// f16 has tf32's 11 significant bits but a 5-bit exponent, so the operands are scaled by powers of two:
//   * Ahat and the bias by 2^se per Gaussian (largest |Ahat| entry in [2^14, 2^15)): z' = 2^se z~;
//   * v = sqrt|w| z~ by 2^tv per launch, from the bounds: sqrt(g) |z~| <= 0.729 and |w| <= g H Amax,
//     so |v'| <= 2^14; S' and M are unscaled at the flush.
// With the hi / lo split the products keep ~22 bits as 3xTF32 does; what falls below f16's normal range
// is below 2^-28 of the largest term of its sum.
// The loop is issue-bound (ncu: 2.5 of 4 issue slots per SM-cycle, tensor pipe 35% busy), so the per-query scalars (g, w, sqrt|w|, gA, loss share, proxy) are computed
// once per (Gaussian, query): the 8 partial |z'|^2 sums a lane holds for the warp's two Gaussians x
// 16 queries (2 n-tiles x 2 queries) are reduce-scattered over the 8 gid lanes of its tig column, so
// lane (gid, tig) ends owning Gaussian gid & 1, n-tile (gid >> 1) & 1, query 2 tig + (gid >> 2) -- the
// 32 lanes own the 32 (Gaussian, query) pairs exactly once -- and w, sqrt|w| go back by shuffles.
__device__ __forceinline__ void mma16(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
    asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
                 "{%0,%1,%2,%3};\n"
                 : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
                 : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// (a, b) -> f16x2 hi (a in the low half) and the f16x2 of the residuals
__device__ __forceinline__ void split_h2(float a, float b, uint32_t& hi, uint32_t& lo) {
    const __half2 h = __floats2half2_rn(a, b);
    const float2 f = __half22float2(h);
    const __half2 l = __floats2half2_rn(a - f.x, b - f.y);
    hi = *reinterpret_cast<const uint32_t*>(&h);
    lo = *reinterpret_cast<const uint32_t*>(&l);
}

__device__ __forceinline__ float pow2f(int e) { return __int_as_float((127 + e) << 23); }   // |e| <= 126

template <int N>
__global__ void __launch_bounds__(kThreads, NDG_MMA_MINB)
    backward_mma_kernel(int64_t T, int tile, const float* __restrict__ qrec, const float* __restrict__ rec_tc,
                        const int64_t* __restrict__ offsets, const int32_t* __restrict__ idx,
                        const int64_t* __restrict__ items, int64_t Gev, const uint32_t* __restrict__ bounds,
                        unsigned long long* __restrict__ accum) {
    static_assert(N >= 9 && N <= 16, "K7-MMA covers 9 <= N <= 16 (one m16 block of dims)");
    constexpr int QS = qrec_floats(N);
    constexpr int K = tc_k(N);
    constexpr int RT = tc_rec_floats(N);
    constexpr int P = n_chol(N);
    constexpr int A = acc_doubles(N);
    extern __shared__ __align__(16) uint4 smem16[];
    const int tile16 = (tile + 15) & ~15;                 // the loop runs over 16-query blocks
    uint4* sX = smem16;                                   // [tile16/8][32 lanes] {xh(d0,d1), xh(d8,d9), xl.., xl..}
    float4* sQ = reinterpret_cast<float4*>(smem16 + (tile16 / 8) * 32);   // [tile16] {dpred0, dpred1, dpred2, ell}

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int gid = lane >> 2, tig = lane & 3, odd = gid & 1;
    float* sMm = reinterpret_cast<float*>(sQ + tile16) + warp * 16 * 17;   // per-warp M^T scratch
    const int64_t item = items[blockIdx.x];   // (tile << 32) | chunk, band order (ndg_work_items)
    if (item < 0) return;                        // unused slot of a worst-case-sized list (graph replay)
    const int64_t t = item >> 32;
    NDG_DCHECK(t >= 0 && t < T);
    const int64_t c0 = offsets[t] + (item & 0xffffffffLL) * kBwdChunk;
    const int64_t rem = offsets[t + 1] - c0;
    NDG_DCHECK(rem > 0);
    const int n_here = rem < kBwdChunk ? (int)rem : kBwdChunk;

    const FxScales fx = fx_scales(bounds, (int64_t)T * tile);
    // v' = 2^tv v with |v'| <= 2^14 (v = sqrt|w| z~, |w| <= H Amax, sqrt(g) |z~| <= 0.729)
    int tv = 0;
    {
        const float vmax = 0.73f * sqrtf(__uint_as_float(bounds[0]) * __uint_as_float(bounds[3]));
        if (vmax > 0.f && vmax < 3.0e38f) {
            int e;
            frexpf(vmax, &e);                            // vmax < 2^e
            tv = min(max(14 - e, -100), 100);
        }
    }

    // ---- the tile's Xhat fragments (f16 hi / lo) and (dpred, ell) in shared memory; a tile of 8 mod 16
    // queries is padded with one n-tile of zero queries (dpred = ell = 0: every term they enter is 0) ----
    const float* qt = qrec + t * tile * QS;
    for (int i = tid; i < tile16 * 4; i += kThreads) {        // (tile16/8) n-tiles x 32 lanes
        const int l = i & 31, nt = i >> 5;
        const int q = nt * 8 + (l >> 2), d0 = 2 * (l & 3);
        float x[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const int d = d0 + (k & 1) + (k >> 1) * 8;
            x[k] = (d < N && q < tile) ? qt[q * QS + d] - 0.5f : 0.f;
        }
        uint4 v;
        split_h2(x[0], x[1], v.x, v.z);
        split_h2(x[2], x[3], v.y, v.w);
        sX[i] = v;
    }
    for (int q = tid; q < tile16; q += kThreads)
        sQ[q] = q < tile ? make_float4(qt[q * QS + N], qt[q * QS + N + 1], qt[q * QS + N + 2], qt[q * QS + N + 3])
                         : make_float4(0.f, 0.f, 0.f, 0.f);
    __syncthreads();
    // the (Gaussian, n-tile, query) this lane owns in every 16-query block
    const int oj = gid & 1, ou = (gid >> 1) & 1, ob = gid >> 2;

    for (int gb = warp * kGpw; gb < n_here; gb += 4 * kGpw) {
        // ---- per-Gaussian operands (warp-uniform Gaussian; an absent second one runs on zeros) ----
        uint32_t ah[kGpw][4], al[kGpw][4];   // Ahat 16 x 16 fragment (rows = dims of z~, k = input dims)
        float bz[kGpw][2], col[kGpw][3], s2[kGpw], rsc[kGpw];
        int ses[kGpw];
        int64_t e[kGpw];
        bool live[kGpw];
#pragma unroll
        for (int j = 0; j < kGpw; ++j) {
            live[j] = gb + j < n_here;
            e[j] = live[j] ? idx[c0 + gb + j] : 0;
            NDG_DCHECK(e[j] >= 0 && e[j] < Gev);
            const float* r = rec_tc + e[j] * RT;
            auto at = [&](int i, int k) -> float {
                return (live[j] && i < N && k < N) ? __ldg(r + ((k / 4) * N + i) * 4 + (k & 3)) : 0.f;
            };
            // fragment order: (gid, 2tig..+1), (gid+8, 2tig..+1), (gid, 2tig+8..+9), (gid+8, 2tig+8..+9)
            float av[8];
#pragma unroll
            for (int f = 0; f < 4; ++f) {
                const int row = gid + (f & 1) * 8, k = 2 * tig + (f >> 1) * 8;
                av[2 * f] = at(row, k);
                av[2 * f + 1] = at(row, k + 1);
            }
            float m = 0.f;
#pragma unroll
            for (int f = 0; f < 8; ++f) m = fmaxf(m, fabsf(av[f]));
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
            int se = 0;
            if (m > 0.f) {
                int ex;
                frexpf(m, &ex);                          // m < 2^ex: scaled max in [2^14, 2^15)
                se = min(max(15 - ex, -100), 100);
            }
            const float sc = pow2f(se);
#pragma unroll
            for (int f = 0; f < 4; ++f) split_h2(av[2 * f] * sc, av[2 * f + 1] * sc, ah[j][f], al[j][f]);
            bz[j][0] = (live[j] && gid < N) ? __ldg(r + ((N / 4) * N + gid) * 4 + (N & 3)) * sc : 0.f;
            bz[j][1] = (live[j] && gid + 8 < N) ? __ldg(r + ((N / 4) * N + gid + 8) * 4 + (N & 3)) * sc : 0.f;
#pragma unroll
            for (int ch = 0; ch < 3; ++ch) col[j][ch] = live[j] ? __ldg(r + N * K + ch) : 0.f;
            s2[j] = pow2f(-2 * se);                      // |z~|^2 = 2^-2se |z'|^2
            rsc[j] = pow2f(tv - se);                     // v' = 2^tv sqrt|w| z~ = 2^(tv-se) sqrt|w| z'
            ses[j] = se;
        }
        // the owned Gaussian's per-query constants
        const float o_s2 = oj ? s2[1] : s2[0], o_rsc = oj ? rsc[1] : rsc[0];
        const float o_c0 = oj ? col[1][0] : col[0][0], o_c1 = oj ? col[1][1] : col[0][1],
                    o_c2 = oj ? col[1][2] : col[0][2];
        float S[kGpw][2][4] = {}, Mx[kGpw][2][4] = {};   // sum s v'_h v'_h^T and sum s v'_h v'_l^T fragments
        float tz[kGpw][2] = {}, gA[3] = {}, ls = 0.f, px = 0.f;   // gA, loss share, proxy: the owned Gaussian

        for (int nb16 = 0; nb16 < tile16 / 16; ++nb16) {
            const uint4 xf[2] = {sX[(nb16 * 2) * 32 + lane], sX[(nb16 * 2 + 1) * 32 + lane]};
            const float4 q = sQ[nb16 * 16 + ou * 8 + 2 * tig + ob];       // the owned query's (dpred, ell)
            // MMA1: z' (dims x 8 queries) = Ahat' xhat + bias' per (Gaussian, n-tile); corrections first
            float z[kGpw][2][4];
#pragma unroll
            for (int j = 0; j < kGpw; ++j)
#pragma unroll
                for (int u = 0; u < 2; ++u) {
                    z[j][u][0] = z[j][u][1] = bz[j][0];
                    z[j][u][2] = z[j][u][3] = bz[j][1];
                    mma16(z[j][u], al[j], xf[u].x, xf[u].y);
                    mma16(z[j][u], ah[j], xf[u].z, xf[u].w);
                    mma16(z[j][u], ah[j], xf[u].x, xf[u].y);
                }
            // |z'|^2 partials of this lane's dims (gid, gid + 8), index j*4 + u*2 + (query 2tig | 2tig+1),
            // reduce-scattered over the gid lanes: xor 4 splits j, xor 8 splits u, xor 16 the query
            float p[8];
#pragma unroll
            for (int j = 0; j < kGpw; ++j)
#pragma unroll
                for (int u = 0; u < 2; ++u) {
                    p[j * 4 + u * 2] = fmaf(z[j][u][2], z[j][u][2], z[j][u][0] * z[j][u][0]);
                    p[j * 4 + u * 2 + 1] = fmaf(z[j][u][3], z[j][u][3], z[j][u][1] * z[j][u][1]);
                }
            float k1[4], k2[2];
#pragma unroll
            for (int i = 0; i < 4; ++i)
                k1[i] = (oj ? p[4 + i] : p[i]) + __shfl_xor_sync(0xffffffffu, oj ? p[i] : p[4 + i], 4);
#pragma unroll
            for (int i = 0; i < 2; ++i)
                k2[i] = (ou ? k1[2 + i] : k1[i]) + __shfl_xor_sync(0xffffffffu, ou ? k1[i] : k1[2 + i], 8);
            const float sm = ((ob ? k2[1] : k2[0]) + __shfl_xor_sync(0xffffffffu, ob ? k2[0] : k2[1], 16)) * o_s2;
            // the owned pair's scalars
            const float gm = ex2_neg(sm);
            const float wm = gm * fmaf(q.z, o_c2, fmaf(q.y, o_c1, q.x * o_c0));
            // sqrt|w| (scaled) carrying the sign of w: one value per query to distribute
            const float rm = __uint_as_float(__float_as_uint(sqrt_approx(fabsf(wm)) * o_rsc) |
                                             (__float_as_uint(wm) & 0x80000000u));
            gA[0] = fmaf(gm, q.x, gA[0]);
            gA[1] = fmaf(gm, q.y, gA[1]);
            gA[2] = fmaf(gm, q.z, gA[2]);
            ls = fmaf(gm, q.w, ls);
            px = fmaf(fabsf(wm), sqrt_approx(sm), px);
#pragma unroll
            for (int j = 0; j < kGpw; ++j) {
                uint32_t ph[2][2], pl[2][2], am[2];      // [n-tile][dims gid | gid+8] packed v' hi / lo
#pragma unroll
                for (int u = 0; u < 2; ++u) {
                    // signed sqrt|w| of queries 2tig (a) and 2tig+1 (b) from their owners (same tig column)
                    const int src = ((j | (u << 1)) << 2) | tig;
                    const float ra = __shfl_sync(0xffffffffu, rm, src), rb = __shfl_sync(0xffffffffu, rm, src | 16);
                    const float v0 = fabsf(ra) * z[j][u][0], v1 = fabsf(rb) * z[j][u][1];
                    const float v2 = fabsf(ra) * z[j][u][2], v3 = fabsf(rb) * z[j][u][3];
                    // t' += w z' as (sign sqrt|w|) (sqrt|w| z') = rsc^2 w z', unscaled at the flush
                    tz[j][0] = fmaf(ra, v0, fmaf(rb, v1, tz[j][0]));
                    tz[j][1] = fmaf(ra, v2, fmaf(rb, v3, tz[j][1]));
                    split_h2(v0, v1, ph[u][0], pl[u][0]);
                    split_h2(v2, v3, ph[u][1], pl[u][1]);
                    am[u] = ((__float_as_uint(ra) & 0x80000000u) >> 16) | (__float_as_uint(rb) & 0x80000000u);
                }
                // MMA2: A = s v'_h (16 dims x 16 queries), B = v'_h | v'_l (16 queries x 8 dims) per column block
                const uint32_t a2[4] = {ph[0][0] ^ am[0], ph[0][1] ^ am[0], ph[1][0] ^ am[1], ph[1][1] ^ am[1]};
                mma16(Mx[j][0], a2, pl[0][0], pl[1][0]);
                mma16(Mx[j][1], a2, pl[0][1], pl[1][1]);
                mma16(S[j][0], a2, ph[0][0], ph[1][0]);
                mma16(S[j][1], a2, ph[0][1], ph[1][1]);
            }
        }

        // ---- flush: S' entries are owned by single lanes; t' reduces over tig, gA / loss share / proxy
        // over the 16 lanes owning each Gaussian. (Packing the slots over the warp -- 5 + 2 fx_adds per
        // lane instead of 8 half-predicated + single-lane tails -- measured the same: 176.1 vs 175.9 ms.)
        const float sS = pow2f(-2 * tv);
#pragma unroll
        for (int j = 0; j < kGpw; ++j) {
            if (!live[j]) continue;                       // warp-uniform
            unsigned long long* hw = accum + e[j] * A;
            unsigned long long* lw = hw + Gev * A;
            unsigned long long* flag = hw + acc_flag(N);
#pragma unroll
            for (int nb = 0; nb < 2; ++nb)
#pragma unroll
                for (int v = 0; v < 4; ++v)
                    sMm[(gid + (v >> 1) * 8) * 17 + nb * 8 + 2 * tig + (v & 1)] = Mx[j][nb][v];
            __syncwarp();
#pragma unroll
            for (int nb = 0; nb < 2; ++nb)
#pragma unroll
                for (int v = 0; v < 4; ++v) {
                    const int row = gid + (v >> 1) * 8, colj = nb * 8 + 2 * tig + (v & 1);
                    if (row < N && colj <= row)
                        fx_add(hw + tri(row, colj), lw + tri(row, colj), flag,
                               (S[j][nb][v] + Mx[j][nb][v] + sMm[colj * 17 + row]) * sS, fx.h);
                }
            __syncwarp();
            const float ts = pow2f(min(max(-tv, -126), 127)) * pow2f(min(max(ses[j] - tv, -126), 127));
            float r[2] = {tz[j][0] * ts, tz[j][1] * ts};     // t' = tz 2^-se / rsc^2 = tz 2^(se - 2 tv)
#pragma unroll
            for (int i = 0; i < 2; ++i) {
                r[i] += __shfl_xor_sync(0xffffffffu, r[i], 1);
                r[i] += __shfl_xor_sync(0xffffffffu, r[i], 2);
            }
            if (tig == 0) {
                fx_add(hw + P + gid, lw + P + gid, flag, r[0], fx.h);
                if (gid + 8 < N) fx_add(hw + P + gid + 8, lw + P + gid + 8, flag, r[1], fx.h);
            }
        }
        float r[5] = {gA[0], gA[1], gA[2], ls, px};
#pragma unroll
        for (int i = 0; i < 5; ++i) {
            r[i] += __shfl_xor_sync(0xffffffffu, r[i], 1);
            r[i] += __shfl_xor_sync(0xffffffffu, r[i], 2);
            r[i] += __shfl_xor_sync(0xffffffffu, r[i], 8);
            r[i] += __shfl_xor_sync(0xffffffffu, r[i], 16);
        }
        const bool o_live = oj ? live[1] : live[0];
        if (lane < 8 && tig == 0 && o_live) {
            unsigned long long* hw = accum + (oj ? e[1] : e[0]) * A;
            unsigned long long* lw = hw + Gev * A;
            unsigned long long* flag = hw + acc_flag(N);
            const int T0 = acc_tail(N);
            fx_add(hw + T0, lw + T0, flag, r[0], fx.g);
            fx_add(hw + T0 + 1, lw + T0 + 1, flag, r[1], fx.g);
            fx_add(hw + T0 + 2, lw + T0 + 2, flag, r[2], fx.g);
            fx_add(hw + T0 + 3, lw + T0 + 3, flag, r[3], fx.l);
            fx_add(hw + T0 + 4, lw + T0 + 4, flag, r[4], fx.h);
            atomicAdd(hw + T0 + 5, (unsigned long long)tile);
        }
    }
}

constexpr size_t kSmemX = sizeof(uint4) * 4;      // per query: Xhat fragments (tile16/8 n-tiles x 32 lanes x 16 B)
constexpr size_t kSmemW = sizeof(float) * 16 * 17;    // per warp: M^T scratch

template <int N>
int launch_backward_mma(int64_t B, int tile, const float* qrec, const float* rec_tc, const int64_t* off,
                        const int32_t* idx, const int64_t* items, int64_t n_chunks, int64_t Gev, const uint32_t* bounds,
                        unsigned long long* accum, cudaStream_t st) {
    const int64_t T = B / tile;
    const size_t tq = (tile + 15) & ~15;                  // the f16 form pads the tile to 16 queries
    const size_t smem = kSmemX * tq + sizeof(float4) * tq + kSmemW * 4;
    static DeviceOnce attr;
    if (attr.first())
        cudaFuncSetAttribute(backward_mma_kernel<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    NDG_REQUIRE(n_chunks <= 0x7fffffffLL, "too many backward work items");
    backward_mma_kernel<N><<<(unsigned)n_chunks, kThreads, smem, st>>>(T, tile, qrec, rec_tc, off, idx, items, Gev, bounds,
                                                                          accum);
    NDG_CHECK_LAUNCH();
    return NDG_OK;
}

}  // namespace

extern "C" int ndg_backward_mma_supported(int n) { return n >= 9 && n <= 16; }

extern "C" int ndg_backward_mma(int n, int64_t B, int tile, const float* qrec, const float* rec_tc,
                                const int64_t* offsets, const int32_t* idx, const int64_t* items,
                                int64_t n_chunks, int64_t Gev, const uint32_t* bounds, int64_t* accum, void* stream) {
    NDG_REQUIRE(tile >= 8 && tile <= 1024 && tile % 8 == 0 && B % tile == 0,
                "K7-MMA needs tile in 8..1024, a multiple of 8, dividing B");
    if (B == 0 || n_chunks == 0) return NDG_OK;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    switch (n) {
#define NDG_CASE(NN) \
    case NN:         \
        return launch_backward_mma<NN>(B, tile, qrec, rec_tc, offsets, idx, items, n_chunks, Gev, bounds, \
                                       reinterpret_cast<unsigned long long*>(accum), st);
        NDG_CASE(9) NDG_CASE(10) NDG_CASE(11) NDG_CASE(12) NDG_CASE(13) NDG_CASE(14) NDG_CASE(15) NDG_CASE(16)
#undef NDG_CASE
        default:
            return NDG_ERR_UNSUPPORTED_DIMS;
    }
}
