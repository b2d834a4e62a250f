// K7-MMA: the fused backward for large N on warp-level tensor cores (sm_100a, mma.sync m16n8k8
// tf32, 3xTF32 products, fp32 accumulation).
//
// Same contract as the FP32 K7 (ndg_backward.cu): per (tile, candidate) it adds
//   S' += (w z~) z~^T (lower),  t' += w z~,  gA += g dpred,  loss_share += g ell,  proxy += |w| sqrt(s~)
// to the fixed-point accumulators (deterministic, ndg_common.cuh), with w = g h, h = dpred . a,
// g = 2^-s~, s~ = |z~|^2, in the scaled z~ units of the FP32 K7, so the K8 epilogue is shared.
//
// Why a second kernel: the FP32 K7 keeps one Gaussian per thread with its record (P + 2N + 3 floats)
// AND its accumulators (P + N + 5) in registers. Past N = 12 that no longer fits in 255 registers;
// at N = 16 the pair loop reloads ~100 spilled floats per query from local memory and the kernel
// runs at a third of the FP32 peak. Here a warp owns a Gaussian and the 16 x 8 (dims x queries)
// block of z~ is one MMA:
//   MMA1  Z^T (16 x 8)  = Ahat (16 x 16) . Xhat^T (16 x 8),  C initialised to the bias column
//   MMA2  S'  (16 x 16) += (s V)^T-block (16 x 8) . V (8 x 16),  V = sqrt|w| Z, s = sign w
// MMA1's C fragment (lane (gid, tig): dims gid, gid+8 of queries 2tig, 2tig+1) IS the A and B
// fragment MMA2 needs once the query index k of MMA2 is relabelled (k = tig <-> query 2tig,
// k = tig + 4 <-> query 2tig + 1; the sum over queries does not care), so z~ never leaves the
// registers. With V = V_h + V_l, S' = sum s V_h V_h^T + M + M^T (M = sum s V_h V_l^T) takes two MMAs
// per column block where the plain 3xTF32 product u z^T takes three (same products kept, same lo.lo
// dropped); M^T is formed once per (tile, Gaussian) in shared memory. Ahat costs 16 registers per lane
// (hi | lo), S' and M 8 each, t' 2. The per-tile Xhat fragments
// (hi | lo, x - 1/2 as in K5) are built once per work item in shared memory and read as LDS.128.
//
// Ahat / bias / colour come from the K5 tensor-core record (rec_tc, ndg_tc_records): row i of Ahat is
// kC L^-1 (lower), column n the bias for xhat = x - 1/2, so z~ is bit-for-bit the K5 z~ up to fp32
// accumulation order. Its error grows like the z-GEMM's (RMS of B_e, engine.py guards it).
#include "ndg_common.cuh"
#include "ndg_tc.cuh"

using namespace ndg;

namespace {

#ifndef NDG_MMA_MINB
#define NDG_MMA_MINB 4
#endif
constexpr int kThreads = 128;   // 4 warps; work item = (tile, chunk of kBwdChunk candidates)
constexpr int kGpw = 2;         // Gaussians per warp in flight: the packed dims-8..15 k-step carries two

__device__ __forceinline__ void mma8(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
    asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
                 "{%0,%1,%2,%3};\n"
                 : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
                 : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

__device__ __forceinline__ uint32_t hi_bits(float x) { return __float_as_uint(x) & 0xFFFFE000u; }

struct Split4 {
    uint32_t hi[4], lo[4];
    __device__ __forceinline__ void set(float v0, float v1, float v2, float v3) {
        const float v[4] = {v0, v1, v2, v3};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            hi[i] = hi_bits(v[i]);
            lo[i] = __float_as_uint(v[i] - __uint_as_float(hi[i]));
        }
    }
};

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
    extern __shared__ __align__(16) float4 smem4[];
    float4* sX = smem4;                       // [tile/8][2 k-steps][32 lanes] {x_hi(b0), x_hi(b1), x_lo(b0), x_lo(b1)}
    float4* sQ = smem4 + (tile / 8) * 64;     // [tile] {dpred0, dpred1, dpred2, ell}

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int gid = lane >> 2, tig = lane & 3, odd = gid & 1;
    float* sM = reinterpret_cast<float*>(sQ + tile) + warp * 16 * 17;   // per-warp M^T scratch
    const int64_t item = items[blockIdx.x];   // (tile << 32) | chunk, band order (ndg_work_items)
    if (item < 0) return;                        // unused slot of a worst-case-sized list (graph replay)
    const int64_t t = item >> 32;
    NDG_DCHECK(t >= 0 && t < T);
    const int64_t c0 = offsets[t] + (item & 0xffffffffLL) * kBwdChunk;
    const int64_t rem = offsets[t + 1] - c0;
    NDG_DCHECK(rem > 0);
    const int n_here = rem < kBwdChunk ? (int)rem : kBwdChunk;

    const FxScales fx = fx_scales(bounds, (int64_t)T * tile);

    // ---- the tile's Xhat fragments and (dpred, ell) in shared memory -----------------------------
    const float* qt = qrec + t * tile * QS;
    for (int i = tid; i < tile * 8; i += kThreads) {          // (tile/8) n-tiles x 2 k-steps x 32 lanes
        const int l = i & 31, ks = (i >> 5) & 1, nt = i >> 6;
        const int q = nt * 8 + (l >> 2), d0 = ks * 8 + (l & 3), d1 = d0 + 4;
        const float x0 = d0 < N ? qt[q * QS + d0] - 0.5f : 0.f;
        const float x1 = d1 < N ? qt[q * QS + d1] - 0.5f : 0.f;
        const float h0 = __uint_as_float(hi_bits(x0)), h1 = __uint_as_float(hi_bits(x1));
        sX[i] = make_float4(h0, h1, x0 - h0, x1 - h1);
    }
    for (int q = tid; q < tile; q += kThreads)
        sQ[q] = make_float4(qt[q * QS + N], qt[q * QS + N + 1], qt[q * QS + N + 2], qt[q * QS + N + 3]);
    __syncthreads();

    for (int gb = warp * kGpw; gb < n_here; gb += 4 * kGpw) {
        // ---- per-Gaussian operands (warp-uniform Gaussian; an absent second one runs on zeros) ----
        // Ahat is lower triangular, so its k-step over dims 8..15 has zero rows 0..7: that k-step runs ONE
        // MMA for both Gaussians in flight, rows 0..7 = Gaussian 0's Ahat[8:16, 8:16], rows 8..15 =
        // Gaussian 1's (the B operand, the queries, is shared). Its C fragment then holds dims 8+gid of
        // Gaussian 0 in c0, c1 and of Gaussian 1 in c2, c3 -- the registers each Gaussian's z~ needs.
        Split4 a0f[kGpw], apk;                // Ahat[:, 0:8] per Gaussian; packed Ahat[8:16, 8:16] pair
        float bz[kGpw][2], col[kGpw][3];
        int64_t e[kGpw];
        bool live[kGpw];
        float pk[kGpw][2];
#pragma unroll
        for (int j = 0; j < kGpw; ++j) {
            live[j] = gb + j < n_here;
            e[j] = live[j] ? idx[c0 + gb + j] : 0;
            NDG_DCHECK(e[j] >= 0 && e[j] < Gev);
            const float* r = rec_tc + e[j] * RT;
            auto at = [&](int i, int k) -> float {
                return (live[j] && i < N && k < N) ? __ldg(r + ((k / 4) * N + i) * 4 + (k & 3)) : 0.f;
            };
            a0f[j].set(at(gid, tig), at(gid + 8, tig), at(gid, tig + 4), at(gid + 8, tig + 4));
            pk[j][0] = at(8 + gid, 8 + tig);
            pk[j][1] = at(8 + gid, 12 + tig);
            bz[j][0] = (live[j] && gid < N) ? __ldg(r + ((N / 4) * N + gid) * 4 + (N & 3)) : 0.f;
            bz[j][1] = (live[j] && gid + 8 < N) ? __ldg(r + ((N / 4) * N + gid + 8) * 4 + (N & 3)) : 0.f;
#pragma unroll
            for (int ch = 0; ch < 3; ++ch) col[j][ch] = live[j] ? __ldg(r + N * K + ch) : 0.f;
        }
        apk.set(pk[0][0], pk[1][0], pk[0][1], pk[1][1]);
        float S[kGpw][2][4] = {}, Mx[kGpw][2][4] = {};   // sum s v_h v_h^T and sum s v_h v_l^T fragments
        float tz[kGpw][2] = {}, gA[kGpw][3] = {}, ls[kGpw] = {}, px[kGpw] = {};

        for (int nt = 0; nt < tile / 8; ++nt) {
            const float4 xa = sX[nt * 64 + lane], xb = sX[nt * 64 + 32 + lane];
            // this lane's own query of the pair (2tig + odd): the per-query scalars are computed once per
            // lane pair (gid, gid ^ 1) instead of by all eight gid lanes
            const float4 qm = sQ[nt * 8 + 2 * tig + odd];
            const uint32_t xh[2][2] = {{__float_as_uint(xa.x), __float_as_uint(xa.y)},
                                       {__float_as_uint(xb.x), __float_as_uint(xb.y)}};
            const uint32_t xl[2][2] = {{__float_as_uint(xa.z), __float_as_uint(xa.w)},
                                       {__float_as_uint(xb.z), __float_as_uint(xb.w)}};
            // MMA1, k-step 1 (dims 8..15) for both Gaussians at once; biases of dims 8+gid in the accumulator,
            // the two correction products before hi.hi, all in one chain (fewer adds; the loop is issue-bound)
            float zp[4] = {bz[0][1], bz[0][1], bz[1][1], bz[1][1]};
            mma8(zp, apk.lo, xh[1][0], xh[1][1]);
            mma8(zp, apk.hi, xl[1][0], xl[1][1]);
            mma8(zp, apk.hi, xh[1][0], xh[1][1]);
#pragma unroll
            for (int j = 0; j < kGpw; ++j) {
                // MMA1, k-step 0 (dims 0..7) per Gaussian, accumulating onto the bias of dims gid and the
                // packed k-step's dims 8+gid
                float z[4] = {bz[j][0], bz[j][0], zp[2 * j], zp[2 * j + 1]};
                mma8(z, a0f[j].lo, xh[0][0], xh[0][1]);
                mma8(z, a0f[j].hi, xl[0][0], xl[0][1]);
                mma8(z, a0f[j].hi, xh[0][0], xh[0][1]);
                // s~ of queries 2tig (a) and 2tig+1 (b) from this lane's two dims, reduce-scattered over the
                // 8 gid lanes: even gid ends with s~(a), odd gid with s~(b)
                const float sa = fmaf(z[2], z[2], z[0] * z[0]), sb = fmaf(z[3], z[3], z[1] * z[1]);
                float sm = (odd ? sb : sa) + __shfl_xor_sync(0xffffffffu, odd ? sa : sb, 4);
                sm += __shfl_xor_sync(0xffffffffu, sm, 8);
                sm += __shfl_xor_sync(0xffffffffu, sm, 16);
                const float gm = ex2_neg(sm);
                const float wm = gm * fmaf(qm.z, col[j][2], fmaf(qm.y, col[j][1], qm.x * col[j][0]));
                const float rm = sqrt_approx(fabsf(wm));
                gA[j][0] = fmaf(gm, qm.x, gA[j][0]);
                gA[j][1] = fmaf(gm, qm.y, gA[j][1]);
                gA[j][2] = fmaf(gm, qm.z, gA[j][2]);
                ls[j] = fmaf(gm, qm.w, ls[j]);
                px[j] = fmaf(fabsf(wm), sqrt_approx(sm), px[j]);
                const float wo = __shfl_xor_sync(0xffffffffu, wm, 4), ro = __shfl_xor_sync(0xffffffffu, rm, 4);
                const float wa = odd ? wo : wm, wb = odd ? wm : wo;
                const float ra = odd ? ro : rm, rb = odd ? rm : ro;
                tz[j][0] = fmaf(wa, z[0], fmaf(wb, z[1], tz[j][0]));
                tz[j][1] = fmaf(wa, z[2], fmaf(wb, z[3], tz[j][1]));
                // S' = sum w z~ z~^T = sum s v v^T with v = sqrt|w| z~, s = sign w. Split v = v_h + v_l:
                // S' = sum s v_h v_h^T + M + M^T (M = sum s v_h v_l^T; v_l v_l^T dropped as in 3xTF32),
                // 2 MMAs per column block instead of 3. A = s v_h (rows = dims, k = relabelled queries),
                // B = v_h | v_l; C-fragment order [c0..c3] = (gid, qa), (gid, qb), (gid+8, qa), (gid+8, qb).
                Split4 vs;
                vs.set(ra * z[0], rb * z[1], ra * z[2], rb * z[3]);
                const uint32_t sga = __float_as_uint(wa) & 0x80000000u, sgb = __float_as_uint(wb) & 0x80000000u;
                const uint32_t av[4] = {vs.hi[0] ^ sga, vs.hi[2] ^ sga, vs.hi[1] ^ sgb, vs.hi[3] ^ sgb};
                // column block 0 = dims 0..7 (b = v(gid, q)); block 1 = dims 8..15 (b = v(gid+8, q))
                mma8(Mx[j][0], av, vs.lo[0], vs.lo[1]);
                mma8(Mx[j][1], av, vs.lo[2], vs.lo[3]);
                mma8(S[j][0], av, vs.hi[0], vs.hi[1]);
                mma8(S[j][1], av, vs.hi[2], vs.hi[3]);
            }
        }

        // ---- flush: S' entries are owned by single lanes; t', gA, loss share, proxy reduce over tig ----
#pragma unroll
        for (int j = 0; j < kGpw; ++j) {
            if (!live[j]) continue;                       // warp-uniform
            unsigned long long* hw = accum + e[j] * A;
            unsigned long long* lw = hw + Gev * A;
            unsigned long long* flag = hw + acc_flag(N);
            // S'[r][c] = P[r][c] + M[r][c] + M[c][r]: M^T through this warp's 16 x 17 scratch
#pragma unroll
            for (int nb = 0; nb < 2; ++nb)
#pragma unroll
                for (int v = 0; v < 4; ++v)
                    sM[(gid + (v >> 1) * 8) * 17 + nb * 8 + 2 * tig + (v & 1)] = Mx[j][nb][v];
            __syncwarp();
#pragma unroll
            for (int nb = 0; nb < 2; ++nb)
#pragma unroll
                for (int v = 0; v < 4; ++v) {
                    const int row = gid + (v >> 1) * 8, colj = nb * 8 + 2 * tig + (v & 1);
                    if (row < N && colj <= row)
                        fx_add(hw + tri(row, colj), lw + tri(row, colj), flag,
                               S[j][nb][v] + Mx[j][nb][v] + sM[colj * 17 + row], fx.h);
                }
            __syncwarp();
            float r[7] = {tz[j][0], tz[j][1], gA[j][0], gA[j][1], gA[j][2], ls[j], px[j]};
#pragma unroll
            for (int i = 0; i < 7; ++i) {
                r[i] += __shfl_xor_sync(0xffffffffu, r[i], 1);
                r[i] += __shfl_xor_sync(0xffffffffu, r[i], 2);
            }
#pragma unroll
            for (int i = 2; i < 7; ++i) r[i] += __shfl_xor_sync(0xffffffffu, r[i], 4);   // both queries of a pair
            if (tig == 0) {
                fx_add(hw + P + gid, lw + P + gid, flag, r[0], fx.h);
                if (gid + 8 < N) fx_add(hw + P + gid + 8, lw + P + gid + 8, flag, r[1], fx.h);
            }
            if (lane == 0) {
                const int T0 = acc_tail(N);
                fx_add(hw + T0, lw + T0, flag, r[2], fx.g);
                fx_add(hw + T0 + 1, lw + T0 + 1, flag, r[3], fx.g);
                fx_add(hw + T0 + 2, lw + T0 + 2, flag, r[4], fx.g);
                fx_add(hw + T0 + 3, lw + T0 + 3, flag, r[5], fx.l);
                fx_add(hw + T0 + 4, lw + T0 + 4, flag, r[6], fx.h);
                atomicAdd(hw + T0 + 5, (unsigned long long)tile);
            }
        }
    }
}

template <int N>
int launch_backward_mma(int64_t B, int tile, const float* qrec, const float* rec_tc, const int64_t* off,
                        const int32_t* idx, const int64_t* items, int64_t n_chunks, int64_t Gev, const uint32_t* bounds,
                        unsigned long long* accum, cudaStream_t st) {
    const int64_t T = B / tile;
    const size_t smem = sizeof(float4) * ((size_t)tile * 8 + tile) + sizeof(float) * 4 * 16 * 17;
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
