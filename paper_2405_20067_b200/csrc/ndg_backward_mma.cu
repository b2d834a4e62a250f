// K7-MMA: the fused backward for large N on warp-level tensor cores (sm_100a, mma.sync m16n8k8
// tf32, 3xTF32 products, fp32 accumulation).
//
// Same contract as the FP32 K7 (ndg_backward.cu): per (tile, candidate) it adds
//   S' += (w z~) z~^T (lower),  t' += w z~,  gA += g dpred,  loss_share += g ell,  proxy += |w| sqrt(s~)
// to the float64 accumulators, with w = g h, h = dpred . a, g = 2^-s~, s~ = |z~|^2, in the scaled z~
// units of the FP32 K7, so the K8 epilogue is shared.
//
// Why a second kernel: the FP32 K7 keeps one Gaussian per thread with its record (P + 2N + 3 floats)
// AND its accumulators (P + N + 5) in registers. Past N = 12 that no longer fits in 255 registers;
// at N = 16 the pair loop reloads ~100 spilled floats per query from local memory and the kernel
// runs at a third of the FP32 peak. Here a warp owns a Gaussian and the 16 x 8 (dims x queries)
// block of z~ is one MMA:
//   MMA1  Z^T (16 x 8)  = Ahat (16 x 16) . Xhat^T (16 x 8),  C initialised to the bias column
//   MMA2  S'  (16 x 16) += (w Z)^T-block (16 x 8) . Z (8 x 16)
// MMA1's C fragment (lane (gid, tig): dims gid, gid+8 of queries 2tig, 2tig+1) IS the A and B
// fragment MMA2 needs once the query index k of MMA2 is relabelled (k = tig <-> query 2tig,
// k = tig + 4 <-> query 2tig + 1; the sum over queries does not care), so z~ never leaves the
// registers. Ahat costs 16 registers per lane (hi | lo), S' 8, t' 2. The per-tile Xhat fragments
// (hi | lo, x - 1/2 as in K5) are built once per work item in shared memory and read as LDS.128.
//
// Ahat / bias / colour come from the K5 tensor-core record (rec_tc, ndg_tc_records): row i of Ahat is
// kC L^-1 (lower), column n the bias for xhat = x - 1/2, so z~ is bit-for-bit the K5 z~ up to fp32
// accumulation order. Its error grows like the z-GEMM's (RMS of B_e, engine.py guards it).
#include "ndg_common.cuh"
#include "ndg_tc.cuh"

using namespace ndg;

namespace {

#ifndef NDG_MMA_GPW
#define NDG_MMA_GPW 2
#endif
#ifndef NDG_MMA_MINB
#define NDG_MMA_MINB 4
#endif
constexpr int kThreads = 128;   // 4 warps; work item = (tile, chunk of kBwdChunk candidates)
constexpr int kGpw = NDG_MMA_GPW;   // Gaussians per warp in flight (independent MMA chains)

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
                        const int64_t* __restrict__ chunk_off, double* __restrict__ accum) {
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
    const int gid = lane >> 2, tig = lane & 3;
    const int64_t w = blockIdx.x;
    int64_t lo = 0, hi = T;                   // tile t with chunk_off[t] <= w < chunk_off[t+1]
    while (hi - lo > 1) {
        const int64_t mid = (lo + hi) >> 1;
        if (chunk_off[mid] <= w) lo = mid;
        else hi = mid;
    }
    const int64_t t = lo;
    const int64_t c0 = offsets[t] + (w - chunk_off[t]) * kBwdChunk;
    const int64_t rem = offsets[t + 1] - c0;
    const int n_here = rem < kBwdChunk ? (int)rem : kBwdChunk;

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
        Split4 ah[kGpw][2];                   // Ahat A-fragments per k-step, hi | lo
        float bz[kGpw][2], col[kGpw][3];
        int64_t e[kGpw];
        bool live[kGpw];
#pragma unroll
        for (int j = 0; j < kGpw; ++j) {
            live[j] = gb + j < n_here;
            e[j] = live[j] ? idx[c0 + gb + j] : 0;
            const float* r = rec_tc + e[j] * RT;
            auto at = [&](int i, int k) -> float {
                return (live[j] && i < N && k < N) ? __ldg(r + ((k / 4) * N + i) * 4 + (k & 3)) : 0.f;
            };
#pragma unroll
            for (int ks = 0; ks < 2; ++ks)
                ah[j][ks].set(at(gid, ks * 8 + tig), at(gid + 8, ks * 8 + tig), at(gid, ks * 8 + tig + 4),
                              at(gid + 8, ks * 8 + tig + 4));
            bz[j][0] = (live[j] && gid < N) ? __ldg(r + ((N / 4) * N + gid) * 4 + (N & 3)) : 0.f;
            bz[j][1] = (live[j] && gid + 8 < N) ? __ldg(r + ((N / 4) * N + gid + 8) * 4 + (N & 3)) : 0.f;
#pragma unroll
            for (int ch = 0; ch < 3; ++ch) col[j][ch] = live[j] ? __ldg(r + N * K + ch) : 0.f;
        }
        float S[kGpw][2][4] = {}, tz[kGpw][2] = {}, gA[kGpw][3] = {}, ls[kGpw] = {}, px[kGpw] = {};

        for (int nt = 0; nt < tile / 8; ++nt) {
            const float4 xa = sX[nt * 64 + lane], xb = sX[nt * 64 + 32 + lane];
            const float4 qa = sQ[nt * 8 + 2 * tig], qb = sQ[nt * 8 + 2 * tig + 1];
            const uint32_t xh[2][2] = {{__float_as_uint(xa.x), __float_as_uint(xa.y)},
                                       {__float_as_uint(xb.x), __float_as_uint(xb.y)}};
            const uint32_t xl[2][2] = {{__float_as_uint(xa.z), __float_as_uint(xa.w)},
                                       {__float_as_uint(xb.z), __float_as_uint(xb.w)}};
#pragma unroll
            for (int j = 0; j < kGpw; ++j) {
                // MMA1: z~ block, bias in the accumulator, correction products in a second chain
                float z[4] = {bz[j][0], bz[j][0], bz[j][1], bz[j][1]};
                float zc[2][4] = {};
#pragma unroll
                for (int ks = 0; ks < 2; ++ks) {
                    mma8(zc[ks], ah[j][ks].lo, xh[ks][0], xh[ks][1]);
                    mma8(zc[ks], ah[j][ks].hi, xl[ks][0], xl[ks][1]);
                    mma8(z, ah[j][ks].hi, xh[ks][0], xh[ks][1]);
                }
#pragma unroll
                for (int i = 0; i < 4; ++i) z[i] += zc[0][i] + zc[1][i];
                // s~ of queries 2tig (a) and 2tig+1 (b): this lane's two dims, then over the 8 gid lanes
                float sa = fmaf(z[2], z[2], z[0] * z[0]), sb = fmaf(z[3], z[3], z[1] * z[1]);
#pragma unroll
                for (int m = 4; m < 32; m <<= 1) {
                    sa += __shfl_xor_sync(0xffffffffu, sa, m);
                    sb += __shfl_xor_sync(0xffffffffu, sb, m);
                }
                const float ga = ex2_neg(sa), gb2 = ex2_neg(sb);
                const float ha = fmaf(qa.z, col[j][2], fmaf(qa.y, col[j][1], qa.x * col[j][0]));
                const float hb = fmaf(qb.z, col[j][2], fmaf(qb.y, col[j][1], qb.x * col[j][0]));
                const float wa = ga * ha, wb = gb2 * hb;
                // MMA2 operands: A = u = w z~ (rows = dims, k = relabelled queries), B = z~
                const float u0 = wa * z[0], u1 = wa * z[2], u2 = wb * z[1], u3 = wb * z[3];
                tz[j][0] += u0 + u2;
                tz[j][1] += u1 + u3;
                Split4 us, zs;
                us.set(u0, u1, u2, u3);
                zs.set(z[0], z[1], z[2], z[3]);
                // n-tile 0: columns = dims 0..7 (b = z~(gid, q)); n-tile 1: dims 8..15 (b = z~(gid+8, q))
                mma8(S[j][0], us.lo, zs.hi[0], zs.hi[1]);
                mma8(S[j][1], us.lo, zs.hi[2], zs.hi[3]);
                mma8(S[j][0], us.hi, zs.lo[0], zs.lo[1]);
                mma8(S[j][1], us.hi, zs.lo[2], zs.lo[3]);
                mma8(S[j][0], us.hi, zs.hi[0], zs.hi[1]);
                mma8(S[j][1], us.hi, zs.hi[2], zs.hi[3]);
                gA[j][0] = fmaf(ga, qa.x, fmaf(gb2, qb.x, gA[j][0]));
                gA[j][1] = fmaf(ga, qa.y, fmaf(gb2, qb.y, gA[j][1]));
                gA[j][2] = fmaf(ga, qa.z, fmaf(gb2, qb.z, gA[j][2]));
                ls[j] = fmaf(ga, qa.w, fmaf(gb2, qb.w, ls[j]));
                px[j] = fmaf(fabsf(wa), sqrt_approx(sa), fmaf(fabsf(wb), sqrt_approx(sb), px[j]));
            }
        }

        // ---- flush: S' entries are owned by single lanes; t', gA, loss share, proxy reduce over tig ----
#pragma unroll
        for (int j = 0; j < kGpw; ++j) {
            if (!live[j]) continue;                       // warp-uniform
            double* out = accum + e[j] * A;
#pragma unroll
            for (int nb = 0; nb < 2; ++nb)
#pragma unroll
                for (int v = 0; v < 4; ++v) {
                    const int row = gid + (v >> 1) * 8, colj = nb * 8 + 2 * tig + (v & 1);
                    if (row < N && colj <= row) atomicAdd(out + tri(row, colj), (double)S[j][nb][v]);
                }
            float r[7] = {tz[j][0], tz[j][1], gA[j][0], gA[j][1], gA[j][2], ls[j], px[j]};
#pragma unroll
            for (int i = 0; i < 7; ++i) {
                r[i] += __shfl_xor_sync(0xffffffffu, r[i], 1);
                r[i] += __shfl_xor_sync(0xffffffffu, r[i], 2);
            }
            if (tig == 0) {
                atomicAdd(out + P + gid, (double)r[0]);
                if (gid + 8 < N) atomicAdd(out + P + gid + 8, (double)r[1]);
            }
            if (lane == 0) {
                atomicAdd(out + acc_tail(N), (double)r[2]);
                atomicAdd(out + acc_tail(N) + 1, (double)r[3]);
                atomicAdd(out + acc_tail(N) + 2, (double)r[4]);
                atomicAdd(out + acc_tail(N) + 3, (double)r[5]);
                atomicAdd(out + acc_tail(N) + 4, (double)r[6]);
                atomicAdd(out + acc_tail(N) + 5, (double)tile);
            }
        }
    }
}

template <int N>
int launch_backward_mma(int64_t B, int tile, const float* qrec, const float* rec_tc, const int64_t* off,
                        const int32_t* idx, const int64_t* chunk_off, int64_t n_chunks, double* accum, cudaStream_t st) {
    const int64_t T = B / tile;
    const size_t smem = sizeof(float4) * ((size_t)tile * 8 + tile);
    static DeviceOnce attr;
    if (attr.first())
        cudaFuncSetAttribute(backward_mma_kernel<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    NDG_REQUIRE(n_chunks <= 0x7fffffffLL, "too many backward work items");
    backward_mma_kernel<N><<<(unsigned)n_chunks, kThreads, smem, st>>>(T, tile, qrec, rec_tc, off, idx, chunk_off, accum);
    NDG_CHECK_LAUNCH();
    return NDG_OK;
}

}  // namespace

extern "C" int ndg_backward_mma_supported(int n) { return n >= 9 && n <= 16; }

extern "C" int ndg_backward_mma(int n, int64_t B, int tile, const float* qrec, const float* rec_tc,
                                const int64_t* offsets, const int32_t* idx, const int64_t* chunk_offsets,
                                int64_t n_chunks, double* accum, void* stream) {
    NDG_REQUIRE(tile >= 8 && tile <= 1024 && tile % 8 == 0 && B % tile == 0,
                "K7-MMA needs tile in 8..1024, a multiple of 8, dividing B");
    if (B == 0 || n_chunks == 0) return NDG_OK;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    switch (n) {
#define NDG_CASE(NN) \
    case NN:         \
        return launch_backward_mma<NN>(B, tile, qrec, rec_tc, offsets, idx, chunk_offsets, n_chunks, accum, st);
        NDG_CASE(9) NDG_CASE(10) NDG_CASE(11) NDG_CASE(12) NDG_CASE(13) NDG_CASE(14) NDG_CASE(15) NDG_CASE(16)
#undef NDG_CASE
        default:
            return NDG_ERR_UNSUPPORTED_DIMS;
    }
}
