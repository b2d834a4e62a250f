// K7 fused backward (sm_100a, FP32 pipe, float64 cross-tile reduction).
//
// Replaces the pair loop of `backward`. Gaussian-stationary mapping: a work item
// is (tile, chunk of kBwdChunk candidates); each thread owns one candidate Gaussian, keeps its
// evaluation record AND all of its accumulators in registers, and sweeps the tile's query records
// (x | dpred | ell, staged in shared memory by one TMA bulk copy) as warp-uniform LDS.128
// broadcasts. Per pair, with h = dpred . a and w = g * h:
//   recompute z~, s~, g                              (as the forward)
//   S' += (w z~) z~^T (lower),  t' += w z~,  gA += g dpred
//   loss_share += g * ell,      proxy += |w| sqrt(s~)        (density-control statistics)
// so the per-query reduction the query-stationary mapping would need (A(N) warp shuffles per pair)
// disappears; the only reduction is one deterministic fixed-point add (two int64 words, ndg_common.cuh)
// per accumulator per (tile, candidate), amortised over the tile's queries, so the result does not
// depend on the order work items finish. Work items come in band order (ndg_work_items): the CTAs in
// flight share their candidates' records and accumulators in L2. ndg_acc_dequant and the epilogue
// (ndg_prep.cu) turn the words into float64 and apply the -1/C^2, -1/C scalings.
#include "ndg_common.cuh"

using namespace ndg;

namespace {

constexpr int kBwdThreads = kBwdChunk;

__host__ __device__ constexpr int srow_start(int i) {   // sum_{r<i} (r/2 + 1): packed S row offsets
    int s = 0;
    for (int r = 0; r < i; ++r) s += r / 2 + 1;
    return s;
}
#ifndef NDG_BWD_QUNROLL
#define NDG_BWD_QUNROLL 1   // query-loop unroll factor; tuning builds only
#endif
constexpr int kQUnroll = NDG_BWD_QUNROLL;
#ifndef NDG_BWD_SCALAR_S_MAXN
#define NDG_BWD_SCALAR_S_MAXN 7   // S' rows as scalar FFMA up to this N, FFMA2 pairs above (A/B: r02_k7_s_update_forms.txt)
#endif
#ifndef NDG_BWD_DIAG_SCALAR_MINN
#define NDG_BWD_DIAG_SCALAR_MINN 9   // from this N, even rows' diagonal S' entry as a scalar FFMA (A/B: r02_k7_s_update_forms.txt)
#endif
#ifndef NDG_BWD_MINB
#define NDG_BWD_MINB 3   // CTAs per SM the register budget is sized for (N <= 10); tuning builds only
#endif

template <int N, bool CTR>
__global__ void __launch_bounds__(kBwdThreads, (N <= 10 ? NDG_BWD_MINB : 1))
    backward_kernel(int64_t T, int tile, const float* __restrict__ qrec, const float* __restrict__ rec,
                    const int64_t* __restrict__ offsets, const int32_t* __restrict__ idx,
                    const int64_t* __restrict__ items, int64_t Gev, const uint32_t* __restrict__ bounds,
                    unsigned long long* __restrict__ accum) {
    constexpr int RS = rec_floats(N);
    constexpr int QS = qrec_floats(N);
    constexpr int P = n_chol(N);
    constexpr int A = acc_doubles(N);
    constexpr int A0 = rec_a(N);
    extern __shared__ __align__(128) float s_q[];   // [tile][QS]
    __shared__ __align__(8) uint64_t bar;

    const int tid = threadIdx.x;
    const int64_t item = items[blockIdx.x];      // (tile << 32) | chunk, band order
    if (item < 0) return;                        // unused slot of a worst-case-sized list (graph replay)
    const int64_t t = item >> 32;
    NDG_DCHECK(t >= 0 && t < T);
    const int64_t c = offsets[t] + (item & 0xffffffffLL) * kBwdChunk + tid;
    const bool active = c < offsets[t + 1];
    NDG_DCHECK(tid > 0 || active);                 // every work item holds at least one candidate

    if (tid == 0) {
        mbar_init(&bar, 1);
        fence_mbar_init();
    }
    __syncthreads();
    if (tid == 0) {
        const uint32_t bytes = (uint32_t)(tile * QS * 4);
        mbar_arrive_expect_tx(&bar, bytes);
        bulk_g2s(s_q, qrec + t * tile * QS, bytes, &bar);
    }

    float r[RS];
    int64_t e = 0;
    if (active) {
        e = idx[c];
        NDG_DCHECK(e >= 0 && e < Gev);
        const float4* r4 = reinterpret_cast<const float4*>(rec + e * RS);
#pragma unroll
        for (int v = 0; v < RS / 4; ++v) {
            const float4 x = __ldg(r4 + v);
            r[4 * v] = x.x;
            r[4 * v + 1] = x.y;
            r[4 * v + 2] = x.z;
            r[4 * v + 3] = x.w;
        }
    }
    mbar_wait(&bar, 0);
    if (!active) return;

    // scalar forward substitution (no added dependencies), packed FFMA2 for u = w z~, t += u and the
    // outer-product rows S_i,(2jp, 2jp+1) += u_i (z~_2jp, z~_2jp+1)
    constexpr int NZP = (N + 1) / 2;
    constexpr int NSP = srow_start(N);
    float2 Sp[NSP], tv2[NZP];
    float gA0 = 0.f, gA1 = 0.f, gA2 = 0.f, ls = 0.f, px = 0.f;
#pragma unroll
    for (int i = 0; i < NSP; ++i) Sp[i] = make_float2(0.f, 0.f);
#pragma unroll
    for (int i = 0; i < NZP; ++i) tv2[i] = make_float2(0.f, 0.f);
#pragma unroll kQUnroll
    for (int q = 0; q < tile; ++q) {
        float xq[QS];
        const float4* q4 = reinterpret_cast<const float4*>(s_q + q * QS);
#pragma unroll
        for (int v = 0; v < QS / 4; ++v) {
            const float4 x = q4[v];
            xq[4 * v] = x.x;
            xq[4 * v + 1] = x.y;
            xq[4 * v + 2] = x.z;
            xq[4 * v + 3] = x.w;
        }
        float2 z2[NZP];
        z2[NZP - 1] = make_float2(0.f, 0.f);
        float s2 = 0.f;
#pragma unroll
        for (int i = 0; i < N; ++i) {
            // centred records hold (m_hi, m_lo) in the nb2 slots: z = rho ((x - m_hi) - m_lo), no cancellation
            float acc = CTR ? r[rec_rho(N) + i] * ((xq[i] - r[rec_nb2(N) + 2 * i]) - r[rec_nb2(N) + 2 * i + 1])
                            : fmaf(r[rec_rho(N) + i], xq[i], r[rec_nb2(N) + 2 * i]);
#ifndef NDG_BWD_KO_SUBST   // knock-out build: drop the triangular solve's off-diagonal terms (wrong results)
#pragma unroll
            for (int k = 0; k < i; ++k) acc = fmaf(r[rec_l(N, i, k)], (k & 1) ? z2[k / 2].y : z2[k / 2].x, acc);
#endif
            if (i & 1) z2[i / 2].y = acc;
            else z2[i / 2].x = acc;
            s2 = fmaf(acc, acc, s2);
        }
        const float g = ex2_neg(s2);
        const float dp0 = xq[N], dp1 = xq[N + 1], dp2 = xq[N + 2], ell = xq[N + 3];
        const float h = fmaf(dp2, r[A0 + 2], fmaf(dp1, r[A0 + 1], dp0 * r[A0]));
        const float wgt = g * h;
        float2 u2[NZP];
#pragma unroll
        for (int kp = 0; kp < NZP; ++kp) {
            u2[kp] = __fmul2_rn(make_float2(wgt, wgt), z2[kp]);
            tv2[kp] = __fadd2_rn(tv2[kp], u2[kp]);
        }
#pragma unroll
        for (int i = 0; i < N; ++i) {
            const float ui = (i & 1) ? u2[i / 2].y : u2[i / 2].x;
#ifndef NDG_BWD_KO_S       // knock-out build: no S' update (wrong results)
            if constexpr (N <= NDG_BWD_SCALAR_S_MAXN) {
                // small N: scalar FFMA rows (no padded lane); the loop is short enough that issue is not the
                // limit (tools/kbench.py, profiles/r02_k7_instruction_forms_rejected.txt)
#pragma unroll
                for (int j = 0; j <= i; ++j) {
                    float2& sp = Sp[srow_start(i) + j / 2];
                    if (j & 1) sp.y = fmaf(ui, z2[j / 2].y, sp.y);
                    else sp.x = fmaf(ui, z2[j / 2].x, sp.x);
                }
            } else if constexpr (N >= NDG_BWD_DIAG_SCALAR_MINN) {
                // FFMA2 over the row's full pairs; an even row's last (diagonal) entry as one scalar FFMA
                // instead of a padded FFMA2: same instruction count, 5 fewer lane-cycles per pair at N = 10
#pragma unroll
                for (int jp = 0; jp < (i + 1) / 2; ++jp)
                    Sp[srow_start(i) + jp] = __ffma2_rn(make_float2(ui, ui), z2[jp], Sp[srow_start(i) + jp]);
                if (!(i & 1)) Sp[srow_start(i) + i / 2].x = fmaf(ui, z2[i / 2].x, Sp[srow_start(i) + i / 2].x);
            } else {
#pragma unroll
                for (int jp = 0; jp <= i / 2; ++jp)
                    Sp[srow_start(i) + jp] = __ffma2_rn(make_float2(ui, ui), z2[jp], Sp[srow_start(i) + jp]);
            }
#endif
        }
        gA0 = fmaf(g, dp0, gA0);
        gA1 = fmaf(g, dp1, gA1);
        gA2 = fmaf(g, dp2, gA2);
        ls = fmaf(g, ell, ls);
        px = fmaf(fabsf(wgt), sqrt_approx(s2), px);
    }

    const FxScales fx = fx_scales(bounds, (int64_t)T * tile);
    unsigned long long* hw = accum + e * A;
    unsigned long long* lw = hw + Gev * A;
    unsigned long long* flag = hw + acc_flag(N);
#pragma unroll
    for (int i = 0; i < N; ++i)
#pragma unroll
        for (int j = 0; j <= i; ++j) {
            const float2 v = Sp[srow_start(i) + j / 2];
            fx_add(hw + tri(i, j), lw + tri(i, j), flag, (j & 1) ? v.y : v.x, fx.h);
        }
#pragma unroll
    for (int i = 0; i < N; ++i) fx_add(hw + P + i, lw + P + i, flag, (i & 1) ? tv2[i / 2].y : tv2[i / 2].x, fx.h);
    const int T0 = acc_tail(N);
    fx_add(hw + T0, lw + T0, flag, gA0, fx.g);
    fx_add(hw + T0 + 1, lw + T0 + 1, flag, gA1, fx.g);
    fx_add(hw + T0 + 2, lw + T0 + 2, flag, gA2, fx.g);
    fx_add(hw + T0 + 3, lw + T0 + 3, flag, ls, fx.l);
    fx_add(hw + T0 + 4, lw + T0 + 4, flag, px, fx.h);
    atomicAdd(hw + T0 + 5, (unsigned long long)tile);
}

template <int N>
int launch_backward(int64_t B, int tile, const float* qrec, const float* rec, int centred, const int64_t* off,
                    const int32_t* idx, const int64_t* items, int64_t n_chunks, int64_t Gev, const uint32_t* bounds,
                    unsigned long long* accum, cudaStream_t st) {
    const int64_t T = B / tile;
    const size_t smem = sizeof(float) * tile * qrec_floats(N);
    static DeviceOnce attr;
    if (attr.first()) {
        cudaFuncSetAttribute(backward_kernel<N, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        cudaFuncSetAttribute(backward_kernel<N, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    }
    NDG_REQUIRE(n_chunks <= 0x7fffffffLL, "too many backward work items");
    auto kern = centred ? backward_kernel<N, true> : backward_kernel<N, false>;
    kern<<<(unsigned)n_chunks, kBwdThreads, smem, st>>>(T, tile, qrec, rec, off, idx, items, Gev, bounds, accum);
    NDG_CHECK_LAUNCH();
    return NDG_OK;
}

}  // namespace

extern "C" int ndg_backward(int n, int64_t B, int tile, const float* qrec, const float* rec, int centred,
                            const int64_t* offsets, const int32_t* idx, const int64_t* items, int64_t n_chunks,
                            int64_t Gev, const uint32_t* bounds, int64_t* accum, void* stream) {
    NDG_REQUIRE(tile >= 1 && tile <= 1024 && B % tile == 0, "tile must be in 1..1024 and divide B");
    if (B == 0 || n_chunks == 0) return NDG_OK;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    switch (n) {
#define NDG_CASE(NN) \
    case NN:         \
        return launch_backward<NN>(B, tile, qrec, rec, centred, offsets, idx, items, n_chunks, Gev, bounds, \
                                   reinterpret_cast<unsigned long long*>(accum), st);
        NDG_CASE(1) NDG_CASE(2) NDG_CASE(3) NDG_CASE(4) NDG_CASE(5) NDG_CASE(6) NDG_CASE(7) NDG_CASE(8)
        NDG_CASE(9) NDG_CASE(10) NDG_CASE(11) NDG_CASE(12) NDG_CASE(13) NDG_CASE(14) NDG_CASE(15) NDG_CASE(16)
#undef NDG_CASE
        default:
            return NDG_ERR_UNSUPPORTED_DIMS;
    }
}
