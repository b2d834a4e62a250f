// K5+K6 fused forward + loss on the 5th-gen tensor cores (tcgen05, kind::tf32, 3xTF32).
//
// Replaces eval_mixture over each tile's candidate list (Eq. 8) + loss_rel_l2
// (SPEC.md:253-261). The Mahalanobis solve becomes a GEMM: with the per-Gaussian record
// Ahat_e = [C L_e^-1 | C L_e^-1 (1/2 - m_e)] (K1 + ndg_tc_records, float64 -> float32) and the
// query features xhat_q = [x_q - 1/2, 1],
//     z~[q, (e,i)] = sum_k xhat_q[k] Ahat_e[i][k]      (= C * z_i of L z = x - m)
// computed by tcgen05.mma (M = 128 queries of one tile half, N = 224 columns = C Gaussians x N rows in
// two 16-aligned groups, K = pad8(N+1)) in 3xTF32 (hi*hi + hi*lo + lo*hi, fp32 accumulate in TMEM):
// tools/tc_precision_study.py shows <= 4.4e-5 block-relative error on pred at sigma 0.02 (bar 1e-4);
// HotPath's conditioning guard keeps sharper mixtures on the FP32 pipe. The epilogue warps read z~
// rows from TMEM and finish on the FP32 pipe:
//     s~ = sum_i z~_i^2 (FFMA2 over column pairs),  g = ex2(-s~),  pred += g * a.
//
// Pipeline (416 threads, one CTA per tile of 256 queries): two producer warps gather whole candidate
// records into a staging ring (cp.async.bulk), two splitter warps convert them to the hi/lo K-major B
// planes, one lane issues the MMAs of item (chunk, half) into TMEM buffer `half`, eight epilogue
// warps (4 lane quarters x 2 Gaussian groups) drain TMEM (2 x 224 accumulator + 64 A columns = 512).
// The hand-off timeline (tools/tc_trace.py) shows the tensor pipe ~85% busy per chunk.
#include <algorithm>

#include "ndg_tc.cuh"

using namespace ndg;

namespace {

#ifndef NDG_TC_SPLITTERS
#define NDG_TC_SPLITTERS 2
#endif
#ifndef NDG_TC_STAGING
#define NDG_TC_STAGING 8
#endif
constexpr int kSplit = NDG_TC_SPLITTERS;   // splitter warps (2 .. 2 + kSplit - 1)
constexpr int kEpi0 = 2 + kSplit;           // first epilogue warp (a multiple of 4: lane quarter = warp % 4)
constexpr int kEpiW = 8;                    // epilogue warps (2 Gaussian groups x 4 lane quarters)
static_assert(kEpi0 % 4 == 0, "epilogue warp w must own TMEM lane quarter w % 4");
#ifndef NDG_TC_PRODUCERS
#define NDG_TC_PRODUCERS 2
#endif
// Producer warps: warp 0 and the kProd - 1 warps after the epilogue. A cp.async.bulk gather issues through the uniform
// datapath one record at a time, so one warp issuing all of a chunk's records paced the pipeline
// (tools/tc_trace.py: half the gathers -> -10%); producer p takes chunks c = p (mod kProd).
constexpr int kProd = NDG_TC_PRODUCERS;
constexpr int kTcWarps = kEpi0 + kEpiW + (kProd - 1);
constexpr int kTcThreads = kTcWarps * 32;
constexpr int kTcStaging = NDG_TC_STAGING;   // raw-record staging ring depth (capped per N by the smem budget)
constexpr int kTBuf = 2;                      // TMEM accumulator buffers: one per query half

constexpr int kARing = 8;                     // colour ring depth (independent of the B ring)
constexpr int kMaxCluster = 2;                // CTAs per tile when the batch has fewer tiles than SMs

__device__ __forceinline__ void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// float at the same shared-memory offset in cluster CTA `rank` (distributed shared memory)
__device__ __forceinline__ float ld_cluster_f32(const float* p, int rank) {
    uint32_t remote;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(smem_u32(p)), "r"(rank));
    float v;
    asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(v) : "r"(remote) : "memory");
    return v;
}

#ifdef NDG_TCX_TRACE
// Timeline probe (tuning builds only): clock64 at each hand-off of the first kTrC chunks of one CTA.
constexpr int kTrC = 64, kTrEv = 10;
__device__ long long g_trace[kTrC * kTrEv];
#define NDG_TR(ev, c)                                                                          \
    do {                                                                                       \
        if (blockIdx.x == kTraceCta && (c) < kTrC) g_trace[(c) * kTrEv + (ev)] = clock64();  \
    } while (0)
constexpr unsigned kTraceCta = 300;
#else
#define NDG_TR(ev, c) \
    do {              \
    } while (0)
#endif

// Items: a chunk's z-GEMM covers C Gaussians (MMA N = 224 at N = 10) and runs one query half at a time
// (item = (chunk, half) -> TMEM buffer = half), so each tcgen05.mma does as much work per issue as TMEM
// allows; the epilogue splits a chunk's Gaussians into two groups per lane quarter (columns
// [0, CG*N) and [GOFF, GOFF + (C-CG)*N), GOFF 16-aligned).

template <int N>
struct TcCfg {
    static constexpr int K = tc_k(N);
    static constexpr int P = K / 4;
    static constexpr int KS = K / 8;
    // TMEM: A operand (2 halves x hi/lo x K columns) + one NCOL-column accumulator buffer per query half
    static constexpr int ACOLS = 4 * K;
    static constexpr int NCOL = ((512 - ACOLS) / kTBuf) & ~15;           // MMA N (224 at N = 10)
    static constexpr int A0 = kTBuf * NCOL;                              // first A column
    static constexpr int PLANE = NCOL * 16;                              // B plane: NCOL rows x 16 B
    static constexpr int items_c() {
        int c = NCOL / N < 32 ? NCOL / N : 32;
        while (c > 1 && ((((c + 1) / 2) * N + 15) / 16) * 16 + (c - (c + 1) / 2) * N > NCOL) --c;
        return c;
    }
    static constexpr int C = items_c();                                  // Gaussians per chunk (<= 32 producer lanes)
    static constexpr int CG = (C + 1) / 2;                               // Gaussians of epilogue group 0
    static constexpr int GOFF = ((CG * N + 15) / 16) * 16;               // first column of group 1
    static constexpr int RT = tc_rec_floats(N);       // floats per raw record (rows | a | pad)
    static constexpr size_t kRing = (size_t)kARing * C * 16;
    static constexpr size_t kSlot = (size_t)C * RT * 4;
    static constexpr size_t kBudget = 222 * 1024;    // 227 KB per CTA minus static shared memory (s_pp, barriers)
    static constexpr size_t stage_bytes = (size_t)2 * P * PLANE;
    static constexpr int STAGES = (4 * stage_bytes + kRing + 2 * kSlot <= kBudget) ? 4 : 3;
    static constexpr size_t kFixed = (size_t)STAGES * stage_bytes + kRing;
    // staging depth: as deep as NDG_TC_STAGING, but the whole ring set must fit in shared memory
    static constexpr int STG = (kFixed + kTcStaging * kSlot <= kBudget) ? kTcStaging : (int)((kBudget - kFixed) / kSlot);
    static_assert(STG >= 2, "shared-memory budget too small for the staging ring");
    static_assert(kARing >= STAGES + kTBuf + 1, "colour-slot reuse relies on the B-stage wait (splitters)");
    static_assert(kTBuf == 2, "one TMEM accumulator buffer per query half");
};

template <int N>
constexpr size_t tc_smem_bytes() {
    using C_ = TcCfg<N>;
    return C_::kFixed + (size_t)C_::STG * C_::kSlot;
}

// Warp roles: 0 and kTcWarps-1 = TMA producers (even / odd chunks; one cp.async.bulk per candidate
// record into the staging ring), 1 = TMEM allocator + MMA issuer, 2..kEpi0-1 = splitters (staging ->
// hi/lo K-major B planes + colours), kEpi0..kEpi0+7 = epilogue (warp w: Gaussian group (w-kEpi0)/4,
// TMEM lane quarter w%4; the A-operand prologue writes query half (w-kEpi0)/4).
template <int N, int CS>
__global__ void __launch_bounds__(kTcThreads, 1)
    forward_tc_kernel(int tile, const float* __restrict__ queries, const float* __restrict__ targets,
                      const float* __restrict__ rec_tc, const int64_t* __restrict__ offsets,
                      const int32_t* __restrict__ idx, float eps, double inv3n, float* __restrict__ pred,
                      float* __restrict__ qrec, double* __restrict__ loss_partial) {
    constexpr int cs = CS;   // CTAs per tile (a cluster when > 1); 1 compiles to the single-CTA kernel
    using Cfg = TcCfg<N>;
    constexpr int K = Cfg::K, P = Cfg::P, KS = Cfg::KS, C = Cfg::C, RT = Cfg::RT, STG = Cfg::STG;
    constexpr int kNCol = Cfg::NCOL, kA0 = Cfg::A0;
    constexpr int kTcStages = Cfg::STAGES, kPlane = Cfg::PLANE, CG = Cfg::CG, GOFF = Cfg::GOFF;
    constexpr int QS = qrec_floats(N);
    constexpr uint32_t IDESC = tc::idesc_tf32(128, kNCol);

    extern __shared__ __align__(1024) uint8_t smem[];
    uint8_t* sB = smem;                                        // [stages][hi,lo][P][128][16 B]
    float* sStage = reinterpret_cast<float*>(sB + kTcStages * 2 * P * kPlane);    // [staging][C][RT]
    float* sAval = sStage + STG * C * RT;                                   // [kARing][C][4]
    __shared__ __align__(8) uint64_t sfull[STG], sempty[STG];
    __shared__ __align__(8) uint64_t full_bar[kTcStages], empty_bar[kTcStages];
    __shared__ __align__(8) uint64_t tfull_bar[kTBuf], tempty_bar[kTBuf];
    __shared__ uint32_t s_tbase;
    __shared__ double s_loss[8];
    __shared__ float s_pp[256 * 3];

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    // cs > 1 (few tiles): a cluster of cs CTAs per tile, CTA `rank` taking the tile's chunks rank, rank + cs,
    // ...; every ring below counts the CTA's own chunks (local index c, global chunk gch(c))
    const int64_t t = CS == 1 ? (int64_t)blockIdx.x : (int64_t)(blockIdx.x / CS);
    const int rank = CS == 1 ? 0 : (int)(blockIdx.x % CS);
    const int64_t beg = offsets[t], end = offsets[t + 1];
    const int ntot = (int)((end - beg + C - 1) / C);
    const int nchunks = ntot > rank ? (ntot - rank + cs - 1) / cs : 0;
    auto gch = [&](int c) -> int64_t { return (int64_t)c * cs + rank; };
    float pp[2][3] = {{0.f, 0.f, 0.f}, {0.f, 0.f, 0.f}};   // epilogue: partial predictions (query half x RGB)

    if (tid == 0) {
        for (int s = 0; s < STG; ++s) {
            mbar_init(&sfull[s], 1);
            mbar_init(&sempty[s], kSplit);
        }
        for (int s = 0; s < kTcStages; ++s) {
            mbar_init(&full_bar[s], kSplit);
            mbar_init(&empty_bar[s], 1);
        }
        for (int b = 0; b < kTBuf; ++b) {
            mbar_init(&tfull_bar[b], 1);
            mbar_init(&tempty_bar[b], kEpiW);
        }
        fence_mbar_init();
    }
    if (warp == 1) tc::alloc(&s_tbase, 512);
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    if (warp >= kEpi0 && warp < kEpi0 + 8) {
        // A operand into TMEM: epilogue warp (half h, lane quarter q4) writes its 32 query rows,
        // xhat = [x - 1/2 | 1 | 0 ...] split hi / lo, at columns [kA0 + 2hK, +K) and [kA0 + 2hK + K, +K)
        const int h = (warp - kEpi0) >> 2, q4 = warp & 3;
        const int qi = h * 128 + q4 * 32 + lane;
        float hi[32], lo[32];
#pragma unroll
        for (int k = 0; k < 32; ++k) hi[k] = lo[k] = 0.f;
        if (qi < tile) {
#pragma unroll
            for (int d = 0; d < N; ++d) tc::split_tf32(queries[(t * tile + qi) * N + d] - 0.5f, hi[d], lo[d]);
            hi[N] = 1.f;
        }
        const uint32_t ta = s_tbase + ((uint32_t)(q4 * 32) << 16) + (uint32_t)(kA0 + h * 2 * K);
#pragma unroll
        for (int k0 = 0; k0 < K; k0 += 8) {      // K is a multiple of 8; st16 writes 16, so go by 8s
            tc::st8(ta + k0, hi + k0);
            tc::st8(ta + K + k0, lo + k0);
        }
        tc::wait_st();
    }
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t tbase = s_tbase;

    if (warp == 0 || warp >= kEpi0 + kEpiW) {      // producers: warp 0 and the warps after the epilogue
        // ------------------------------ TMA producer -------------------------------------------
        // lane g < C owns candidate g of every chunk; its index is loaded two chunks ahead so the
        // dependent idx -> record address load never sits on the chunk's critical path.
        auto load_idx = [&](int c) -> int64_t {
            const int64_t pos = beg + gch(c) * C + lane;
            return (lane < C && c < nchunks && pos < end) ? (int64_t)__ldg(idx + pos) : 0;
        };
        const int pid = warp == 0 ? 0 : warp - (kEpi0 + kEpiW) + 1;
        int64_t e0 = load_idx(pid), e1 = load_idx(pid + kProd);
        for (int c = pid; c < nchunks; c += kProd) {
            const int64_t e2 = load_idx(c + 2 * kProd);
            const int sl = c % STG;
            if (c >= STG) mbar_wait(&sempty[sl], (uint32_t)((c / STG) - 1) & 1);
            const int64_t cb = beg + gch(c) * C;
            const int n_in = (int)imin64(C, end - cb);
#ifdef NDG_TCX_HALFCOPY
            const int n_cp = min(n_in, C / 2);     // knock-out: half the gathers (wrong results)
#else
            const int n_cp = n_in;
#endif
            if (lane == 0) mbar_arrive_expect_tx(&sfull[sl], (uint32_t)(n_cp * RT * 4));
            __syncwarp();
#ifdef NDG_TCX_ONECOPY
            if (lane == 0) bulk_g2s(sStage + (sl * C) * RT, rec_tc, n_in * RT * 4, &sfull[sl]);
#else
            if (lane < n_cp) bulk_g2s(sStage + (sl * C + lane) * RT, rec_tc + e0 * RT, RT * 4, &sfull[sl]);
            if (lane == 0) NDG_TR(0, c);
#endif
            e0 = e1;
            e1 = e2;
        }
    } else if (warp == 1) {
        // ------------------------------ MMA issuer ---------------------------------------------
        if (lane == 0) {
            const uint32_t b_base = smem_u32(sB);
            for (int c = 0; c < nchunks; ++c) {
                const int s = c % kTcStages;
                mbar_wait(&full_bar[s], (uint32_t)(c / kTcStages) & 1);
                NDG_TR(3, c);
                NDG_TR(4, c);
#pragma unroll
                for (int h = 0; h < 2; ++h) {              // item (c, h) -> TMEM buffer h
                    if (c >= 1) mbar_wait(&tempty_bar[h], (uint32_t)(c - 1) & 1);
                    tc::fence_after();
                    const uint32_t d = tbase + (uint32_t)(h * kNCol);
                    const uint32_t ahi = tbase + (uint32_t)(kA0 + h * 2 * K), alo = ahi + K;
#pragma unroll
                    for (int ks = 0; ks < KS; ++ks) {
                        const uint64_t bhi = tc::smem_desc(b_base + ((s * 2 + 0) * P + 2 * ks) * kPlane, kPlane);
                        const uint64_t blo = tc::smem_desc(b_base + ((s * 2 + 1) * P + 2 * ks) * kPlane, kPlane);
                        tc::mma_tf32_ta(d, ahi + 8 * ks, bhi, IDESC, ks > 0 ? 1u : 0u);
#ifndef NDG_TCX_ONEPASS
                        tc::mma_tf32_ta(d, ahi + 8 * ks, blo, IDESC, 1u);
                        tc::mma_tf32_ta(d, alo + 8 * ks, bhi, IDESC, 1u);
#endif
                    }
                    tc::commit(&tfull_bar[h]);             // item (c, h) is ready
                }
                tc::commit(&empty_bar[s]);                 // B stage s may be refilled
                NDG_TR(5, c);
            }
        }
        __syncwarp();
    } else if (warp < kEpi0) {
        // ------------------------------ splitters ----------------------------------------------
        constexpr int NSL = kSplit * 32;
        constexpr int KU = (C * N * P + NSL - 1) / NSL;      // units per thread of a full chunk
        const int pl = (warp - 2) * 32 + lane;
        // unit u = pl + k * NSL = (gaussian g, plane p, row i): staging float offset and B-plane byte
        // offset depend only on (pl, k), so they are computed once
        int src_off[KU], dst_off[KU];
#pragma unroll
        for (int k = 0; k < KU; ++k) {
            const int u = pl + k * NSL;
            const int g = u / (N * P), rem = u - g * (N * P);
            const int p = rem / N, i = rem - p * N;
            src_off[k] = g * RT + rem * 4;
            const int row = g >= CG ? GOFF + (g - CG) * N + i : g * N + i;   // D column of (g, i)
            dst_off[k] = p * kPlane + row * 16;
        }
        for (int c = 0; c < nchunks; ++c) {
            const int sl = c % STG, s = c % kTcStages;
            const int n_in = (int)imin64(C, end - beg - gch(c) * C);
            mbar_wait(&sfull[sl], (uint32_t)(c / STG) & 1);
            if (warp == 2 && lane == 0) NDG_TR(1, c);
            const int as = c % kARing;
            // B stage s free again. This also frees colour slot `as` (last used by chunk c - kARing):
            // MMA(c - kTcStages) was issued after tempty(c - kTcStages - kTBuf), which every epilogue
            // warp arrives only after finishing chunk c - kTcStages - kTBuf - 1 >= c - kARing.
            if (c >= kTcStages) mbar_wait(&empty_bar[s], (uint32_t)((c / kTcStages) - 1) & 1);
            const float* stg = sStage + sl * C * RT;
            uint8_t* bhi = sB + (s * 2 + 0) * P * kPlane;
            uint8_t* blo = sB + (s * 2 + 1) * P * kPlane;
#ifndef NDG_TCX_NOSPLIT
            // records are plane-major ([p][i][4]): consecutive lanes read consecutive 16-B staging
            // units and write consecutive rows of one plane -> both conflict-free
            auto split_store = [&](int k, const float4& v) {
                float4 hi, lo;
                tc::split_tf32(v.x, hi.x, lo.x);
                tc::split_tf32(v.y, hi.y, lo.y);
                tc::split_tf32(v.z, hi.z, lo.z);
                tc::split_tf32(v.w, hi.w, lo.w);
                *reinterpret_cast<float4*>(bhi + dst_off[k]) = hi;
                *reinterpret_cast<float4*>(blo + dst_off[k]) = lo;
            };
            if (n_in == C) {      // full chunk: all loads in flight before the first split
                constexpr int kLast = C * N * P - (KU - 1) * NSL;   // threads active in the last round
                float4 v[KU];
#pragma unroll
                for (int k = 0; k < KU; ++k)
                    if (k < KU - 1 || pl < kLast) v[k] = *reinterpret_cast<const float4*>(stg + src_off[k]);
#pragma unroll
                for (int k = 0; k < KU; ++k)
                    if (k < KU - 1 || pl < kLast) split_store(k, v[k]);
            } else {
                const int n_units = n_in * N * P;
#pragma unroll
                for (int k = 0; k < KU; ++k) {
                    if (pl + k * NSL >= n_units) break;
                    split_store(k, *reinterpret_cast<const float4*>(stg + src_off[k]));
                }
            }
#endif
            for (int u = pl; u < n_in; u += NSL)
                *reinterpret_cast<float4*>(sAval + (as * C + u) * 4) =
                    *reinterpret_cast<const float4*>(stg + u * RT + N * K);
            fence_proxy_async();
            __syncwarp();
            if (lane == 0) {
                mbar_arrive(&full_bar[s]);
                if (warp == 2) NDG_TR(2, c);
                mbar_arrive(&sempty[sl]);
            }
        }
    } else {
        // ------------------------------ epilogue -----------------------------------------------
        // warp (wh, q4): TMEM lane quarter q4, Gaussian group wh of both halves' items; pp[hh] is the
        // partial prediction of the thread's query in half hh (group 1 hands its partials to group 0
        // at tile end).
        const int wh = (warp - kEpi0) >> 2, q4 = warp & 3;
        constexpr int NGW = CG;                         // Gaussian slots per warp per item
        constexpr int NLD = (NGW * N + 15) / 16;
        constexpr int NIT = 2;                          // items per chunk
        const int g0 = wh * CG;
        const int ngw = wh ? C - CG : CG;
        for (int c = 0; c < nchunks; ++c) {
            const int as = c % kARing;
            const int n_in = (int)imin64(C, end - beg - gch(c) * C);
#pragma unroll
            for (int it = 0; it < NIT; ++it) {
                const int b = it;
                mbar_wait(&tfull_bar[b], (uint32_t)c & 1);
                if (warp == kEpi0 && lane == 0 && it == 0) NDG_TR(6, c);
                tc::fence_after();
                float v[NLD * 16];
                const uint32_t col = (uint32_t)(it * kNCol + wh * GOFF);
                const uint32_t ta = tbase + ((uint32_t)(q4 * 32) << 16) + col;
#ifdef NDG_TCX_NOLD
                for (int j = 0; j < NLD * 16; ++j) v[j] = (float)(ta + j);
#else
#pragma unroll
                for (int j = 0; j < NLD; ++j) tc::ld16(ta + 16 * j, v + 16 * j);
                tc::wait_ld();
#endif
                tc::fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&tempty_bar[b]);      // TMEM buffer b may be overwritten
                if (warp == kEpi0 && lane == 0 && it == 0) NDG_TR(7, c);
#ifndef NDG_TCX_NOEPI
                auto gauss = [&](int gl) {
                    float sum;
                    if constexpr ((N & 1) == 0) {
                        float2 acc = make_float2(0.f, 0.f);
#pragma unroll
                        for (int i = 0; i < N; i += 2) {
                            const float2 zz = make_float2(v[gl * N + i], v[gl * N + i + 1]);
                            acc = __ffma2_rn(zz, zz, acc);
                        }
                        sum = acc.x + acc.y;
                    } else {
                        sum = 0.f;
#pragma unroll
                        for (int i = 0; i < N; ++i) sum = fmaf(v[gl * N + i], v[gl * N + i], sum);
                    }
                    const float gv = ex2_neg(sum);
                    const float4 av = *reinterpret_cast<const float4*>(sAval + (as * C + g0 + gl) * 4);
                    pp[it][0] = fmaf(gv, av.x, pp[it][0]);
                    pp[it][1] = fmaf(gv, av.y, pp[it][1]);
                    pp[it][2] = fmaf(gv, av.z, pp[it][2]);
                };
                if (n_in == C && C == 2 * CG) {       // full chunk: no per-Gaussian predicates
#pragma unroll
                    for (int gl = 0; gl < NGW; ++gl) gauss(gl);
                } else {
#pragma unroll
                    for (int gl = 0; gl < NGW; ++gl)
                        if (gl < ngw && g0 + gl < n_in) gauss(gl);
                }
#else
                pp[it][0] += v[0] + v[NLD * 16 - 1];
#endif
            }
            if (warp == kEpi0 && lane == 0) NDG_TR(8, c);
            if (warp == kEpi0 + 7 && lane == 0) NDG_TR(9, c);
        }
        {                            // fold group 1's partial predictions into group 0
            if (wh == 1)
#pragma unroll
                for (int hh = 0; hh < 2; ++hh)
#pragma unroll
                    for (int ch = 0; ch < 3; ++ch) s_pp[(hh * 128 + q4 * 32 + lane) * 3 + ch] = pp[hh][ch];
            asm volatile("bar.sync 1, %0;" ::"r"(kEpiW * 32) : "memory");
            if (wh == 0)
#pragma unroll
                for (int hh = 0; hh < 2; ++hh)
#pragma unroll
                    for (int ch = 0; ch < 3; ++ch) pp[hh][ch] += s_pp[(hh * 128 + q4 * 32 + lane) * 3 + ch];
        }
        if (cs > 1 && rank > 0 && wh == 0)          // publish this CTA's partials for the cluster's rank 0
#pragma unroll
            for (int hh = 0; hh < 2; ++hh)
#pragma unroll
                for (int ch = 0; ch < 3; ++ch) s_pp[(hh * 128 + q4 * 32 + lane) * 3 + ch] = pp[hh][ch];
    }
    if (cs > 1) {
        cluster_sync();                               // every rank's partials are in its s_pp
        if (rank == 0 && warp >= kEpi0 && warp < kEpi0 + 4) {
            const int q4 = warp & 3;
            for (int r = 1; r < cs; ++r)              // fixed rank order: deterministic sums
#pragma unroll
                for (int hh = 0; hh < 2; ++hh)
#pragma unroll
                    for (int ch = 0; ch < 3; ++ch)
                        pp[hh][ch] += ld_cluster_f32(&s_pp[(hh * 128 + q4 * 32 + lane) * 3 + ch], r);
        }
        cluster_sync();                               // the remote reads are done: ranks > 0 may leave
    }
    if (rank == 0 && warp >= kEpi0 && warp < kEpi0 + kEpiW) {
        const int wh = (warp - kEpi0) >> 2, q4 = warp & 3;
        constexpr int NIT = 2;
        // tile end: pred, rel-L2 loss, backward query records (group 0 finishes both halves' queries)
        double loss_acc = 0.0;
#pragma unroll
        for (int hh = 0; hh < NIT; ++hh) {
            const int qi = hh * 128 + q4 * 32 + lane;
            if (wh == 0 && qi < tile) {
                const int64_t bq = t * tile + qi;
                pred[bq * 3] = pp[hh][0];
                pred[bq * 3 + 1] = pp[hh][1];
                pred[bq * 3 + 2] = pp[hh][2];
                if (targets) {
                    float* qr = qrec + bq * QS;
                    double ell = 0.0;
#pragma unroll
                    for (int ch = 0; ch < 3; ++ch) {
                        const double pv = pp[hh][ch], dv = pv - (double)targets[bq * 3 + ch], den = pv * pv + (double)eps;
                        ell += dv * dv / den;
                        qr[N + ch] = (float)(2.0 * dv / den * inv3n);
                    }
                    ell *= inv3n;
#pragma unroll
                    for (int d = 0; d < N; ++d) qr[d] = queries[bq * N + d];
                    qr[N + 3] = (float)ell;
#pragma unroll
                    for (int d = N + 4; d < QS; ++d) qr[d] = 0.f;
                    loss_acc += ell;
                }
            }
        }
        if (targets) {
#pragma unroll
            for (int o = 16; o; o >>= 1) loss_acc += __shfl_xor_sync(0xffffffffu, loss_acc, o);
            if (lane == 0) s_loss[warp - kEpi0] = loss_acc;
        }
    }
    tc::fence_before();
    __syncthreads();
    if (targets && tid == 0 && rank == 0) {
        double sl = 0.0;
        for (int w = 0; w < 8; ++w) sl += s_loss[w];
        loss_partial[t] = sl;
    }
    if (warp == 1) {
        tc::fence_after();
        tc::dealloc(tbase, 512);
    }
}

template <int N>
int launch_forward_tc(int64_t B, int tile, const float* q, const float* tgt, const float* rec_tc, const int64_t* off,
                      const int32_t* idx, float eps, int64_t n_total, float* pred, float* qrec, double* lp,
                      cudaStream_t st) {
    const int64_t T = B / tile;
    const size_t smem = tc_smem_bytes<N>();
    static DeviceOnce attr;
    if (attr.first()) {
        cudaFuncSetAttribute(forward_tc_kernel<N, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        cudaFuncSetAttribute(forward_tc_kernel<N, kMaxCluster>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    }
    const double inv3n = 1.0 / (3.0 * (double)n_total);
    // few tiles (T < 148, e.g. cfg1's 64): a cluster of cs CTAs per tile splits its chunks so every SM works
    const int cs = T * kMaxCluster <= 148 ? kMaxCluster : 1;
    if (cs == 1) {
        forward_tc_kernel<N, 1><<<(unsigned)T, kTcThreads, smem, st>>>(tile, q, tgt, rec_tc, off, idx, eps, inv3n, pred,
                                                                       qrec, lp);
    } else {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3((unsigned)(T * kMaxCluster));
        cfg.blockDim = dim3(kTcThreads);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = st;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = (unsigned)kMaxCluster;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        cudaLaunchKernelEx(&cfg, forward_tc_kernel<N, kMaxCluster>, tile, q, tgt, rec_tc, off, idx, eps, inv3n, pred,
                           qrec, lp);
    }
    NDG_CHECK_LAUNCH();
    return NDG_OK;
}

// Ahat records for the tensor-core pair kernels: one per evaluated Gaussian, N rows x K floats stored
// plane-major ([K/4][N][4], the order the B operand's planes need), then a[3] and a pad;
// row i = [C (L^-1)_i0 .. C (L^-1)_i,N-1 | C (L^-1 (1/2 - m))_i | 0 ...], computed in float64 from
// K1's activated / composed factor (forward substitution on the identity, never forming V^-1).
//
// Conditioning (cond, optional, 3 doubles zeroed by the caller): B_e = max_i (1/2 sum_k<N |Ahat_ik| +
// |Ahat_iN|) bounds the magnitude of the terms the z-GEMM adds for any query in [0,1]^N
// (|x - 1/2| <= 1/2). z~ itself is O(1) where g matters, so the fp32-accumulated 3xTF32 GEMM loses
// ~1e-7 * B_e absolute to cancellation. cond = [max_e B_e, sum_e B_e^2, count] over live,
// non-degenerate e; the host compares the RMS with the measured-safe bound (engine.py) and evaluates
// the step on the FP32 pipe when it is exceeded (very sharp mixtures, sigma ~ 1e-3).
__global__ void tc_records_kernel(int n, int64_t Gev, const double* __restrict__ mean64,
                                  const double* __restrict__ chol64, const uint8_t* __restrict__ eflags,
                                  const float* __restrict__ rec, float* __restrict__ rec_tc,
                                  double* __restrict__ cond) {
    const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    double b = -1.0;                                  // this Gaussian's B_e (< 0: not counted)
    if (e < Gev) {
        const int P = n_chol(n), K = tc_k(n), RT = tc_rec_floats(n);
        float4* out4 = reinterpret_cast<float4*>(rec_tc + e * RT);   // RT is a multiple of 4
        const bool live = eflags[e] & 1;
        double W[n_chol(NMAX)];
        if (live) {
            double L[n_chol(NMAX)];
            for (int t = 0; t < P; ++t) L[t] = chol64[e * P + t];
            for (int j = 0; j < n; ++j)                 // W = L^-1 (lower), column by column
                for (int i = j; i < n; ++i) {
                    double acc = (i == j) ? 1.0 : 0.0;
                    for (int k = j; k < i; ++k) acc -= L[tri(i, k)] * W[tri(k, j)];
                    W[tri(i, j)] = acc / L[tri(i, i)];
                }
        }
        // plane-major rows: element (row i, column k) at ((k / 4) * n + i) * 4 + k % 4, written as one
        // 16-B store per (plane, row); columns past the row's diagonal (but the bias at k = n) are 0
        double bound = 0.0;
        for (int i = 0; i < n; ++i) {
            double bias = 0.0, lin = 0.0;
            float row[NMAX + 8];
            for (int k = 0; k < K; ++k) row[k] = 0.f;
            if (live) {
                for (int j = 0; j <= i; ++j) {
                    const double w = kC * W[tri(i, j)];
                    row[j] = (float)w;
                    bias += w * (0.5 - mean64[e * n + j]);
                    lin += fabs(w);
                }
                row[n] = (float)bias;
                bound = fmax(bound, 0.5 * lin + fabs(bias));
            }
            for (int p = 0; p < K / 4; ++p)
                out4[p * n + i] = make_float4(row[4 * p], row[4 * p + 1], row[4 * p + 2], row[4 * p + 3]);
        }
        const float* ra = rec + e * rec_floats(n) + rec_a(n);
        out4[n * K / 4] = live ? make_float4(ra[0], ra[1], ra[2], 0.f) : make_float4(0.f, 0.f, 0.f, 0.f);   // colour a
        if (live && !(eflags[e] & 2)) b = isfinite(bound) ? bound : 1.0e300;
    }
    if (cond) {
        // warp-reduce [max, sum of squares, count] first: one set of atomics per warp, not per Gaussian
        // (same-address atomics serialise in L2; positive doubles order like their bit patterns)
        unsigned long long mx = b >= 0.0 ? (unsigned long long)__double_as_longlong(b) : 0ull;
        double ss = b >= 0.0 ? b * b : 0.0, cnt = b >= 0.0 ? 1.0 : 0.0;
#pragma unroll
        for (int o = 16; o; o >>= 1) {
            const unsigned long long m2 = __shfl_xor_sync(0xffffffffu, mx, o);
            mx = m2 > mx ? m2 : mx;
            ss += __shfl_xor_sync(0xffffffffu, ss, o);
            cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
        }
        if ((threadIdx.x & 31) == 0 && cnt > 0.0) {
            atomicMax(reinterpret_cast<unsigned long long*>(cond), mx);
            atomicAdd(cond + 1, ss);
            atomicAdd(cond + 2, cnt);
        }
    }
}

}  // namespace

#ifdef NDG_TCX_TRACE
extern "C" int ndg_trace_dump(long long* out) {
    return cudaMemcpyFromSymbol(out, g_trace, sizeof(long long) * kTrC * kTrEv) == cudaSuccess ? 0 : -3;
}
#endif

extern "C" int ndg_tc_records(int n, int64_t Gev, const double* mean64, const double* chol64, const uint8_t* eflags,
                              const float* rec, float* rec_tc, double* cond, void* stream) {
    if (!ndg_supported_dims(n)) return NDG_ERR_UNSUPPORTED_DIMS;
    if (Gev == 0) return NDG_OK;
    const int threads = spread_threads(Gev, 128);
    tc_records_kernel<<<(unsigned)((Gev + threads - 1) / threads), threads, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
        n, Gev, mean64, chol64, eflags, rec, rec_tc, cond);
    NDG_CHECK_LAUNCH();
    return NDG_OK;
}

extern "C" int ndg_forward_tc(int n, int64_t B, int tile, const float* queries, const float* targets,
                              const float* rec_tc, const int64_t* offsets, const int32_t* idx, float eps,
                              int64_t n_total, float* pred, float* qrec, double* loss_partial, void* stream) {
    NDG_REQUIRE(tile >= 1 && tile <= 256 && B % tile == 0, "tensor-core forward needs tile in 1..256 dividing B");
    NDG_REQUIRE(!targets || (qrec && loss_partial && n_total > 0), "targets need qrec, loss_partial, n_total");
    if (B == 0) return NDG_OK;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    switch (n) {
#define NDG_CASE(NN)                                                                                             \
    case NN:                                                                                                     \
        return launch_forward_tc<NN>(B, tile, queries, targets, rec_tc, offsets, idx, eps, n_total, pred, qrec, \
                                     loss_partial, st);
        NDG_CASE(1) NDG_CASE(2) NDG_CASE(3) NDG_CASE(4) NDG_CASE(5) NDG_CASE(6) NDG_CASE(7) NDG_CASE(8)
        NDG_CASE(9) NDG_CASE(10) NDG_CASE(11) NDG_CASE(12) NDG_CASE(13) NDG_CASE(14) NDG_CASE(15) NDG_CASE(16)
#undef NDG_CASE
        default:
            return NDG_ERR_UNSUPPORTED_DIMS;
    }
}
