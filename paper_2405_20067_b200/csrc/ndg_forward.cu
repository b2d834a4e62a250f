// K5+K6 fused forward + loss (sm_100a, FP32 pipe).
//
// Replaces eval_mixture at every query over its tile's candidate list (Eq. 8,
// PAPER.md:368-371) plus loss_rel_l2. Query-stationary mapping: one CTA per tile,
// each thread owns kQPT queries in registers; the tile's candidate records are streamed through a
// double-buffered shared-memory ring, each record brought in by one 1-D bulk copy on the TMA engine
// (cp.async.bulk + mbarrier complete_tx), and read back as warp-uniform LDS.128 broadcasts. Per pair:
//   z~_i = fma(rho_i, x_i, nb_i) + sum_{j<i} nlu_ij z~_j      (forward substitution)
//   s~ = |z~|^2,  g = ex2(-s~) = exp(-|z|^2/2),  pred += g * a
// i.e. N + N(N-1)/2 + N FFMA, one MUFU.EX2 and 3 FFMA: the whole per-pair cost is FP32-pipe issue.
// When targets are given the CTA finishes the tile with the relative-L2 loss: dpred, each query's
// loss share, the backward query record (x | dpred | ell) and a per-tile float64 loss partial.
#include "ndg_common.cuh"

using namespace ndg;

namespace {

#ifndef NDG_FWD_CHUNK
#define NDG_FWD_CHUNK 16
#endif
#ifndef NDG_FWD_STAGES
#define NDG_FWD_STAGES 4
#endif
constexpr int kChunk = NDG_FWD_CHUNK;       // candidate records per ring stage (one per lane of warp 0)

// Launch shape per N: QPT queries per thread x NT threads = 256 queries per pass (one tile).
#ifndef NDG_FWD_QPT
#define NDG_FWD_QPT 4
#endif
template <int N> struct FwdCfg { static constexpr int QPT = NDG_FWD_QPT, NT = 256 / NDG_FWD_QPT, STAGES = NDG_FWD_STAGES; };
template <> struct FwdCfg<11> { static constexpr int QPT = 2, NT = 128, STAGES = 4; };
template <> struct FwdCfg<12> { static constexpr int QPT = 2, NT = 128, STAGES = 4; };
template <> struct FwdCfg<13> { static constexpr int QPT = 2, NT = 128, STAGES = 4; };
template <> struct FwdCfg<14> { static constexpr int QPT = 2, NT = 128, STAGES = 3; };
template <> struct FwdCfg<15> { static constexpr int QPT = 2, NT = 128, STAGES = 3; };
template <> struct FwdCfg<16> { static constexpr int QPT = 2, NT = 128, STAGES = 3; };

// Ring protocol (no CTA-wide barrier in the loop): full[s] completes when the TMA engine has
// landed the stage's records (expect_tx by lane 0 of warp 0); empty[s] completes when every warp
// has finished reading the stage (one arrive per warp). Only warp 0 (the producer) ever waits on
// empty[s], just before refilling it; consumer warps never wait on each other.
template <int N, int QPT, int NT, int STAGES, bool CTR>
__global__ void __launch_bounds__(NT)
    forward_kernel(int tile, const float* __restrict__ queries, const float* __restrict__ targets,
                   const float* __restrict__ rec, const int64_t* __restrict__ offsets,
                   const int32_t* __restrict__ idx, float eps, double inv3n, float* __restrict__ pred,
                   float* __restrict__ qrec, double* __restrict__ loss_partial) {
    constexpr int RS = rec_floats(N);
    constexpr int QS = qrec_floats(N);
    constexpr int A0 = rec_a(N);
    constexpr int NW = NT / 32;
    extern __shared__ __align__(128) float s_rec[];           // [STAGES][kChunk][RS]
    __shared__ __align__(8) uint64_t full_bar[STAGES], empty_bar[STAGES];
    __shared__ double s_loss[NW];

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t t = blockIdx.x;
    const int64_t beg = offsets[t], end = offsets[t + 1];
    const int nchunks = (int)((end - beg + kChunk - 1) / kChunk);

    if (tid == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full_bar[s], 1);
            mbar_init(&empty_bar[s], NW);
        }
        fence_mbar_init();
    }
    __syncthreads();

    // producer (warp 0): lane l copies candidate l of chunk c into stage s
    auto issue = [&](int c, int s) {
        const int64_t cb = beg + (int64_t)c * kChunk;
        const int n_in = (int)imin64(kChunk, end - cb);
        if (lane == 0) mbar_arrive_expect_tx(&full_bar[s], (uint32_t)(n_in * RS * 4));
        __syncwarp();
        if (lane < n_in) {
            const int64_t e = idx[cb + lane];
            bulk_g2s(s_rec + (s * kChunk + lane) * RS, rec + e * RS, RS * 4, &full_bar[s]);
        }
    };

    double loss_acc = 0.0;
    uint32_t ring = 0;   // ring position across passes (stage = ring % STAGES, parity = ring / STAGES)
    for (int q0 = 0; q0 < tile; q0 += NT * QPT) {
        // queries j and j + QPT/2 of this thread form packed pair jp: x2[jp][d] = (x_j[d], x_{j+QPT/2}[d])
        constexpr int NP = QPT / 2;
        float2 x2[NP][N], p2[NP][3];
        bool valid[QPT];
#pragma unroll
        for (int j = 0; j < QPT; ++j) {
            const int qi = q0 + tid + j * NT;
            valid[j] = qi < tile;
            const float* src = queries + (t * tile + qi) * N;
#pragma unroll
            for (int d = 0; d < N; ++d) {
                const float v = valid[j] ? src[d] : 0.f;
                if (j < NP) x2[j][d].x = v;
                else x2[j - NP][d].y = v;
            }
        }
#pragma unroll
        for (int jp = 0; jp < NP; ++jp) p2[jp][0] = p2[jp][1] = p2[jp][2] = make_float2(0.f, 0.f);
        if (warp == 0) {
            for (int c = 0; c < STAGES && c < nchunks; ++c) {
                const uint32_t pos = ring + c;
                if (pos >= STAGES) mbar_wait(&empty_bar[pos % STAGES], ((pos / STAGES) - 1) & 1);
                issue(c, (int)(pos % STAGES));
            }
        }
        for (int c = 0; c < nchunks; ++c) {
            const uint32_t pos = ring + c;
            const int s = (int)(pos % STAGES);
            mbar_wait(&full_bar[s], (pos / STAGES) & 1);
            const int n_in = (int)imin64(kChunk, end - beg - (int64_t)c * kChunk);
            const float4* r4 = reinterpret_cast<const float4*>(s_rec + s * kChunk * RS);
            for (int ci = 0; ci < n_in; ++ci, r4 += RS / 4) {   // pointer bump: no IMAD on the FMA pipe
                float r[RS];
#pragma unroll
                for (int v = 0; v < RS / 4; ++v) {
                    const float4 w = r4[v];
                    r[4 * v] = w.x;
                    r[4 * v + 1] = w.y;
                    r[4 * v + 2] = w.z;
                    r[4 * v + 3] = w.w;
                }
#pragma unroll
                for (int jp = 0; jp < NP; ++jp) {
                    // two queries per FFMA2: the record coefficient is the broadcast scalar operand
                    float2 z[N];
                    float2 s2 = make_float2(0.f, 0.f);
#pragma unroll
                    for (int i = 0; i < N; ++i) {
                        float2 acc;
                        if constexpr (CTR) {   // centred records: slots (m_hi, m_lo), z = rho ((x - m_hi) - m_lo)
                            const float2 d = __fadd2_rn(__fadd2_rn(x2[jp][i], make_float2(-r[rec_nb2(N) + 2 * i], -r[rec_nb2(N) + 2 * i])),
                                                        make_float2(-r[rec_nb2(N) + 2 * i + 1], -r[rec_nb2(N) + 2 * i + 1]));
                            acc = __fmul2_rn(make_float2(r[rec_rho(N) + i], r[rec_rho(N) + i]), d);
                        } else {
                            acc = __ffma2_rn(make_float2(r[rec_rho(N) + i], r[rec_rho(N) + i]), x2[jp][i],
                                             make_float2(r[rec_nb2(N) + 2 * i], r[rec_nb2(N) + 2 * i + 1]));
                        }
#pragma unroll
                        for (int k = 0; k < i; ++k)
                            acc = __ffma2_rn(make_float2(r[rec_l(N, i, k)], r[rec_l(N, i, k)]), z[k], acc);
                        z[i] = acc;
                        s2 = __ffma2_rn(acc, acc, s2);
                    }
                    const float2 g = make_float2(ex2_neg(s2.x), ex2_neg(s2.y));
#pragma unroll
                    for (int ch = 0; ch < 3; ++ch)
                        p2[jp][ch] = __ffma2_rn(make_float2(r[A0 + ch], r[A0 + ch]), g, p2[jp][ch]);
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty_bar[s]);       // this warp is done with stage s
            if (warp == 0 && c + STAGES < nchunks) {
                mbar_wait(&empty_bar[s], (pos / STAGES) & 1);  // all warps done with stage s
                issue(c + STAGES, s);
            }
        }
        float p[QPT][3], x[QPT][N];
#pragma unroll
        for (int j = 0; j < QPT; ++j) {
#pragma unroll
            for (int ch = 0; ch < 3; ++ch) p[j][ch] = j < NP ? p2[j][ch].x : p2[j - NP][ch].y;
#pragma unroll
            for (int d = 0; d < N; ++d) x[j][d] = j < NP ? x2[j][d].x : x2[j - NP][d].y;
        }
        ring += (uint32_t)nchunks;

#pragma unroll
        for (int j = 0; j < QPT; ++j) {
            if (!valid[j]) continue;
            const int64_t b = t * tile + q0 + tid + j * NT;
            pred[b * 3] = p[j][0];
            pred[b * 3 + 1] = p[j][1];
            pred[b * 3 + 2] = p[j][2];
            if (targets) {
                float* qr = qrec + b * QS;
                double ell = 0.0;
#pragma unroll
                for (int ch = 0; ch < 3; ++ch) {
                    const double pv = p[j][ch], dv = pv - (double)targets[b * 3 + ch], den = pv * pv + (double)eps;
                    ell += dv * dv / den;
                    qr[N + ch] = (float)(2.0 * dv / den * inv3n);
                }
                ell *= inv3n;
#pragma unroll
                for (int d = 0; d < N; ++d) qr[d] = x[j][d];
                qr[N + 3] = (float)ell;
#pragma unroll
                for (int d = N + 4; d < QS; ++d) qr[d] = 0.f;
                loss_acc += ell;
            }
        }
    }
    if (targets) {   // fixed-order block reduction -> per-tile partial (deterministic)
#pragma unroll
        for (int o = 16; o; o >>= 1) loss_acc += __shfl_xor_sync(0xffffffffu, loss_acc, o);
        if (lane == 0) s_loss[warp] = loss_acc;
        __syncthreads();
        if (tid == 0) {
            double s = 0.0;
            for (int w = 0; w < NW; ++w) s += s_loss[w];
            loss_partial[t] = s;
        }
    }
}

template <int N>
int launch_forward(int64_t B, int tile, const float* q, const float* tgt, const float* rec, int centred,
                   const int64_t* off, const int32_t* idx, float eps, int64_t n_total, float* pred, float* qrec,
                   double* lp, cudaStream_t st) {
    using C = FwdCfg<N>;
    const int64_t T = B / tile;
    const size_t smem = sizeof(float) * C::STAGES * kChunk * rec_floats(N);
    auto kern = centred ? forward_kernel<N, C::QPT, C::NT, C::STAGES, true> : forward_kernel<N, C::QPT, C::NT, C::STAGES, false>;
    static DeviceOnce attr;
    if (attr.first()) {
        cudaFuncSetAttribute(forward_kernel<N, C::QPT, C::NT, C::STAGES, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        cudaFuncSetAttribute(forward_kernel<N, C::QPT, C::NT, C::STAGES, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    }
    kern<<<(unsigned)T, C::NT, smem, st>>>(tile, q, tgt, rec, off, idx, eps, 1.0 / (3.0 * (double)n_total), pred,
                                           qrec, lp);
    NDG_CHECK_LAUNCH();
    return NDG_OK;
}

}  // namespace

extern "C" int ndg_forward(int n, int64_t B, int tile, const float* queries, const float* targets, const float* rec,
                           int centred, const int64_t* offsets, const int32_t* idx, float eps, int64_t n_total,
                           float* pred, float* qrec, double* loss_partial, void* stream) {
    NDG_REQUIRE(tile >= 1 && tile <= 1024 && B % tile == 0, "tile must be in 1..1024 and divide B");
    NDG_REQUIRE(!targets || (qrec && loss_partial && n_total > 0), "targets need qrec, loss_partial, n_total");
    if (B == 0) return NDG_OK;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    switch (n) {
#define NDG_CASE(NN) \
    case NN:         \
        return launch_forward<NN>(B, tile, queries, targets, rec, centred, offsets, idx, eps, n_total, pred, qrec, \
                                  loss_partial, st);
        NDG_CASE(1) NDG_CASE(2) NDG_CASE(3) NDG_CASE(4) NDG_CASE(5) NDG_CASE(6) NDG_CASE(7) NDG_CASE(8)
        NDG_CASE(9) NDG_CASE(10) NDG_CASE(11) NDG_CASE(12) NDG_CASE(13) NDG_CASE(14) NDG_CASE(15) NDG_CASE(16)
#undef NDG_CASE
        default:
            return NDG_ERR_UNSUPPORTED_DIMS;
    }
}
