/*
 * ndg.h -- C ABI of libndg.so, the B200 (sm_100a) kernels of the culled N-D Gaussian-mixture hot path.
 *
 * This library takes the slot of the reference's compiled inner-loop module `ndgauss.kernels._core`
 * (/root/reference/pkg/setup.py:32-53: Cython -> C + OpenMP, selected at import time, source absent)
 * behind the reference package's module-level operations. The
 * reference never published `_core`'s signatures, so each entry point below names the SPEC
 * operation it replaces; INTEGRATION.md shows the ctypes binding `ndgauss/kernels/__init__.py`
 * would add.
 *
 * Conventions (all entry points):
 *   - Every pointer is a DEVICE pointer owned by the caller (PyTorch tensors in the Python host).
 *     The library never allocates device memory; sizes come from ndg_*_floats / _doubles below.
 *   - `stream` is a cudaStream_t; work is enqueued on it and the call returns without syncing.
 *   - Return value: NDG_OK (0) or a negative launch/argument error (see ndg_last_error()).
 *     Data errors (non-finite raw parameters, non-finite gradients) are written to the device
 *     `ndg_status` and read back by the host once per step; they map 1:1 onto the reference's
 *     exception classes InvalidParameterError / NonFiniteGradientError
 *     (/root/reference/pkg/src/ndgauss/errors.py:8-33).
 *   - Layouts (row-major, float32 unless noted):
 *       raw component row  : mean_raw[N] | chol_raw[P] | color_raw[3] | amp_raw[1]   (
 *                            chol_raw is the row-major lower packing of SPEC.md:31, P = N(N+1)/2)
 *       raw child row      : rel_mean_raw[N] | rel_chol_raw[P] | color_raw[3] | amp_raw
 *       component flags    : uint8, bit0 = has live child, bit1 = frozen
 *       evaluated index e  : e < G is parent e; G <= e < 2G is the child of component e - G
 *       projection vectors : float64 [k][N]
 *       projected bounds   : float64 [k][Gev]; tile bounds float64 [T][k]
 *       candidate lists    : CSR, offsets int64 [T+1], indices int32 ascending per tile
 *   - Supported N: 1..16 (ndg_supported_dims). Tile size: 1..1024 queries.
 */
#ifndef NDG_H
#define NDG_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define NDG_ABI_VERSION 1

enum ndg_error {
    NDG_OK = 0,
    NDG_ERR_INVALID_PARAMETER = 1,    /* data error: non-finite raw parameter       */
    NDG_ERR_NONFINITE_GRADIENT = 2,   /* data error: non-finite gradient           */
    NDG_ERR_BAD_ARGUMENT = -1,        /* launch error: invalid sizes / pointers                  */
    NDG_ERR_UNSUPPORTED_DIMS = -2,    /* launch error: N outside 1..16                           */
    NDG_ERR_CUDA = -3                 /* launch error: CUDA runtime failure                      */
};

enum ndg_block { NDG_BLOCK_MEAN = 0, NDG_BLOCK_CHOL = 1, NDG_BLOCK_COLOR = 2, NDG_BLOCK_AMP = 3 };
enum ndg_amp_mode { NDG_BRIGHTNESS = 0, NDG_OPACITY = 1 };

/*
 * Device-side status word (zero-initialised by the caller before a step). Offenders are recorded
 * deterministically as the lowest key = which * G * R + component * R + entry (which: 0 parent row,
 * 1 child row; R = ndg_raw_floats(N)), stored as INT64_MAX - key (0 = no error) so that an atomicMax
 * on zero-initialised memory keeps the lowest key. The host decodes component / block / entry.
 */
typedef struct ndg_status {
    int64_t invalid_key;    /* non-finite raw parameter -> InvalidParameterError      */
    int64_t nonfinite_key;  /* non-finite gradient     -> NonFiniteGradientError     */
    int64_t n_degenerate;   /* live Gaussians flagged degenerate this step       */
    int64_t reserved;
} ndg_status;

int ndg_abi_version(void);
const char* ndg_last_error(void);
int ndg_supported_dims(int n);
int ndg_raw_floats(int n);        /* N + P + 4                                       */
int ndg_record_floats(int n);     /* evaluation record stride (float32, 16-B multiple) */
int ndg_query_floats(int n);      /* backward query record stride: x[N] | dpred[3] | ell */
int ndg_accum_doubles(int n);     /* accumulator stride: S[P] | t[N] | flag | gA[3] | stats[3] */
int ndg_num_stats(void);          /* density-control statistics per evaluated Gaussian (3) */
int ndg_backward_chunk(void);     /* candidates per backward work item (chunk_offsets unit) */

/*
 * K1 prologue. Replaces activate_cholesky + compose_child + the colour/amplitude activations
 * (SPEC.md:63-71, 93-101, 86). Writes per evaluated Gaussian the float32 evaluation record,
 * the float64 mean and packed lower factor (composed for children), and eflags
 * (bit0 live, bit1 degenerate). Non-finite raw values -> status INVALID_PARAMETER.
 */
int ndg_prologue(int n, int64_t G, int64_t Gev, int amp_mode, const float* params, const float* child,
                 const uint8_t* flags, float* rec, double* mean64, double* chol64, uint8_t* eflags,
                 ndg_status* status, void* stream);

/* K2 projected bounds. Replaces project_components: m_r = m.r, s_r = ||L^T r||
 * (FP64, sequential, no FMA); thr = multiplier * s_r, or -1 for non-live Gaussians. */
int ndg_project(int n, int64_t Gev, const double* mean64, const double* chol64, const uint8_t* eflags,
                const double* dirs, int k, double multiplier, double* m_r, double* s_r, double* thr, void* stream);

/* K3 tile bounds. Replaces TileBounds construction. */
int ndg_tile_bounds(int n, int64_t B, int tile, const float* queries, const double* dirs, int k, double* lo,
                    double* hi, void* stream);

/* K4a binning, phase 1. cull_tile for every tile: bit-mask [T][ceil(Gev/32)]
 * of kept candidates (warp ballot) and counts[T] (must be zeroed by the caller). 1 <= k <= 256. */
int ndg_cull_mask(int64_t T, int k, int64_t Gev, const double* lo, const double* hi, const double* m_r,
                  const double* thr, uint32_t* mask, int64_t* counts, void* stream);

/* K4a with a bucket pre-filter (the north_star's hash bucketing): live Gaussians
 * are bucketed on a 64 x 64 grid over their projections on vectors 0 and 1; a tile runs the exact K4a
 * test only on the Gaussians of the cells its intervals can reach, so the mask and counts are
 * bit-identical to ndg_cull_mask's. A device-side plan (summed-area table of the cell populations)
 * picks the pre-filtered or the dense pass per call (mode 0; 1 forces the pre-filter, 2 the dense
 * pass); the other pass's kernels exit at once. workspace: ndg_cull_prefilter_workspace(Gev, k)
 * bytes, no initialisation needed; counts zeroed by the caller; 2 <= k <= 256. */
int64_t ndg_cull_prefilter_workspace(int64_t Gev, int k);
int ndg_cull_prefilter(int64_t T, int k, int64_t Gev, const double* lo, const double* hi, const double* m_r,
                       const double* thr, int mode, void* workspace, uint32_t* mask, int64_t* counts, void* stream);

/* K4b exclusive scan of counts -> offsets[T+1] and backward work-item offsets[T+1]
 * (ceil(count / ndg_backward_chunk()) per tile). */
int ndg_scan_counts(int64_t T, const int64_t* counts, int64_t* offsets, int64_t* chunk_offsets, void* stream);

/* K4c compaction of the mask into ascending CSR indices (prefix scan of popcounts). */
int ndg_cull_compact(int64_t T, int64_t Gev, const uint32_t* mask, const int64_t* offsets, int32_t* idx,
                     void* stream);

/*
 * K5+K6 fused forward + loss. Replaces eval_mixture per query over its tile's candidates
 * (Eq. 8) and loss_rel_l2. `targets` may be NULL (evaluation only;
 * qrec and loss_partial are then untouched). With targets: qrec[b] = x | dpred | ell and
 * loss_partial[t] = sum of the tile's per-query loss shares (float64); n_total is the global batch
 * size the mean divides by (3 * n_total entries).
 */
int ndg_forward(int n, int64_t B, int tile, const float* queries, const float* targets, const float* rec,
                int centred, const int64_t* offsets, const int32_t* idx, float eps, int64_t n_total, float* pred,
                float* qrec, double* loss_partial, void* stream);

/* K1c: records for the centred FP32 kernels (`centred` = 1 in ndg_forward / ndg_backward): a copy of
 * rec whose nb2 pair of row i holds (m_hi, m_lo), the float32 head and tail of mean64, so the first
 * forward-substitution term is rho ((x - m_hi) - m_lo) instead of the cancelling rho x + nb2 (very
 * sharp Gaussians; the engine decides from ndg_tc_records' conditioning). */
int ndg_centre_records(int n, int64_t Gev, const double* mean64, const float* rec, float* rec_c, void* stream);

/* Tensor-core records (float32 [Gev][N*pad8(N+1) + 4], rows stored plane-major [K/4][N][4]):
 * Ahat_e = [C L^-1 | C L^-1 (1/2 - m)] from K1's
 * float64 factor (the B operand of the tcgen05 z-GEMM), followed by the colour a[3] and a pad.
 * cond (optional, 3 doubles zeroed by the caller) receives [max, sum of squares, count] over live,
 * non-degenerate e of B_e = max_i (1/2 sum_k |Ahat_ik| + |bias_i|), the conditioning of the z-GEMM
 * (engine.py keeps very sharp mixtures on the FP32 pipe with it). */
int ndg_tc_records(int n, int64_t Gev, const double* mean64, const double* chol64, const uint8_t* eflags,
                   const float* rec, float* rec_tc, double* cond, void* stream);

/* K5+K6 on the tensor cores (tcgen05 kind::tf32, 3xTF32): same contract as ndg_forward, plus the
 * rec_tc records; tile must be <= 256. */
int ndg_forward_tc(int n, int64_t B, int tile, const float* queries, const float* targets,
                   const float* rec_tc, const int64_t* offsets, const int32_t* idx, float eps, int64_t n_total,
                   float* pred, float* qrec, double* loss_partial, void* stream);

/* Standalone loss_rel_l2 for the module-level API (the step fuses it into K5):
 * loss_partial[ceil(B/256)] float64 block partials of mean((p - t)^2 / (p^2 + eps)) over 3 * n_total
 * entries, and dpred[B][3] (may be NULL) with the denominator detached; sum the partials
 * with ndg_loss_finalize. */
int ndg_loss_rel_l2(int64_t B, const float* pred, const float* target, double eps, int64_t n_total, float* dpred,
                    double* loss_partial, void* stream);

/* Deterministic fixed-order sum of the per-tile loss partials. */
int ndg_loss_finalize(int64_t T, const double* loss_partial, double* loss, void* stream);

/* K7 work items in band order: items[n_chunks] int64 = (tile << 32) | chunk, the band of 512 tiles
 * chunk-major over the chunks every tile of it has (the CTAs in flight share one candidate chunk's
 * records and accumulators in L2), tile-major over the rest. A bijection onto the work items that
 * chunk_offsets (ndg_scan_counts) numbers tile-major. */
int ndg_work_items(int64_t T, const int64_t* chunk_offsets, int64_t* items, void* stream);

/* Bounds of the deterministic backward reduction: bounds[4] (uint32, zeroed by the caller) receive the
 * float bit patterns of H = max_q sum_c |dpred_c|, max_q,c |dpred_c|, max_q ell (over qrec[B]) and
 * max |a_c| over live Gaussians (rec, eflags). Run after the forward, before K7. */
int ndg_bwd_bounds(int n, int64_t B, const float* qrec, int64_t Gev, const float* rec, const uint8_t* eflags,
                   uint32_t* bounds, void* stream);

/*
 * K7 fused backward. Replaces the pair loop of `backward`: per (tile, chunk of
 * candidates) one thread per Gaussian sweeps the tile's queries and accumulates the sufficient
 * statistics S, t, gA and the density-control statistics, then adds them to accum[2][Gev][A] (int64
 * fixed point: hi words then lo words, zeroed by the caller) with scales derived from `bounds`. The
 * sums are exact integers, so the result is independent of the order work items run in (SPEC.md:294,
 * bit-reproducible training :380, :581). `items` from ndg_work_items; n_chunks may exceed the real
 * count (a worst-case-sized list for CUDA-graph replay) when the extra slots hold -1, which exit.
 */
int ndg_backward(int n, int64_t B, int tile, const float* qrec, const float* rec, int centred, const int64_t* offsets,
                 const int32_t* idx, const int64_t* items, int64_t n_chunks, int64_t Gev, const uint32_t* bounds,
                 int64_t* accum, void* stream);

/*
 * K7 on warp-level tensor cores for large N (mma.sync m16n8k16 f16 with hi / lo splits and power-of-two
 * operand scaling, fp32 accumulation). Same work items (chunk_offsets, n_chunks) and the same accum
 * contract as ndg_backward, but z~ comes from the K5 record rec_tc (z~ = Ahat [x - 1/2] + bias, as in
 * ndg_forward_tc): a warp owns two Gaussians, MMA1 forms 16 x 8 (dims x queries) blocks of z~ and MMA2
 * adds (w z~) z~^T over 16 queries to S' in the MMA accumulators. Tile must be a multiple of 8. Returns NDG_ERR_UNSUPPORTED_DIMS when
 * ndg_backward_mma_supported(n) is 0 (n outside 9..16).
 */
int ndg_backward_mma_supported(int n);
int ndg_backward_mma(int n, int64_t B, int tile, const float* qrec, const float* rec_tc, const int64_t* offsets,
                     const int32_t* idx, const int64_t* items, int64_t n_chunks, int64_t Gev, const uint32_t* bounds,
                     int64_t* accum, void* stream);

/* Fixed point -> float64: accum[2][Gev][A] int64 from K7 becomes float64 accum[Gev][A] in place over its
 * first half (hi / s + lo / (s 2^40) with the scales of `bounds` and B); a Gaussian whose flag slot is
 * set (a non-finite or out-of-bound partial) gets NaN in every slot, which K8 reports. */
int ndg_acc_dequant(int n, int64_t Gev, int64_t B, const uint32_t* bounds, int64_t* accum, void* stream);

/*
 * Diagnostic (not on the training path): brute_force_active for every tile as a
 * bit-mask [T][ceil(Gev/32)] (+ per-tile popcounts, zeroed by the caller): bit (t, e) = 1 iff a live,
 * non-degenerate evaluated Gaussian e has |z|^2 <= max_s2 (float64 forward substitution) at some query
 * of tile t, i.e. eval_gaussian >= epsilon with max_s2 = -2 ln epsilon. The culling ablation
 * (cmd_bench_cull) counts false culls against it.
 */
int ndg_active_mask(int n, int64_t B, int tile, const float* queries, const double* mean64, const double* chol64,
                    const uint8_t* eflags, int64_t Gev, double max_s2, uint32_t* mask, int64_t* counts,
                    void* stream);

/*
 * Diagnostic for cmd_gradcheck: the rel-L2 loss of M raw-parameter variants
 * (params / child: float64 [M][G][N+P+4], flags [G]) at B queries in float64, culling off. With
 * inv_den = NULL the kernel writes variant 0's prediction to pred_out[B][3] (the base pass); with
 * inv_den = 1 / (pred_base^2 + eps) [B][3] it writes loss[m] (the denominator held at the base
 * prediction, as the finite differences of SPEC.md:273-281 with a detached denominator require).
 */
int ndg_loss_f64(int n, int G, int amp_mode, int M, const double* params, const double* child, const uint8_t* flags,
                 int64_t B, const float* queries, const float* targets, const double* inv_den, double* pred_out,
                 double* loss, void* stream);

/*
 * Error path of NonFiniteGradientError (the error names component, block and batch index):
 * out[0] (int64, set to INT64_MAX by the caller) receives the lowest query index b of the step whose pair
 * with evaluated Gaussian e1 or e2 (-1 = none), on a tile where it is a candidate in `mask`, gives a
 * non-finite backward term in K7's float32 arithmetic (qrec / rec as passed to ndg_backward).
 */
int ndg_nonfinite_query(int n, int64_t B, int tile, const float* qrec, const float* rec, const uint32_t* mask,
                        int64_t Gev, int64_t e1, int64_t e2, int64_t* out, void* stream);

/*
 * Diagnostic for cmd_gradcheck / finite_diff_grad: central finite differences of the
 * rel-L2 loss in float64 (culling off, denominator held at pred_base: inv_den = 1 / (pred_base^2 + eps))
 * for M raw coordinates coords[M][2] = (row, column), row < G a parent row, G <= row < 2G a child row;
 * points = 2 ((l(+h) - l(-h)) / 2h) or 4 (the O(h^4) stencil). Only the Gaussians that read the
 * perturbed row are re-evaluated, and the stencil is summed as sum_s w_s (2 d delta_s + delta_s^2)
 * (d = pred_base - target, delta_s = their change), so the O(1) loss terms cancel exactly.
 */
int ndg_fd_f64(int n, int G, int amp_mode, const double* params, const double* child, const uint8_t* flags, int64_t B,
               const float* queries, const float* targets, const double* pred_base, const double* inv_den, int M,
               const int* coords, double h, int points, double* fd, void* stream);

/*
 * Diagnostic for cmd_gradcheck: the backward pair loop in float64 (culling off, every query, one thread
 * per evaluated Gaussian) with K7's accumulator contract, written to accum[Gev][A] (float64) for
 * ndg_epilogue. dpred [B][3] and ell [B] (may be NULL) in float64; a = alpha * sigmoid(color) is
 * activated in float64 from the raw rows. Lets gradcheck hold the analytic gradient to SPEC.md:572's
 * per-coordinate bar (the float32 product kernels are checked against the oracle instead).
 */
int ndg_backward_f64(int n, int64_t G, int64_t Gev, int amp_mode, const float* params, const float* child,
                     const double* mean64, const double* chol64, const uint8_t* eflags, int64_t B,
                     const float* queries, const double* dpred, const double* ell, double* accum, void* stream);

/*
 * K8 epilogue. Replaces the tail of `backward`: raw-parameter gradients of parents
 * and live children including the child->parent cross terms; stats[Gev][3] =
 * (loss share, gradient proxy, pairs). Non-finite gradients -> status NONFINITE_GRADIENT.
 */
int ndg_epilogue(int n, int64_t G, int64_t Gev, int amp_mode, const float* params, const float* child,
                 const uint8_t* flags, const uint8_t* eflags, const double* chol64, const double* accum,
                 float* grad_params, float* grad_child, float* stats, ndg_status* status, void* stream);

/* K9 Adam. Replaces adam_step with per-block learning rates.
 * Rows whose row_mask byte is 0 are left untouched (absent children, frozen components). */
int ndg_adam(int n, int64_t rows, float* params, const float* grad, float* m1, float* m2, const uint8_t* row_mask,
             int step, float lr_mean, float lr_chol, float lr_color, float lr_amp, float beta1, float beta2,
             float eps, void* stream);
/* K9 with the row selection taken from the mixture's flag bytes (bit0 live child, bit1 frozen): row r is
 * updated iff (flags[r] & require) == require and (flags[r] & forbid) == 0 -- parents: require 0, forbid
 * frozen; live children: require child, forbid frozen. Same arithmetic as ndg_adam. */
int ndg_adam_flags(int n, int64_t rows, float* params, const float* grad, float* m1, float* m2, const uint8_t* flags,
                   int require, int forbid, int step, float lr_mean, float lr_chol, float lr_color, float lr_amp,
                   float beta1, float beta2, float eps, void* stream);

/*
 * Device-side sample_batch: B fresh uniform queries in [0,1)^N sorted by the first
 * dimension into contiguous tiles of `tile`, as the rows of the tiles t with t % world == rank (the
 * rank's strided share of the global batch, in tile order). The sorted first coordinates are generated
 * directly as uniform order statistics (normalised prefix sums of B + 1 exponentials, exact in 32.32
 * fixed point, so non-decreasing by construction), the others iid; randomness is Philox4x32-10 keyed by
 * (seed, draw), so a batch is a pure function of those two integers. B <= 2^24.
 * workspace: ndg_sample_workspace(B) bytes of scratch.
 */
int64_t ndg_sample_workspace(int64_t B);
int ndg_sample_batch(int n, int64_t B, int tile, int rank, int world, uint64_t seed, uint64_t draw, int64_t* workspace,
                     float* queries, void* stream);

/* shading_toy_target at queries[B][n] (4 <= n <= 10): params = freq[3] | phase[3];
 * out[B][3] float32. */
int ndg_shading_target(int n, int64_t B, const float* queries, const float* params, float* out, void* stream);

/* FP32-pipe peak probe (roofline denominator for K5 / K7; not part of the reference interface):
 * `blocks` CTAs of 256 threads, each running 8 independent FFMA chains for 16 * iters steps. */
int ndg_fp32_probe(float* out, int blocks, int iters, void* stream);
double ndg_fp32_probe_flops(int blocks, int iters);
/* TF32 tensor-core peak probe (tcgen05.mma kind::tf32 M=128 N=256 K=8 on resident operands). */
int ndg_tf32_probe(float* out, int blocks, int iters, void* stream);
double ndg_tf32_probe_flops(int blocks, int iters);
/* Warp-level tensor-core peak probe (mma.sync m16n8k16 f16 -> f32, K7-MMA's instruction; 16 warps x 8 chains). */
int ndg_hmma_probe(float* out, int blocks, int iters, void* stream);
double ndg_hmma_probe_flops(int blocks, int iters);

#ifdef __cplusplus
}
#endif

#endif /* NDG_H */
