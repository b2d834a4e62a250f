/*
 * C / OpenMP restatement of the culled N-D Gaussian-mixture hot path -- TEST INFRASTRUCTURE ONLY.
 *
 * Same algorithm as oracle/ndg_oracle.py (the NumPy restatement of /root/reference/SPEC.md), in
 * float64, parallelised the way SPEC.md's concurrency model allows: tiles are independent for the
 * bounds / cull / forward, and the backward reduces per Gaussian over its tiles in
 * ascending tile order -- the "fixed component order" of SPEC.md:294 -- so the result does not
 * depend on the thread count. It stands in for the reference's intended compiled `_core`
 * (Cython -> C, -O3 -fopenmp; /root/reference/pkg/setup.py:36-43), whose source is absent.
 *
 * Used as (a) the checker for parity sizes the NumPy oracle cannot finish in seconds and
 * (b) bench.py's cpu_baseline / --impl reference leg ("kind": "port"). Never linked by the product.
 *
 * Culling arithmetic: sequential float64 sums, separate multiply and add (compile with
 * -ffp-contract=off), so candidate lists equal the NumPy oracle's bit for bit.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define TRI(i, j) ((i) * ((i) + 1) / 2 + (j))
#define NMAX 16

static inline double sigm(double x) { return 1.0 / (1.0 + exp(-x)); }

int ndgo_max_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

void ndgo_set_threads(int n) {
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
#else
    (void)n;
#endif
}

/* Activation of one packed chol row into a dense lower N x N. */
static void activate(const double* raw, int N, double* L) {
    memset(L, 0, sizeof(double) * N * N);
    for (int i = 0; i < N; ++i)
        for (int j = 0; j <= i; ++j) {
            double r = raw[TRI(i, j)];
            L[i * N + j] = (i == j) ? exp(r) : 2.0 * sigm(r) - 1.0;
        }
}

/*
 * Evaluated-Gaussian set: e < G parents, e >= G children (if gev == 2G).
 * Outputs mean[Gev*N], L[Gev*N*N] (dense lower), a[Gev*3], live[Gev], degen[Gev],
 * plus Lp[G*N*N] / U[G*N*N] for the chain rule.
 */
void ndgo_eval_set(int N, int64_t G, int64_t Gev, int amp_mode, const double* params, const double* child,
                   const uint8_t* has_child, const uint8_t* frozen, double* mean, double* L, double* a,
                   uint8_t* live, uint8_t* degen, double* Lp, double* Uc) {
    const int P = N * (N + 1) / 2, R = N + P + 4;
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < G; ++i) {
        const double* row = params + i * R;
        double* Li = Lp + i * N * N;
        activate(row + N, N, Li);
        memcpy(L + i * N * N, Li, sizeof(double) * N * N);
        memcpy(mean + i * N, row, sizeof(double) * N);
        double alpha = amp_mode == 0 ? exp(row[N + P + 3]) : sigm(row[N + P + 3]);
        for (int c = 0; c < 3; ++c) a[i * 3 + c] = alpha * sigm(row[N + P + c]);
        live[i] = !frozen[i];
        if (Gev == 2 * G) {
            const double* cr = child + i * R;
            double* U = Uc + i * N * N;
            activate(cr + N, N, U);
            double* mc = mean + (G + i) * N;
            double* Lc = L + (G + i) * N * N;
            for (int r = 0; r < N; ++r) {           /* m_c = L m_u + m_p, ascending k */
                double acc = Li[r * N] * cr[0];
                for (int k = 1; k <= r; ++k) acc = acc + Li[r * N + k] * cr[k];
                mc[r] = acc + row[r];
            }
            memset(Lc, 0, sizeof(double) * N * N);
            for (int r = 0; r < N; ++r)             /* L U, ascending k */
                for (int c = 0; c <= r; ++c) {
                    double acc = Li[r * N + c] * U[c * N + c];
                    for (int k = c + 1; k <= r; ++k) acc = acc + Li[r * N + k] * U[k * N + c];
                    Lc[r * N + c] = acc;
                }
            double ca = amp_mode == 0 ? exp(cr[N + P + 3]) : sigm(cr[N + P + 3]);
            for (int c = 0; c < 3; ++c) a[(G + i) * 3 + c] = ca * sigm(cr[N + P + c]);
            live[G + i] = has_child[i] && !frozen[i];
        }
    }
#pragma omp parallel for schedule(static)
    for (int64_t e = 0; e < Gev; ++e) {
        int bad = 0;
        for (int i = 0; i < N; ++i)
            for (int j = 0; j <= i; ++j) bad |= !isfinite(L[e * N * N + i * N + j]);
        for (int i = 0; i < N; ++i) bad |= L[e * N * N + i * N + i] < 1e-30;
        degen[e] = (uint8_t)bad;
        if (bad) live[e] = 0;
    }
}

/* Projected bounds: mr, sr, thr laid out [k][Gev]. */
void ndgo_project(int N, int64_t Gev, const double* mean, const double* L, const uint8_t* live,
                  const uint8_t* degen, const double* Rv, int k, double mult, double* mr, double* sr,
                  double* thr) {
#pragma omp parallel for schedule(static)
    for (int64_t e = 0; e < Gev; ++e) {
        const double* m = mean + e * N;
        const double* Le = L + e * N * N;
        for (int ri = 0; ri < k; ++ri) {
            const double* r = Rv + ri * N;
            double acc = m[0] * r[0];
            for (int j = 1; j < N; ++j) acc = acc + m[j] * r[j];
            double ss = 0.0;
            for (int j = 0; j < N; ++j) {
                double u = Le[j * N + j] * r[j];
                for (int i = j + 1; i < N; ++i) u = u + Le[i * N + j] * r[i];
                ss = (j == 0) ? u * u : ss + u * u;
            }
            double s = degen[e] ? 0.0 : sqrt(ss);
            mr[ri * Gev + e] = acc;
            sr[ri * Gev + e] = s;
            thr[ri * Gev + e] = live[e] ? mult * s : -1.0;
        }
    }
}

/* Tile bounds: lo/hi laid out [T][k]. */
void ndgo_tile_bounds(int N, int64_t B, int tile, const float* q, const double* Rv, int k, double* lo,
                      double* hi) {
    int64_t T = B / tile;
#pragma omp parallel for schedule(static)
    for (int64_t t = 0; t < T; ++t)
        for (int ri = 0; ri < k; ++ri) {
            const double* r = Rv + ri * N;
            double mn = INFINITY, mx = -INFINITY;
            for (int qi = 0; qi < tile; ++qi) {
                const float* x = q + (t * tile + qi) * N;
                double acc = (double)x[0] * r[0];
                for (int j = 1; j < N; ++j) acc = acc + (double)x[j] * r[j];
                if (acc < mn) mn = acc;
                if (acc > mx) mx = acc;
            }
            lo[t * k + ri] = mn;
            hi[t * k + ri] = mx;
        }
}

static inline int culled(const double* lo, const double* hi, const double* mr, const double* thr, int64_t Gev,
                         int k, int64_t e) {
    if (thr[e] < 0.0) return 1;
    for (int ri = 0; ri < k; ++ri) {
        double m = mr[ri * Gev + e], t = thr[ri * Gev + e];
        if (lo[ri] - m > t || m - hi[ri] > t) return 1;
    }
    return 0;
}

/*
 * cull_tile for every tile. Work items are (tile, block of CULL_EB Gaussians) so
 * every thread has work even when only a few tiles are culled (a sampled-tile parity check or the
 * CPU baseline's bounded sample); indices stay ascending because each item writes its own range.
 */
#define CULL_EB 2048

static void cull_part_counts(int64_t T, int k, int64_t Gev, const double* lo, const double* hi, const double* mr,
                             const double* thr, int64_t nb, int64_t* part) {
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t w = 0; w < T * nb; ++w) {
        int64_t t = w / nb, e0 = (w % nb) * CULL_EB, e1 = e0 + CULL_EB < Gev ? e0 + CULL_EB : Gev, c = 0;
        for (int64_t e = e0; e < e1; ++e) c += !culled(lo + t * k, hi + t * k, mr, thr, Gev, k, e);
        part[w] = c;
    }
}

/* phase 1: counts[T]. */
void ndgo_cull_counts(int64_t T, int k, int64_t Gev, const double* lo, const double* hi, const double* mr,
                      const double* thr, int64_t* counts) {
    int64_t nb = (Gev + CULL_EB - 1) / CULL_EB;
    int64_t* part = (int64_t*)calloc((size_t)(T * nb + 1), sizeof(int64_t));
    cull_part_counts(T, k, Gev, lo, hi, mr, thr, nb, part);
    for (int64_t t = 0; t < T; ++t) {
        int64_t c = 0;
        for (int64_t b = 0; b < nb; ++b) c += part[t * nb + b];
        counts[t] = c;
    }
    free(part);
}

/* phase 2: ascending candidate indices into idx[offsets[t] .. offsets[t+1]). */
void ndgo_cull_fill(int64_t T, int k, int64_t Gev, const double* lo, const double* hi, const double* mr,
                    const double* thr, const int64_t* offsets, int32_t* idx) {
    int64_t nb = (Gev + CULL_EB - 1) / CULL_EB;
    int64_t* part = (int64_t*)calloc((size_t)(T * nb + 1), sizeof(int64_t));
    cull_part_counts(T, k, Gev, lo, hi, mr, thr, nb, part);
    for (int64_t t = 0; t < T; ++t) {           /* exclusive prefix within the tile */
        int64_t o = offsets[t];
        for (int64_t b = 0; b < nb; ++b) {
            int64_t c = part[t * nb + b];
            part[t * nb + b] = o;
            o += c;
        }
    }
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t w = 0; w < T * nb; ++w) {
        int64_t t = w / nb, e0 = (w % nb) * CULL_EB, e1 = e0 + CULL_EB < Gev ? e0 + CULL_EB : Gev, o = part[w];
        for (int64_t e = e0; e < e1; ++e)
            if (!culled(lo + t * k, hi + t * k, mr, thr, Gev, k, e)) idx[o++] = (int32_t)e;
    }
    free(part);
}

static inline double pair_eval(int N, const double* x, const double* m, const double* Le, double* z) {
    double s = 0.0;
    for (int i = 0; i < N; ++i) {
        double acc = x[i] - m[i];
        for (int j = 0; j < i; ++j) acc = acc - Le[i * N + j] * z[j];
        z[i] = acc / Le[i * N + i];
        s += z[i] * z[i];
    }
    return s;
}

/* eval_mixture over each tile's candidates. pred [B*3]. Queries are independent
 * (SPEC.md:136), so the work items are single queries: all threads are busy even on one tile. */
void ndgo_forward(int N, int64_t B, int tile, const float* q, const double* mean, const double* L,
                  const double* a, const int64_t* offsets, const int32_t* idx, double* pred) {
#pragma omp parallel for schedule(dynamic, 4)
    for (int64_t b = 0; b < B; ++b) {
        double x[NMAX], z[NMAX];
        int64_t t = b / tile;
        for (int j = 0; j < N; ++j) x[j] = (double)q[b * N + j];
        double p0 = 0, p1 = 0, p2 = 0;
        for (int64_t c = offsets[t]; c < offsets[t + 1]; ++c) {
            int64_t e = idx[c];
            double g = exp(-0.5 * pair_eval(N, x, mean + e * N, L + e * N * N, z));
            p0 += g * a[e * 3];
            p1 += g * a[e * 3 + 1];
            p2 += g * a[e * 3 + 2];
        }
        pred[b * 3] = p0;
        pred[b * 3 + 1] = p1;
        pred[b * 3 + 2] = p2;
    }
}

/* loss_rel_l2, detached denominator; dpred, ell per query. Returns the loss. */
double ndgo_loss(int64_t B, const double* pred, const float* tgt, double eps, int64_t n_total, double* dpred,
                 double* ell) {
    double inv = 1.0 / (3.0 * (double)n_total), tot = 0.0;
    for (int64_t b = 0; b < B; ++b) {
        double l = 0.0;
        for (int c = 0; c < 3; ++c) {
            double p = pred[b * 3 + c], d = p - (double)tgt[b * 3 + c], den = p * p + eps;
            l += d * d / den;
            dpred[b * 3 + c] = 2.0 * d / den * inv;
        }
        ell[b] = l * inv;
        tot += ell[b];
    }
    return tot;
}

/*
 * Backward accumulation, Gaussian-major over the transposed candidate lists so
 * each Gaussian's sum runs over its tiles in ascending order.
 * accum layout per e: S lower packed [P] | t [N] | gA [3] | stats [3].
 */
void ndgo_backward(int N, int64_t B, int tile, int64_t Gev, const float* q, const double* dpred, const double* ell,
                   const double* mean, const double* L, const double* a, const int64_t* offsets,
                   const int32_t* idx, double* accum) {
    const int P = N * (N + 1) / 2, A = P + N + 6;
    int64_t T = B / tile, nnz = offsets[T];
    int64_t* cnt = (int64_t*)calloc((size_t)Gev + 1, sizeof(int64_t));
    int32_t* tl = (int32_t*)malloc(sizeof(int32_t) * (size_t)(nnz > 0 ? nnz : 1));
    for (int64_t c = 0; c < nnz; ++c) cnt[idx[c] + 1]++;
    for (int64_t e = 0; e < Gev; ++e) cnt[e + 1] += cnt[e];
    int64_t* pos = (int64_t*)malloc(sizeof(int64_t) * (size_t)(Gev + 1));
    memcpy(pos, cnt, sizeof(int64_t) * (size_t)(Gev + 1));
    for (int64_t t = 0; t < T; ++t)
        for (int64_t c = offsets[t]; c < offsets[t + 1]; ++c) tl[pos[idx[c]]++] = (int32_t)t;
    free(pos);
#pragma omp parallel for schedule(dynamic, 16)
    for (int64_t e = 0; e < Gev; ++e) {
        double* acc = accum + e * A;
        memset(acc, 0, sizeof(double) * A);
        double x[NMAX], z[NMAX];
        const double* m = mean + e * N;
        const double* Le = L + e * N * N;
        const double* ae = a + e * 3;
        for (int64_t c = cnt[e]; c < cnt[e + 1]; ++c) {
            int64_t t = tl[c];
            for (int qi = 0; qi < tile; ++qi) {
                int64_t b = t * tile + qi;
                for (int j = 0; j < N; ++j) x[j] = (double)q[b * N + j];
                double s = pair_eval(N, x, m, Le, z);
                double g = exp(-0.5 * s);
                const double* dp = dpred + b * 3;
                double h = dp[0] * ae[0] + dp[1] * ae[1] + dp[2] * ae[2];
                double coef = -g * h;
                for (int i = 0; i < N; ++i) {
                    double w = coef * z[i];
                    for (int j = 0; j <= i; ++j) acc[TRI(i, j)] += w * z[j];
                    acc[P + i] += w;
                }
                for (int ch = 0; ch < 3; ++ch) acc[P + N + ch] += g * dp[ch];
                acc[P + N + 3] += g * ell[b];
                acc[P + N + 4] += fabs(coef) * sqrt(s);
                acc[P + N + 5] += 1.0;
            }
        }
    }
    free(cnt);
    free(tl);
}

/* X = L^-T Y for dense lower L (back substitution per column). */
static void solve_upper_T(int N, const double* L, const double* Y, double* X) {
    for (int c = 0; c < N; ++c)
        for (int i = N - 1; i >= 0; --i) {
            double acc = Y[i * N + c];
            for (int k = i + 1; k < N; ++k) acc -= L[k * N + i] * X[k * N + c];
            X[i * N + c] = acc / L[i * N + i];
        }
}

static void chol_chain(int N, const double* GL, const double* L, double* out) {
    for (int i = 0; i < N; ++i)
        for (int j = 0; j <= i; ++j)
            out[TRI(i, j)] = (i == j) ? GL[i * N + i] * L[i * N + i] : GL[i * N + j] * (1.0 - L[i * N + j] * L[i * N + j]) * 0.5;
}

/*
 * Raw-parameter gradients from the accumulators (child cross terms :266).
 * gp / gc [G*R]; grads of non-live Gaussians are zero.
 */
void ndgo_epilogue(int N, int64_t G, int64_t Gev, int amp_mode, const double* params, const double* child,
                   const uint8_t* live, const double* L, const double* Lp, const double* Uc, const double* accum,
                   double* gp, double* gc) {
    const int P = N * (N + 1) / 2, R = N + P + 4, A = P + N + 6;
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < G; ++i) {
        double GLp[NMAX * NMAX] = {0}, dmp[NMAX] = {0};
        double Sf[NMAX * NMAX], X[NMAX * NMAX];
        double* op = gp + i * R;
        double* oc = gc + i * R;
        memset(op, 0, sizeof(double) * R);
        memset(oc, 0, sizeof(double) * R);
        for (int which = 0; which < (Gev == 2 * G ? 2 : 1); ++which) {
            int64_t e = which ? G + i : i;
            if (!live[e]) continue;
            const double* acc = accum + e * A;
            const double* Le = L + e * N * N;
            for (int r = 0; r < N; ++r)
                for (int c = 0; c <= r; ++c) Sf[r * N + c] = Sf[c * N + r] = acc[TRI(r, c)];
            solve_upper_T(N, Le, Sf, X);
            double GL[NMAX * NMAX] = {0}, dm[NMAX], tv[NMAX * NMAX] = {0};
            for (int r = 0; r < N; ++r)
                for (int c = 0; c <= r; ++c) GL[r * N + c] = -X[r * N + c];
            for (int r = 0; r < N; ++r) tv[r * N] = acc[P + r];
            solve_upper_T(N, Le, tv, X);
            for (int r = 0; r < N; ++r) dm[r] = -X[r * N];
            const double* row = which ? child + i * R : params + i * R;
            double* out = which ? oc : op;
            double alpha = amp_mode == 0 ? exp(row[N + P + 3]) : sigm(row[N + P + 3]);
            double dalpha = 0.0;
            for (int c = 0; c < 3; ++c) {
                double cc = sigm(row[N + P + c]);
                out[N + P + c] = acc[P + N + c] * alpha * cc * (1.0 - cc);
                dalpha += acc[P + N + c] * cc;
            }
            out[N + P + 3] = dalpha * (amp_mode == 0 ? alpha : alpha * (1.0 - alpha));
            if (!which) {
                for (int r = 0; r < N * N; ++r) GLp[r] += GL[r];
                for (int r = 0; r < N; ++r) dmp[r] += dm[r];
            } else {
                const double* Lpi = Lp + i * N * N;
                const double* U = Uc + i * N * N;
                const double* mu = child + i * R;
                double dU[NMAX * NMAX] = {0};
                for (int r = 0; r < N; ++r)
                    for (int c = 0; c <= r; ++c) {
                        double s1 = 0.0, s2 = 0.0;
                        for (int k = 0; k < N; ++k) s1 += GL[r * N + k] * U[c * N + k];   /* G U^T */
                        for (int k = 0; k < N; ++k) s2 += Lpi[k * N + r] * GL[k * N + c]; /* L^T G */
                        GLp[r * N + c] += s1 + dm[r] * mu[c];
                        dU[r * N + c] = s2;
                    }
                for (int r = 0; r < N; ++r) {
                    double s = 0.0;
                    for (int k = 0; k < N; ++k) s += Lpi[k * N + r] * dm[k];
                    oc[r] = s;
                    dmp[r] += dm[r];
                }
                chol_chain(N, dU, U, oc + N);
            }
        }
        for (int r = 0; r < N; ++r) op[r] = dmp[r];
        chol_chain(N, GLp, Lp + i * N * N, op + N);
    }
}
