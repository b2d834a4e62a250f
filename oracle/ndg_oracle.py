"""CPU oracle for the culled N-D Gaussian-mixture hot path -- TEST INFRASTRUCTURE ONLY.

This module is the *checker*, never the product. Only ``tests/``, ``__graft_entry__.smoke()``
and ``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import it. The product path
(``paper_2405_20067_b200``) never imports anything under ``oracle/`` and fails loudly when its CUDA
library is missing.

What it restates (NumPy float64, following /root/reference/SPEC.md):
  * activation / evaluation / composition        SPEC.md:63-101 (gmm-core)
  * projection set, projected bounds, tile bounds SPEC.md:152-206 (culling)
  * relative-L2 loss and analytic backward        SPEC.md:253-271 (grad)
  * brute-force and finite-difference oracles
  * Adam, spawn / check / materialize, freeze     SPEC.md:336-374, 388 (trainer)
  * tiling by stable sort on the first dimension  SPEC.md:440-448 (datasets)
and the paper's equations: Eq. 1-2, Eq. 3-5,
Eq. 6-7, Eq. 8.

Parity pinning. The reference ships no runnable implementation of this path (only
``pkg/src/ndgauss/errors.py`` exists; ``_core.pyx`` and the NumPy backend named in
``pkg/setup.py:3-4,38`` are absent), so there is no reference binary or importable module to run.
The oracle is pinned against every worked example / known-answer test SPEC.md gives for the path
(``tests/golden/spec_kats.json``, checked by ``tests/test_oracle_kats.py``) and against the SPEC's
own derived oracles (explicit-inverse density, dense quadratic form, finite differences,
brute-force culling). Choices SPEC.md leaves open are pinned here and listed in DESIGN.md §"Parity
pins": projection RNG stream, child culled by its own composed bounds, FP64 sequential no-FMA cull
arithmetic, equality at the threshold = kept, stable sort for tiling.

Culling arithmetic is written element-wise (``a = a + x*y`` on float64 arrays) on purpose: NumPy
never fuses these into FMAs and evaluates them in the written order, which is the order the CUDA
kernels reproduce with ``__dmul_rn`` / ``__dadd_rn`` so candidate lists match bit for bit.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

BRIGHTNESS = 0
OPACITY = 1
DEGENERATE_DIAG = 1e-30
LOG2E = 1.4426950408889634


# ----------------------------------------------------------------------------------------------
# layout helpers
# ----------------------------------------------------------------------------------------------
def n_chol(n: int) -> int:
    return n * (n + 1) // 2


def tri(i: int, j: int) -> int:
    """Row-major lower-triangle packing index, SPEC.md:31 ("row-major packing of the lower triangle")."""
    return i * (i + 1) // 2 + j


def raw_width(n: int) -> int:
    """Floats per component row: mean_raw[N] | chol_raw[P] | color_raw[3] | amp_raw[1]."""
    return n + n_chol(n) + 4


def raw_slices(n: int):
    p = n_chol(n)
    return slice(0, n), slice(n, n + p), slice(n + p, n + p + 3), n + p + 3


# ----------------------------------------------------------------------------------------------
# gmm-core
# ----------------------------------------------------------------------------------------------
def sigmoid(x):
    x = np.asarray(x, dtype=np.float64)
    with np.errstate(over="ignore"):
        return 1.0 / (1.0 + np.exp(-x))


def activate_cholesky(chol_raw, n: int) -> np.ndarray:
    """L_ii = exp(raw), L_ij = 2*sigmoid(raw) - 1 (i > j), zero above the diagonal."""
    chol_raw = np.asarray(chol_raw, dtype=np.float64)
    if chol_raw.shape[-1] != n_chol(n):
        raise ValueError("chol_raw has wrong length")
    L = np.zeros(chol_raw.shape[:-1] + (n, n), dtype=np.float64)
    for i in range(n):
        for j in range(i + 1):
            r = chol_raw[..., tri(i, j)]
            if i == j:
                with np.errstate(over="ignore", under="ignore"):
                    L[..., i, i] = np.exp(r)
            else:
                L[..., i, j] = 2.0 * sigmoid(r) - 1.0
    return L


def inverse_activate_cholesky(L, n: int, clamp: float = 1.0 - 1e-6):
    """Inverse of activate_cholesky used by materialize: log on the diagonal,
    logit((x+1)/2) on off-diagonals with the value clamped to +-(1-1e-6). Returns (raw, n_clamped)."""
    L = np.asarray(L, dtype=np.float64)
    raw = np.zeros(L.shape[:-2] + (n_chol(n),), dtype=np.float64)
    clamped = 0
    for i in range(n):
        for j in range(i + 1):
            v = L[..., i, j]
            if i == j:
                raw[..., tri(i, j)] = np.log(v)
            else:
                vc = np.clip(v, -clamp, clamp)
                clamped += int(np.count_nonzero(vc != v))
                s = (vc + 1.0) / 2.0
                raw[..., tri(i, j)] = np.log(s) - np.log1p(-s)
    return raw, clamped


def amp_activate(amp_raw, amp_mode: int):
    """alpha = exp(amp_raw) (Brightness) or sigmoid(amp_raw) (Opacity)."""
    amp_raw = np.asarray(amp_raw, dtype=np.float64)
    if amp_mode == BRIGHTNESS:
        return np.exp(amp_raw)
    return sigmoid(amp_raw)


def amp_inverse(alpha, amp_mode: int):
    alpha = np.asarray(alpha, dtype=np.float64)
    if amp_mode == BRIGHTNESS:
        return np.log(alpha)
    return np.log(alpha) - np.log1p(-alpha)


def solve_lower(L, d):
    """Forward substitution L z = d (never forms V^-1). Broadcasts over leading dims."""
    n = L.shape[-1]
    z = np.empty(np.broadcast_shapes(L.shape[:-1], d.shape), dtype=np.float64)
    for i in range(n):
        acc = d[..., i].astype(np.float64, copy=True)
        for j in range(i):
            acc = acc - L[..., i, j] * z[..., j]
        z[..., i] = acc / L[..., i, i]
    return z


def eval_gaussian(mean, L, x):
    """exp(-0.5 ||z||^2) with L z = x - m."""
    d = np.asarray(x, np.float64) - np.asarray(mean, np.float64)
    z = solve_lower(np.asarray(L, np.float64), d)
    return np.exp(-0.5 * np.sum(z * z, axis=-1))


def compose_child(m_p, L, m_u, U):
    """SPEC.md:93-101 / Eq. 6-7: m_c = L m_u + m_p (sequential in k), factor L U (sequential in k).

    Sums run in ascending k with separate multiply and add so the CUDA prologue reproduces them.
    """
    m_p = np.asarray(m_p, np.float64)
    L = np.asarray(L, np.float64)
    m_u = np.asarray(m_u, np.float64)
    U = np.asarray(U, np.float64)
    n = L.shape[-1]
    m_c = np.empty(np.broadcast_shapes(m_p.shape, m_u.shape), dtype=np.float64)
    for i in range(n):
        acc = L[..., i, 0] * m_u[..., 0]
        for k in range(1, i + 1):
            acc = acc + L[..., i, k] * m_u[..., k]
        m_c[..., i] = acc + m_p[..., i]
    LU = np.zeros(np.broadcast_shapes(L.shape, U.shape), dtype=np.float64)
    for i in range(n):
        for j in range(i + 1):
            acc = L[..., i, j] * U[..., j, j]
            for k in range(j + 1, i + 1):
                acc = acc + L[..., i, k] * U[..., k, j]
            LU[..., i, j] = acc
    return m_c, LU


def covariance_from_factor(L):
    L = np.asarray(L, np.float64)
    return L @ np.swapaxes(L, -1, -2)


# ----------------------------------------------------------------------------------------------
# Mixture container -- host-side numpy form used by tests
# ----------------------------------------------------------------------------------------------
@dataclass
class OMixture:
    """Raw mixture: parent rows, child rows, has_child / frozen masks."""
    n_dims: int
    amp_mode: int
    params: np.ndarray                 # [G, R] float
    child: np.ndarray | None = None    # [G, R] float
    has_child: np.ndarray | None = None
    frozen: np.ndarray | None = None

    def __post_init__(self):
        self.params = np.asarray(self.params, dtype=np.float64)
        G = self.params.shape[0]
        if self.child is None:
            self.child = np.zeros_like(self.params)
        self.child = np.asarray(self.child, dtype=np.float64)
        if self.has_child is None:
            self.has_child = np.zeros(G, dtype=bool)
        if self.frozen is None:
            self.frozen = np.zeros(G, dtype=bool)
        self.has_child = np.asarray(self.has_child, bool)
        self.frozen = np.asarray(self.frozen, bool)

    @property
    def G(self):
        return self.params.shape[0]

    @property
    def any_child(self):
        return bool(np.any(self.has_child & ~self.frozen))


@dataclass
class EvalSet:
    """Evaluated Gaussians in the fixed index space e = parent i (i < G) | child of i (G + i)."""
    G: int
    Gev: int
    mean: np.ndarray        # [Gev, N]
    L: np.ndarray           # [Gev, N, N]
    a: np.ndarray           # [Gev, 3] premultiplied alpha * color
    live: np.ndarray        # [Gev] evaluated (not absent / frozen / degenerate)
    degenerate: np.ndarray  # [Gev]
    # per-component activations kept for the chain rule
    Lp: np.ndarray = field(default=None)
    Uc: np.ndarray = field(default=None)
    mu: np.ndarray = field(default=None)


class OracleInvalidParameter(ValueError):
    def __init__(self, msg, component, block, entry):
        super().__init__(msg)
        self.component, self.block, self.entry = component, block, entry


def _check_finite(rows, which):
    bad = ~np.isfinite(rows)
    if bad.any():
        comp, ent = np.argwhere(bad)[0]
        raise OracleInvalidParameter(f"non-finite raw parameter in {which}", int(comp), which, int(ent))


def build_eval_set(mix: OMixture, gev: int | None = None) -> EvalSet:
    """Activate parents and compose live children.

    Index space: e < G is parent e; e >= G is the child of component e - G. Absent / frozen /
    degenerate Gaussians are not live: they are always culled and contribute 0.
    """
    N, G = mix.n_dims, mix.G
    ms, cs, cols, amp = raw_slices(N)
    _check_finite(mix.params, "parent")
    use_child = mix.any_child if gev is None else (gev == 2 * G)
    if use_child:
        _check_finite(mix.child[mix.has_child], "child")
    Gev = 2 * G if use_child else G
    Lp = activate_cholesky(mix.params[:, cs], N)
    mp = mix.params[:, ms].copy()
    ap = amp_activate(mix.params[:, amp], mix.amp_mode)[:, None] * sigmoid(mix.params[:, cols])
    mean = np.zeros((Gev, N))
    L = np.zeros((Gev, N, N))
    a = np.zeros((Gev, 3))
    live = np.zeros(Gev, bool)
    mean[:G], L[:G], a[:G] = mp, Lp, ap
    live[:G] = ~mix.frozen
    Uc = mu = None
    if use_child:
        Uc = activate_cholesky(mix.child[:, cs], N)
        mu = mix.child[:, ms].copy()
        mc, Lc = compose_child(mp, Lp, mu, Uc)
        mean[G:], L[G:] = mc, Lc
        a[G:] = amp_activate(mix.child[:, amp], mix.amp_mode)[:, None] * sigmoid(mix.child[:, cols])
        live[G:] = mix.has_child & ~mix.frozen
    diag = np.diagonal(L, axis1=-2, axis2=-1)
    degenerate = np.any(diag < DEGENERATE_DIAG, axis=-1) | ~np.all(np.isfinite(L.reshape(Gev, -1)), axis=-1)
    live &= ~degenerate
    return EvalSet(G=G, Gev=Gev, mean=mean, L=L, a=a, live=live, degenerate=degenerate & (live | degenerate),
                   Lp=Lp, Uc=Uc, mu=mu)


# ----------------------------------------------------------------------------------------------
# culling
# ----------------------------------------------------------------------------------------------
def make_projection_set(n_dims: int, k: int, seed: int) -> np.ndarray:
    """SPEC.md:178-186. Pinned stream: default_rng(seed).standard_normal((k, N)), rows normalized.
    The norm is a sequential float64 sum of squares followed by sqrt (bitwise reproducible)."""
    if n_dims < 1 or k < 1:
        raise ValueError("n_dims and k must be >= 1")
    v = np.random.default_rng(seed).standard_normal((k, n_dims))
    ss = v[:, 0] * v[:, 0]
    for j in range(1, n_dims):
        ss = ss + v[:, j] * v[:, j]
    return v / np.sqrt(ss)[:, None]


def dot_seq(X, r):
    """sum_j X[..., j] * r[j], float64, ascending j, no FMA (the culling dot-product order)."""
    X = np.asarray(X, dtype=np.float64)
    acc = X[..., 0] * r[0]
    for j in range(1, X.shape[-1]):
        acc = acc + X[..., j] * r[j]
    return acc


def project_components(ev: EvalSet, R: np.ndarray, multiplier: float = 3.0):
    """m_r = m^T r (Eq. 3), sigma_r = ||L^T r|| (Eq. 4), degenerate -> sigma 0.

    Returns (m_r [k, Gev], sigma_r [k, Gev], thr [k, Gev]) with thr = multiplier * sigma_r for live
    Gaussians and -1 for absent / frozen / degenerate ones (always culled)."""
    k, N = R.shape
    mr = np.empty((k, ev.Gev))
    sr = np.empty((k, ev.Gev))
    for ri in range(k):
        r = R[ri]
        mr[ri] = dot_seq(ev.mean, r)
        ss = None
        for j in range(N):
            u = ev.L[:, j, j] * r[j]                    # u_j = sum_{i>=j} L_ij r_i, ascending i
            for i in range(j + 1, N):
                u = u + ev.L[:, i, j] * r[i]
            ss = u * u if ss is None else ss + u * u
        sr[ri] = np.sqrt(ss)
    sr[:, ev.degenerate] = 0.0
    thr = multiplier * sr
    thr[:, ~ev.live] = -1.0
    return mr, sr, thr


def tile_bounds(queries, R: np.ndarray, tile_size: int = 256):
    """per tile and vector [min, max] of q^T r over the tile's queries."""
    q = np.asarray(queries, dtype=np.float32).astype(np.float64)
    B = q.shape[0]
    if B % tile_size:
        raise ValueError("batch size must be a multiple of tile_size (SPEC.md:441-442)")
    T = B // tile_size
    k = R.shape[0]
    lo = np.empty((T, k))
    hi = np.empty((T, k))
    for ri in range(k):
        p = dot_seq(q, R[ri]).reshape(T, tile_size)
        lo[:, ri] = p.min(axis=1)
        hi[:, ri] = p.max(axis=1)
    return lo, hi


def cull_mask(lo, hi, mr, thr):
    """culled iff for ANY vector max(lo - m_r, m_r - hi, 0) > multiplier*sigma_r.

    Written as (lo - m_r > thr) | (m_r - hi > thr), which is the same predicate exactly (max is a
    selection). Equality is kept. thr = -1 marks never-evaluated Gaussians (always culled).
    Returns kept[T, Gev] (bool)."""
    T, k = lo.shape
    Gev = mr.shape[1]
    kept = np.ones((T, Gev), dtype=bool)
    for ri in range(k):
        d1 = lo[:, ri][:, None] - mr[ri][None, :]
        d2 = mr[ri][None, :] - hi[:, ri][:, None]
        culled = (d1 > thr[ri][None, :]) | (d2 > thr[ri][None, :])
        kept &= ~culled
    kept &= (thr[0] >= 0.0)[None, :]
    return kept


def cull_csr(lo, hi, mr, thr, block: int = 256):
    """Candidate lists as CSR: offsets[T+1] (int64), idx (int32, ascending per tile)."""
    T = lo.shape[0]
    counts = np.zeros(T, np.int64)
    parts = []
    for t0 in range(0, T, block):
        kept = cull_mask(lo[t0:t0 + block], hi[t0:t0 + block], mr, thr)
        counts[t0:t0 + block] = kept.sum(axis=1)
        for row in kept:
            parts.append(np.flatnonzero(row).astype(np.int32))
    offsets = np.zeros(T + 1, np.int64)
    offsets[1:] = np.cumsum(counts)
    idx = np.concatenate(parts) if parts else np.zeros(0, np.int32)
    return offsets, idx


def brute_force_active(queries, ev: EvalSet, epsilon: float):
    """components with eval_gaussian >= epsilon at some tile query."""
    q = np.asarray(queries, np.float64)
    out = []
    for e in range(ev.Gev):
        if not ev.live[e]:
            continue
        g = eval_gaussian(ev.mean[e], ev.L[e], q)
        if np.any(g >= epsilon):
            out.append(e)
    return np.asarray(out, dtype=np.int64)


def all_active_csr(T: int, ev: EvalSet):
    """Culling disabled: every live Gaussian is a candidate of every tile (finite_diff_grad, --no-cull)."""
    live = np.flatnonzero(ev.live).astype(np.int32)
    offsets = np.arange(T + 1, dtype=np.int64) * live.size
    return offsets, np.tile(live, T)


# ----------------------------------------------------------------------------------------------
# forward / loss / backward
# ----------------------------------------------------------------------------------------------
def _pair_terms(ev: EvalSet, cand, qt):
    d = qt[None, :, :] - ev.mean[cand][:, None, :]
    z = solve_lower(ev.L[cand][:, None, :, :], d)          # [C, TQ, N]
    s = np.sum(z * z, axis=-1)
    g = np.exp(-0.5 * s)
    return z, s, g


def forward(queries, ev: EvalSet, offsets, idx, tile_size: int = 256, chunk: int = 512):
    """eval_mixture at every query over its tile's candidates (Eq. 8)."""
    q = np.asarray(queries, np.float32).astype(np.float64)
    B = q.shape[0]
    T = B // tile_size
    pred = np.zeros((B, 3))
    for t in range(T):
        cand = idx[offsets[t]:offsets[t + 1]]
        qt = q[t * tile_size:(t + 1) * tile_size]
        acc = np.zeros((tile_size, 3))
        for c0 in range(0, cand.size, chunk):
            c = cand[c0:c0 + chunk]
            _, _, g = _pair_terms(ev, c, qt)
            acc += g.T @ ev.a[c]
        pred[t * tile_size:(t + 1) * tile_size] = acc
    return pred


def loss_rel_l2(pred, target, eps: float = 0.01, n_total: int | None = None):
    """mean over entries of (p - t)^2 / (sg(p)^2 + eps), denominator detached.

    Returns (loss, dpred [B,3], ell [B]) where ell is each query's share of the loss and
    dpred = 2 (p - t) / (p^2 + eps) / (3 * n_total)."""
    p = np.asarray(pred, np.float64)
    t = np.asarray(target, np.float64)
    n = p.shape[0] if n_total is None else n_total
    den = p * p + eps
    diff = p - t
    ell = np.sum(diff * diff / den, axis=1) / (3.0 * n)
    dpred = 2.0 * diff / den / (3.0 * n)
    return float(np.sum(ell)), dpred, ell


N_STATS = 3   # density-control statistics per evaluated Gaussian: [sum g*ell_q, sum |coef|*||z||, pairs]


def backward_accum(queries, dpred, ell, ev: EvalSet, offsets, idx, tile_size: int = 256, chunk: int = 512):
    """Per evaluated Gaussian sufficient statistics of the pair terms.

    coef = -g (dp . a); S = sum coef z z^T; t = sum coef z; gA = sum g dp;
    density stats (north_star addition, parity pinned only to this oracle):
    loss_share = sum g * ell_q, grad_proxy = sum |coef| * ||z||, pairs = number of (query, e) pairs."""
    q = np.asarray(queries, np.float32).astype(np.float64)
    N = ev.mean.shape[1]
    B = q.shape[0]
    T = B // tile_size
    S = np.zeros((ev.Gev, N, N))
    tv = np.zeros((ev.Gev, N))
    gA = np.zeros((ev.Gev, 3))
    stats = np.zeros((ev.Gev, N_STATS))
    for t in range(T):
        cand = idx[offsets[t]:offsets[t + 1]]
        sl = slice(t * tile_size, (t + 1) * tile_size)
        qt, dpt, et = q[sl], dpred[sl], ell[sl]
        for c0 in range(0, cand.size, chunk):
            c = cand[c0:c0 + chunk]
            z, s, g = _pair_terms(ev, c, qt)
            h = dpt @ ev.a[c].T                            # [TQ, C]
            coef = -g * h.T                                # [C, TQ]
            S[c] += np.einsum("cq,cqi,cqj->cij", coef, z, z)
            tv[c] += np.einsum("cq,cqi->ci", coef, z)
            gA[c] += g @ dpt
            stats[c, 0] += g @ et
            stats[c, 1] += np.sum(np.abs(coef) * np.sqrt(s), axis=1)
            stats[c, 2] += tile_size
    return S, tv, gA, stats


def _chol_chain(GL, L, n):
    """d loss / d chol_raw from d loss / d L (lower): diag * L_ii, off-diag * (1 - L_ij^2) / 2."""
    out = np.zeros(GL.shape[:-2] + (n_chol(n),))
    for i in range(n):
        for j in range(i + 1):
            if i == j:
                out[..., tri(i, j)] = GL[..., i, i] * L[..., i, i]
            else:
                out[..., tri(i, j)] = GL[..., i, j] * (1.0 - L[..., i, j] ** 2) * 0.5
    return out


def epilogue(mix: OMixture, ev: EvalSet, S, tv, gA):
    """Raw-parameter gradients (incl. the child -> parent cross terms of :266).

    Per evaluated Gaussian: G_L = -tril(L^-T S), dm = -L^-T t. Child e = G + i with parent L,
    relative U, m_u: dU = tril(L^T G_Lc), dm_u = L^T dm_c, and the parent gains
    tril(G_Lc U^T) + tril(dm_c m_u^T) on L and dm_c on its mean."""
    N, G = mix.n_dims, mix.G
    ms, cs, cols, amp = raw_slices(N)
    Linv = np.linalg.inv(ev.L[ev.live]) if np.any(ev.live) else None
    GL = np.zeros((ev.Gev, N, N))
    dm = np.zeros((ev.Gev, N))
    if Linv is not None:
        LinvT = np.swapaxes(Linv, -1, -2)
        GL[ev.live] = -np.tril(LinvT @ S[ev.live])
        dm[ev.live] = -np.einsum("eij,ej->ei", LinvT, tv[ev.live])
    gp = np.zeros((G, raw_width(N)))
    gc = np.zeros((G, raw_width(N)))

    def color_amp(rows, gAe, out):
        c = sigmoid(rows[:, cols])
        alpha = amp_activate(rows[:, amp], mix.amp_mode)
        out[:, cols] = gAe * alpha[:, None] * c * (1.0 - c)
        dalpha = np.sum(gAe * c, axis=1)
        out[:, amp] = dalpha * (alpha if mix.amp_mode == BRIGHTNESS else alpha * (1.0 - alpha))

    GLp = GL[:G].copy()
    dmp = dm[:G].copy()
    color_amp(mix.params, gA[:G], gp)
    if ev.Gev == 2 * G:
        GLc, dmc = GL[G:], dm[G:]
        Lp, U, mu = ev.Lp, ev.Uc, ev.mu
        GLp += np.tril(GLc @ np.swapaxes(U, -1, -2)) + np.tril(dmc[:, :, None] * mu[:, None, :])
        dmp += dmc
        dU = np.tril(np.swapaxes(Lp, -1, -2) @ GLc)
        gc[:, ms] = np.einsum("eki,ek->ei", Lp, dmc)
        gc[:, cs] = _chol_chain(dU, U, N)
        color_amp(mix.child, gA[G:], gc)
        gc[~(mix.has_child & ~mix.frozen)] = 0.0
    gp[:, ms] = dmp
    gp[:, cs] = _chol_chain(GLp, ev.Lp, N)
    return gp, gc


def fwd_bwd(mix: OMixture, queries, targets, R, *, tile_size=256, multiplier=3.0, eps=0.01,
            cull=True, n_total=None):
    """One full oracle step: eval set, projections, tile bounds, cull, forward, loss, backward."""
    ev = build_eval_set(mix)
    B = np.asarray(queries).shape[0]
    T = B // tile_size
    if cull:
        mr, sr, thr = project_components(ev, R, multiplier)
        lo, hi = tile_bounds(queries, R, tile_size)
        offsets, idx = cull_csr(lo, hi, mr, thr)
    else:
        offsets, idx = all_active_csr(T, ev)
    pred = forward(queries, ev, offsets, idx, tile_size)
    loss, dpred, ell = loss_rel_l2(pred, targets, eps, n_total)
    S, tv, gA, stats = backward_accum(queries, dpred, ell, ev, offsets, idx, tile_size)
    gp, gc = epilogue(mix, ev, S, tv, gA)
    return dict(ev=ev, offsets=offsets, idx=idx, pred=pred, loss=loss, dpred=dpred, ell=ell,
                grad_parent=gp, grad_child=gc, stats=stats)


def predict_all(mix: OMixture, queries):
    """Prediction with culling disabled (finite_diff_grad re-runs the full forward)."""
    ev = build_eval_set(mix)
    q = np.asarray(queries, np.float64)
    live = np.flatnonzero(ev.live)
    if not live.size:
        return np.zeros((q.shape[0], 3))
    _, _, g = _pair_terms(ev, live, q)
    return g.T @ ev.a[live]


def finite_diff_grad(mix: OMixture, queries, targets, which: str, comp: int, entry: int,
                     h: float = 1e-4, eps: float = 0.01):
    """central difference (loss(θ+h) - loss(θ-h)) / 2h, culling disabled.

    The loss's denominator is detached, so the differenced function keeps the
    denominator at the unperturbed prediction: this is the function whose gradient `backward`
    returns, which is what "gradient oracle tests pin the chosen convention" asks."""
    t = np.asarray(targets, np.float64)
    p0 = predict_all(mix, queries)
    den = p0 * p0 + eps

    def shifted(delta):
        m2 = OMixture(mix.n_dims, mix.amp_mode, mix.params.copy(), mix.child.copy(),
                      mix.has_child.copy(), mix.frozen.copy())
        arr = m2.params if which == "parent" else m2.child
        arr[comp, entry] += delta
        d = predict_all(m2, queries) - t
        return float(np.mean(d * d / den))
    return (shifted(h) - shifted(-h)) / (2.0 * h)


# ----------------------------------------------------------------------------------------------
# trainer pieces
# ----------------------------------------------------------------------------------------------
def block_lr(n: int, lr_mean=2e-3, lr_chol=5e-3, lr_color=1e-2, lr_amp=1e-2):
    """Per-element learning rates for a raw row (SPEC.md:386 per-block defaults)."""
    ms, cs, cols, amp = raw_slices(n)
    lr = np.empty(raw_width(n))
    lr[ms], lr[cs], lr[cols], lr[amp] = lr_mean, lr_chol, lr_color, lr_amp
    return lr


def adam_step(p, g, m1, m2, step, lr, b1=0.9, b2=0.999, eps=1e-8):
    """standard bias-corrected Adam; returns (p, m1, m2). float32 arithmetic."""
    p, g, m1, m2 = (np.asarray(x, np.float32) for x in (p, g, m1, m2))
    lr = np.asarray(lr, np.float32)
    b1, b2, eps = np.float32(b1), np.float32(b2), np.float32(eps)
    m1 = b1 * m1 + (np.float32(1) - b1) * g
    m2 = b2 * m2 + (np.float32(1) - b2) * g * g
    c1 = np.float32(1.0 - float(b1) ** step)
    c2 = np.float32(1.0 - float(b2) ** step)
    p = p - lr * (m1 / c1) / (np.sqrt(m2 / c2) + eps)
    return p, m1, m2


def default_threshold(amp_mode: int) -> float:
    """t = 0.1 opacity / 0.01 brightness."""
    return 0.1 if amp_mode == OPACITY else 0.01


def spawn_child_rows(n: int, count: int, amp_mode: int, t: float, rng) -> np.ndarray:
    """U = I, m_u = 0, color_raw uniform in +-0.1, activated amp = t/10."""
    ms, cs, cols, amp = raw_slices(n)
    rows = np.zeros((count, raw_width(n)))
    rows[:, cols] = rng.uniform(-0.1, 0.1, size=(count, 3))
    rows[:, amp] = amp_inverse(t / 10.0, amp_mode)
    return rows


def check_materialize(mix: OMixture, t: float):
    """components whose live child has activated amplitude >= t."""
    ms, cs, cols, amp = raw_slices(mix.n_dims)
    alpha = amp_activate(mix.child[:, amp], mix.amp_mode)
    return np.flatnonzero(mix.has_child & ~mix.frozen & (alpha >= t))


def materialize_rows(mix: OMixture, indices):
    """new standalone rows for the given children (composed mean and factor,
    activations inverted with off-diagonal clamping). Returns (rows [len, R], n_clamped)."""
    N = mix.n_dims
    ms, cs, cols, amp = raw_slices(N)
    indices = np.asarray(indices, np.int64)
    Lp = activate_cholesky(mix.params[indices][:, cs], N)
    U = activate_cholesky(mix.child[indices][:, cs], N)
    mc, Lc = compose_child(mix.params[indices][:, ms], Lp, mix.child[indices][:, ms], U)
    rows = np.zeros((indices.size, raw_width(N)))
    rows[:, ms] = mc
    rows[:, cs], clamped = inverse_activate_cholesky(Lc, N)
    rows[:, cols] = mix.child[indices][:, cols]
    rows[:, amp] = mix.child[indices][:, amp]
    return rows, clamped


# ----------------------------------------------------------------------------------------------
# synthetic inputs; shared by tests, smoke() and bench.py
# ----------------------------------------------------------------------------------------------
def nn_sigma0(means, sample: int = 512, seed: int = 0) -> float:
    """sigma_0 = half the mean nearest-neighbour distance among the means,
    estimated on a fixed subsample of at most `sample` points against all points."""
    m = np.asarray(means, np.float64)
    G = m.shape[0]
    if G < 2:
        return 0.1
    rng = np.random.default_rng(seed)
    sel = rng.choice(G, size=min(G, sample), replace=False)
    d = []
    for i in sel:
        dd = np.sum((m - m[i]) ** 2, axis=1)
        dd[i] = np.inf
        d.append(math.sqrt(float(dd.min())))
    return 0.5 * float(np.mean(d))


def synthetic_mixture(n: int, G: int, seed: int = 0, *, amp_mode: int = BRIGHTNESS, children: bool = False,
                      sigma0: float | None = None):
    """Seeded synthetic mixture of the named shape: means U[0,1)^N, diagonal raw
    ln(sigma0) + U[-1/2, 1/2], off-diagonal raw N(0, sigma0^2), color_raw N(0,1), amp_raw
    N(ln 0.1, 0.5^2) (brightness) / N(-2, 0.5^2) (opacity). Children: m_u N(0, 0.3^2),
    rel_chol_raw N(0, 0.1^2), amp at t/10. Returned as float32 rows (the device precision)."""
    rng = np.random.default_rng(seed)
    ms, cs, cols, amp = raw_slices(n)
    R = raw_width(n)
    params = np.zeros((G, R))
    params[:, ms] = rng.random((G, n))
    s0 = nn_sigma0(params[:, ms]) if sigma0 is None else sigma0
    for i in range(n):
        for j in range(i + 1):
            if i == j:
                params[:, cs.start + tri(i, j)] = math.log(s0) + rng.uniform(-0.5, 0.5, G)
            else:
                params[:, cs.start + tri(i, j)] = rng.normal(0.0, s0, G)
    params[:, cols] = rng.normal(0.0, 1.0, (G, 3))
    params[:, amp] = rng.normal(math.log(0.1) if amp_mode == BRIGHTNESS else -2.0, 0.5, G)
    child = np.zeros((G, R))
    has_child = np.zeros(G, bool)
    if children:
        child[:, ms] = rng.normal(0.0, 0.3, (G, n))
        child[:, cs] = rng.normal(0.0, 0.1, (G, n_chol(n)))
        child[:, cols] = rng.normal(0.0, 1.0, (G, 3))
        child[:, amp] = amp_inverse(default_threshold(amp_mode) / 10.0, amp_mode) + rng.normal(0.0, 0.5, G)
        has_child[:] = True
    return OMixture(n, amp_mode, params.astype(np.float32).astype(np.float64),
                    child.astype(np.float32).astype(np.float64), has_child, np.zeros(G, bool)), s0


def synthetic_queries(n: int, B: int, seed: int = 1, *, regime: str = "R", tile_size: int = 256,
                      spread: float = 0.01):
    """Queries of the two SURVEY.md §8(d) regimes (float32):
    R -- U[0,1)^N, stable-sorted by dim 0, contiguous tiles (the reference sampler);
    C -- coherent tiles: per tile a centre U[0,1)^N plus N(0, spread^2), clipped to [0,1]."""
    rng = np.random.default_rng(seed)
    if regime == "R":
        q = rng.random((B, n))
        q = q[np.argsort(q[:, 0], kind="stable")]
    elif regime == "C":
        T = B // tile_size
        centre = rng.random((T, 1, n))
        q = np.clip(centre + rng.normal(0.0, spread, (T, tile_size, n)), 0.0, 1.0).reshape(B, n)
    elif regime == "G":
        return gbuffer_queries(n, B, seed, tile_size)
    else:
        raise ValueError(regime)
    return q.astype(np.float32)


def gbuffer_queries(n: int, B: int, seed: int = 1, tile_size: int = 256):
    """Oracle copy of paper_2405_20067_b200.datasets.gbuffer_queries (test infrastructure). Regime G: G-buffer-like queries on a 2-D manifold in N-D. Pixels of a
    W x H image (W = 2^ceil(log2(B)/2)), grouped into square tiles of tile_size pixels (16 x 16 at 256):
    position (u, v, height(u, v)) | view direction to a fixed camera (mapped to [0,1]) | albedo(u, v) |
    roughness(u, v) | further smooth "variable" dims for N > 10; the first N features, float32. Tiles
    are tight in every dimension, so culling keeps only a few tens of Gaussians per tile and the
    binning (K4), not the pair loops, dominates the step."""
    rng = np.random.default_rng(seed)
    ph = rng.uniform(0.0, 1.0, 16)
    W = 1 << int(math.ceil(math.log2(max(B, 1)) / 2))
    H = B // W
    ts = int(round(math.sqrt(tile_size)))
    if ts * ts != tile_size or W % ts or H % ts or W * H != B:
        raise ValueError("regime G needs B = W * H with square tiles dividing the image")
    ty, tx, j, i = np.meshgrid(np.arange(H // ts), np.arange(W // ts), np.arange(ts), np.arange(ts), indexing="ij")
    px, py = (tx * ts + i).reshape(-1), (ty * ts + j).reshape(-1)
    u, v = (px + 0.5) / W, (py + 0.5) / H
    tau = 2.0 * np.pi
    h = 0.5 + 0.2 * np.sin(tau * (1.3 * u + ph[0])) * np.cos(tau * (0.9 * v + ph[1])) + 0.1 * np.sin(tau * (3.1 * u + 2.7 * v))
    cam = np.array([0.5, -0.8, 1.6])
    d = cam[None, :] - np.stack([u, v, h], 1)
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    feats = [u, v, h, 0.5 * (d[:, 0] + 1), 0.5 * (d[:, 1] + 1), 0.5 * (d[:, 2] + 1)]
    for c in range(3):
        feats.append(0.5 + 0.4 * np.sin(tau * (2.0 * u + ph[2 + c])) * np.cos(tau * (1.5 * v + ph[5 + c])))
    feats.append(0.5 + 0.45 * np.sin(tau * (u + v + ph[8])))
    k = 0
    while len(feats) < n:
        k += 1
        feats.append(0.5 + 0.4 * np.sin(tau * (k * u + (k + 1) * v + ph[9 + k % 7])))
    return np.stack(feats[:n], 1).astype(np.float32)


def gbuffer_mixture(n: int, G: int, seed: int = 0, *, sigma0: float = 0.005, amp_mode: int = BRIGHTNESS):
    """Oracle copy of paper_2405_20067_b200.datasets.gbuffer_mixture (test infrastructure). Mixture for regime G: means at the manifold features of G random pixels of a 1024 x 1024 image
    (gbuffer_queries' geometry), diagonal raw ln(sigma0) + U[-1/2, 1/2], off-diagonal raw N(0, sigma0^2),
    colour N(0, 1), amplitude as synthetic_mixture. Float32 rows."""
    rng = np.random.default_rng(seed)
    feats = gbuffer_queries(n, 1 << 20, seed=1)
    ms, cs, cols, amp = raw_slices(n)
    R = raw_width(n)
    params = np.zeros((G, R))
    params[:, ms] = feats[rng.integers(0, feats.shape[0], G)]
    for i in range(n):
        for j in range(i + 1):
            if i == j:
                params[:, cs.start + tri(i, j)] = math.log(sigma0) + rng.uniform(-0.5, 0.5, G)
            else:
                params[:, cs.start + tri(i, j)] = rng.normal(0.0, sigma0, G)
    params[:, cols] = rng.normal(0.0, 1.0, (G, 3))
    params[:, amp] = rng.normal(math.log(0.1) if amp_mode == BRIGHTNESS else -2.0, 0.5, G)
    return OMixture(n, amp_mode, params.astype(np.float32).astype(np.float64), np.zeros((G, R)),
                    np.zeros(G, bool), np.zeros(G, bool))

def synthetic_targets(B: int, seed: int = 3):
    return np.random.default_rng(seed).random((B, 3)).astype(np.float32)


# ----------------------------------------------------------------------------------------------
# device sampler and shading toy target; oracle copies of
# csrc/ndg_sample.cu for the GPU parity tests (test infrastructure)
# ----------------------------------------------------------------------------------------------
_M0, _M1, _W0, _W1 = np.uint64(0xD2511F53), np.uint64(0xCD9E8D57), 0x9E3779B9, 0xBB67AE85
_U32 = np.uint64(0xFFFFFFFF)


def philox4x32_10(c0, c1, c2, c3, k0, k1):
    """Philox4x32-10 (Salmon, Moraes, Dror, Shaw, SC'11 -- the Random123 generator); vectorised over
    counters. Pinned by the Random123 known-answer vectors in tests/test_oracle_kats.py."""
    c = [np.asarray(x, np.uint64) & _U32 for x in (c0, c1, c2, c3)]
    k0, k1 = int(k0) & 0xFFFFFFFF, int(k1) & 0xFFFFFFFF
    for _ in range(10):
        p0, p1 = _M0 * c[0], _M1 * c[2]
        c = [(p1 >> np.uint64(32)) ^ c[1] ^ np.uint64(k0), p1 & _U32, (p0 >> np.uint64(32)) ^ c[3] ^ np.uint64(k1),
             p0 & _U32]
        k0, k1 = (k0 + _W0) & 0xFFFFFFFF, (k1 + _W1) & 0xFFFFFFFF
    return [x.astype(np.uint32) for x in c]


def _sample_key(seed: int, draw: int):
    return seed & 0xFFFFFFFF, ((seed >> 32) ^ (draw >> 32)) & 0xFFFFFFFF


def sample_spacings_fx(B: int, seed: int, draw: int) -> np.ndarray:
    """The B + 1 exponential spacings E_i = -log(u_i) in 32.32 fixed point (int64), u_i a 53-bit
    uniform in (0, 1] from Philox stream 0 at counter (i, 0, draw)."""
    i = np.arange(B + 1, dtype=np.uint64)
    k0, k1 = _sample_key(seed, draw)
    r = philox4x32_10(i & _U32, i >> np.uint64(32), 0, draw & 0xFFFFFFFF, k0, k1)
    u = ((r[0] >> 5).astype(np.float64) * 67108864.0 + (r[1] >> 6).astype(np.float64) + 1.0) / 9007199254740992.0
    return np.rint(-np.log(u) * 4294967296.0).astype(np.int64)


def sample_batch(n: int, B: int, tile: int, seed: int, draw: int, rank: int = 0, world: int = 1) -> np.ndarray:
    """Oracle of ndg_sample_batch: the global batch sorted by dimension 0 (uniform order statistics
    S_k / S_{B+1}, exact int64 prefix sums), other dimensions iid 24-bit uniforms from Philox streams
    1, 3, 5, ... (four dimensions per call); returns the rows of the tiles t % world == rank."""
    E = sample_spacings_fx(B, seed, draw)
    S = np.cumsum(E)
    x0 = np.minimum((S[:B].astype(np.float64) / float(S[B])).astype(np.float32), np.float32(0.99999994))
    q = np.empty((B, n), np.float32)
    q[:, 0] = x0
    k = np.arange(B, dtype=np.uint64)
    k0, k1 = _sample_key(seed, draw)
    for d in range(1, n, 4):
        r = philox4x32_10(k & _U32, k >> np.uint64(32), 1 + 2 * (d // 4), draw & 0xFFFFFFFF, k0, k1)
        for j in range(4):
            if d + j < n:
                q[:, d + j] = (r[j] >> 8).astype(np.float32) * np.float32(1.0 / 16777216.0)
    T = B // tile
    return q.reshape(T, tile, n)[rank::world].reshape(-1, n)


def shading_toy(q, freq, phase) -> np.ndarray:
    """Oracle of ndg_shading_target / datasets.ShadingToyTarget in float64."""
    q = np.asarray(q, np.float64)
    n = q.shape[1]
    pos = q[:, :3]
    shade = 0.55 + 0.45 * np.prod(np.sin(2 * np.pi * np.asarray(freq) * pos + np.asarray(phase)), axis=1, keepdims=True)
    alb = q[:, 6:9] if n >= 9 else np.full((q.shape[0], 3), 0.6)
    rough = q[:, 9:10] if n >= 10 else np.full((q.shape[0], 1), 0.5)
    v = np.concatenate([2.0 * q[:, 3:min(n, 6)] - 1.0, np.ones((q.shape[0], max(0, 6 - n)))], 1)
    v = v / np.maximum(np.linalg.norm(v, axis=1, keepdims=True), 1e-6)
    refl = np.stack([np.sin(2 * np.pi * pos[:, 0]), np.cos(2 * np.pi * pos[:, 1]), 0.5 + pos[:, 2]], 1)
    refl = refl / np.linalg.norm(refl, axis=1, keepdims=True)
    lobe = np.maximum((v * refl).sum(1, keepdims=True), 0.0) ** (2.0 + 40.0 * (1.0 - rough))
    return alb * shade * 0.6 + 0.4 * lobe
