"""Slicing ops of the gmm-core module, off the training hot path (host, float64, batched over
components): condition_gaussian and covariance_from_factor.

condition_gaussian realises the paper's "projection from N-D to 3D" (§4.2) as Gaussian conditioning
on the fixed dimensions b: with V = L L^T partitioned into free a / fixed b blocks,
    mean   m_a + V_ab V_bb^-1 (x_b - m_b)
    cov    V_aa - V_ab V_bb^-1 V_ba
    weight exp(-1/2 (x_b - m_b)^T V_bb^-1 (x_b - m_b))
so that weight * N_a(x_a; mean, cov) (unnormalised, peak 1) equals the joint eval_gaussian on the slice.
V_bb is factored by Cholesky (never inverted); a non-positive-definite V_bb raises
DegenerateSliceError.
"""
from __future__ import annotations

import numpy as np

from .errors import DegenerateSliceError
from .gmm import raw_slices
from .trainer import _activate


def covariance_from_factor(L) -> np.ndarray:
    """V = L L^T, exact product, symmetric by construction; L [..., N, N]."""
    L = np.tril(np.asarray(L, dtype=np.float64))
    V = L @ np.swapaxes(L, -1, -2)
    return 0.5 * (V + np.swapaxes(V, -1, -2))


def condition_factor(mean, L, fixed_dims, fixed_values):
    """condition_gaussian on activated parameters: mean [..., N], L [..., N, N] lower; returns
    (mean_a [..., Na], cov_a [..., Na, Na], weight [...])."""
    mean = np.asarray(mean, dtype=np.float64)
    N = mean.shape[-1]
    b = sorted({int(d) for d in np.atleast_1d(fixed_dims)})
    if not b or len(b) >= N or b[0] < 0 or b[-1] >= N:
        raise ValueError("fixed_dims must be a strict, nonempty subset of range(N)")
    a = [d for d in range(N) if d not in b]
    xb = np.asarray(fixed_values, dtype=np.float64)
    if xb.shape[-1] != len(b):
        raise ValueError("fixed_values must have one entry per fixed dimension")
    V = covariance_from_factor(L)
    Vaa = V[..., a, :][..., :, a]
    Vab = V[..., a, :][..., :, b]
    Vbb = V[..., b, :][..., :, b]
    try:
        Cb = np.linalg.cholesky(Vbb)
    except np.linalg.LinAlgError as e:
        raise DegenerateSliceError("fixed-block covariance V_bb is singular") from e
    if not np.all(np.isfinite(Cb)) or np.any(np.diagonal(Cb, axis1=-2, axis2=-1) <= 0):
        raise DegenerateSliceError("fixed-block covariance V_bb is singular")
    db = xb - mean[..., b]
    # Vbb^-1 db and Vbb^-1 Vba through the Cholesky factor (two triangular solves each)
    y = np.linalg.solve(Cb, db[..., None])                       # Cb y = db
    K = np.linalg.solve(Cb, np.swapaxes(Vab, -1, -2))            # Cb K = Vba
    mean_a = mean[..., a] + (np.swapaxes(K, -1, -2) @ y)[..., 0]
    cov_a = Vaa - np.swapaxes(K, -1, -2) @ K
    cov_a = 0.5 * (cov_a + np.swapaxes(cov_a, -1, -2))
    weight = np.exp(-0.5 * np.sum(y[..., 0] ** 2, axis=-1))
    return mean_a, cov_a, weight


def condition_gaussian(params, n_dims: int, fixed_dims, fixed_values):
    """`params` are raw GaussianParams rows [..., N + P + 4] (mean_raw | chol_raw | ...);
    returns (conditional mean, conditional covariance, weight) per row."""
    p = np.asarray(params, dtype=np.float64)
    ms, cs, _, _ = raw_slices(n_dims)
    return condition_factor(p[..., ms], _activate(p[..., cs], n_dims), fixed_dims, fixed_values)
