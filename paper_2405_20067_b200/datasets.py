"""Batch tiling and seeded synthetic inputs of the named shapes (reference module datasets,
/root/reference/SPEC.md:402-498; synthetic recipe SURVEY.md §8(d)).

Only what the hot path needs: the tile definition of sample_batch (queries sorted by the first
dimension, contiguous tiles of tile_size) and the synthetic mixture / query /
target generators the benchmark and the fit loop use. The generators are host-side NumPy (not on
the timed path); tests/test_datasets.py checks they match the oracle's copies value for value.
"""
from __future__ import annotations

import math

import numpy as np

from .gmm import BRIGHTNESS, n_chol, raw_slices, raw_width, tri


def nn_sigma0(means, sample: int = 512, seed: int = 0) -> float:
    """Half the mean nearest-neighbour distance among the means, on a fixed subsample."""
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


def default_threshold(amp_mode: int) -> float:
    """Materialisation threshold t: 0.1 opacity / 0.01 brightness."""
    return 0.01 if amp_mode == BRIGHTNESS else 0.1


def amp_inverse(alpha, amp_mode: int):
    alpha = np.asarray(alpha, dtype=np.float64)
    return np.log(alpha) if amp_mode == BRIGHTNESS else np.log(alpha) - np.log1p(-alpha)


def synthetic_mixture(n: int, G: int, seed: int = 0, *, amp_mode: int = BRIGHTNESS, children: bool = False,
                      sigma0: float | None = None):
    """Seeded synthetic mixture; returns dict(params, child, has_child, frozen),
    float32 rows, and sigma0."""
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
    return dict(params=params.astype(np.float32), child=child.astype(np.float32), has_child=has_child,
                frozen=np.zeros(G, bool)), s0


def sort_into_tiles(q: np.ndarray, targets: np.ndarray | None = None):
    """Tile formation of sample_batch: stable sort by the first (position) dimension."""
    order = np.argsort(q[:, 0], kind="stable")
    return (q[order], None if targets is None else targets[order])


def synthetic_queries(n: int, B: int, seed: int = 1, *, regime: str = "R", tile_size: int = 256,
                      spread: float = 0.01) -> np.ndarray:
    """R: U[0,1)^N sorted by dim 0 (the reference sampler); C: coherent tiles (centre + N(0, spread^2))."""
    rng = np.random.default_rng(seed)
    if regime == "R":
        q = rng.random((B, n))
        q = q[np.argsort(q[:, 0], kind="stable")]
    elif regime == "C":
        T = B // tile_size
        centre = rng.random((T, 1, n))
        q = np.clip(centre + rng.normal(0.0, spread, (T, tile_size, n)), 0.0, 1.0).reshape(B, n)
    else:
        raise ValueError(f"unknown regime {regime!r}")
    return q.astype(np.float32)


def synthetic_targets(B: int, seed: int = 3) -> np.ndarray:
    return np.random.default_rng(seed).random((B, 3)).astype(np.float32)
