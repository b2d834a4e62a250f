"""Tiling-order study (CPU, NumPy; "tile tightness drives the cull rate").

cfg2 shapes: 100k-Gaussian synthetic mixture (N = 10), 2^20 uniform queries, 256-query tiles, k = 16 projection
vectors, multiplier 3. Kept fraction of (tile, Gaussian) pairs on 48 evenly spaced tiles for the reference's
dim-0 sort against Morton (Z-order) sorts and a kd split on the widest dimension. The cull test is
the oracle's (project_components / tile bounds / SPEC.md:198-206). Tuning aid, not a test."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import ndg_oracle as O  # noqa: E402  (checker / study only)

n, G, B, TILE = 10, 100_000, 1 << 20, 256
om, _ = O.synthetic_mixture(n, G, seed=0)
ev = O.build_eval_set(om)
R = O.make_projection_set(n, 16, 2)
mr, sr, thr = O.project_components(ev, R, 3.0)
q = np.random.default_rng(1).random((B, n))


def kept(qs, ntiles=48):
    sel = np.linspace(0, B // TILE - 1, ntiles).astype(int)
    tot = 0
    for t in sel:
        p = qs[t * TILE:(t + 1) * TILE] @ R.T
        lo, hi = p.min(0), p.max(0)
        d = np.maximum(np.maximum(lo[:, None] - mr, mr - hi[:, None]), 0)
        tot += (d <= thr).all(0).sum()
    return tot / (ntiles * G)


def morton(x01, bits):
    x = np.minimum((x01 * (1 << bits)).astype(np.int64), (1 << bits) - 1)
    code = np.zeros(len(x01), dtype=np.int64)
    for b in range(bits - 1, -1, -1):
        for d in range(n):
            code = code * 2 + ((x[:, d] >> b) & 1)
    return code


def kd(x):
    if len(x) <= TILE:
        return [x]
    d = np.argmax(x.max(0) - x.min(0))
    o = np.argsort(x[:, d], kind="stable")
    h = len(x) // 2
    return kd(x[o[:h]]) + kd(x[o[h:]])


print(f"dim-0 sort (reference)  kept {kept(q[np.argsort(q[:, 0], kind='stable')]):.4f}")
for bits in (1, 2, 3, 6):
    print(f"Morton {bits} bit/dim        kept {kept(q[np.argsort(morton(q, bits), kind='stable')]):.4f}")
t0 = time.time()
print(f"kd split (widest dim)   kept {kept(np.concatenate(kd(q))):.4f}")
