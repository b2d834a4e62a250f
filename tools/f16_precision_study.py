"""Would K5's z-GEMM meet 1e-4 in kind::f16 (fp16 operands, fp32 accumulate) instead of kind::tf32?
NumPy emulation of the 3-product split hi*hi + hi*lo + lo*hi with IEEE fp16 operands (subnormals kept),
exact products and float32 accumulation, on the same mixtures as tools/tc_precision_study.py; the
query features may be scaled by 2^sx (and Ahat by 2^-sx) to keep the lo parts out of fp16's subnormal
range. Prints the block-relative pred error vs float64."""
import sys, os
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import ndg_oracle as O


def split16(a):
    a = np.asarray(a, np.float32)
    hi = a.astype(np.float16)
    lo = (a - hi.astype(np.float32)).astype(np.float16)
    return hi.astype(np.float64), lo.astype(np.float64)


def gemm16(A, B):
    ah, al = split16(A)
    bh, bl = split16(B)
    return (ah @ bh + ah @ bl + al @ bh).astype(np.float32)   # products exact, fp32-accumulated (approx.)


def study(n=10, G=1500, B=4096, regime="R", sigma0=0.15, sx=0, seed=0):
    om, _ = O.synthetic_mixture(n, G, seed=seed, sigma0=sigma0)
    ev = O.build_eval_set(om)
    q = O.synthetic_queries(n, B, seed=seed + 1, regime=regime).astype(np.float64)
    Linv = np.linalg.inv(ev.L)
    C = np.sqrt(0.5 * np.log2(np.e))
    pred_ref = np.zeros((B, 3)); pred = np.zeros((B, 3))
    for t0 in range(0, B, 256):
        X = q[t0:t0 + 256]
        d = X[None] - ev.mean[:, None]
        z = np.einsum("gij,gqj->gqi", Linv, d)
        pred_ref[t0:t0 + 256] = np.exp(-0.5 * np.sum(z * z, -1)).T @ ev.a
        Xh = np.concatenate([(X - 0.5) * 2.0 ** sx, np.ones((X.shape[0], 1)) * 2.0 ** sx], 1)
        Ah = np.concatenate([C * Linv, (C * np.einsum("gij,gj->gi", Linv, 0.5 - ev.mean))[:, :, None]], 2) * 2.0 ** -sx
        Z = gemm16(Xh, Ah.reshape(G * n, n + 1).T).reshape(-1, G, n).astype(np.float64)
        pred[t0:t0 + 256] = np.exp2(-np.sum(Z * Z, -1)) @ ev.a
    return float(np.linalg.norm(pred - pred_ref) / np.linalg.norm(pred_ref))


if __name__ == "__main__":
    for regime, s0 in (("R", 0.15), ("C", 0.15), ("R", 0.05), ("C", 0.05), ("R", 0.02)):
        print(regime, s0, {sx: f"{study(regime=regime, sigma0=s0, sx=sx):.2e}" for sx in (0, 4, 8)}, flush=True)
