"""Tensor-core feasibility study (CPU, NumPy): can the pair math run on tcgen05 in 3xTF32 and still
meet the 1e-4 block-relative tolerance? Emulates TF32 operand rounding (round-to-nearest, 10-bit
mantissa), the 3-product split (hi*hi + hi*lo + lo*hi) and float32 accumulation.

F1  forward exponent by the quadratic-feature expansion  s = <theta_e, phi(x - c_tile)>
F2  forward exponent via the linear z-GEMM               z = A_e [x - c_tile; 1]
B1  backward S, t via per-tile x-space moments M = sum_q w_eq phi(x_q - c_tile) (fp32 within a tile),
    re-centred and converted to z-space in float64.
Prints block-relative errors of pred and of the backward sufficient statistics vs float64.
"""
import sys, os
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import ndg_oracle as O


def tf32(a):
    a = np.asarray(a, np.float32)
    u = a.view(np.uint32).astype(np.uint64)
    u = ((u + 0x1000) & 0xFFFFE000).astype(np.uint32)
    return u.view(np.float32)


def split3_matmul(A, B):
    """A @ B with 3xTF32 operands and float32 accumulation."""
    A = np.asarray(A, np.float32); B = np.asarray(B, np.float32)
    ah, bh = tf32(A), tf32(B)
    al, bl = tf32(A - ah), tf32(B - bh)
    return (ah @ bh + ah @ bl + al @ bh).astype(np.float32)


def quad_features(X):
    """phi(x) = [x_i x_j (i<=j), x_i, 1]  (N(N+1)/2 + N + 1 features)."""
    n = X.shape[1]
    cols = [X[:, i] * X[:, j] for i in range(n) for j in range(i + 1)]
    return np.stack(cols + [X[:, i] for i in range(n)] + [np.ones(X.shape[0])], 1)


def theta(Linv, m):
    """s = (x-m)^T W (x-m) with W = Linv^T Linv, written against phi(x)."""
    n = m.shape[0]
    W = Linv.T @ Linv
    t = [W[i, j] * (1.0 if i == j else 2.0) for i in range(n) for j in range(i + 1)]
    lin = list(-2.0 * (W @ m))
    return np.array(t + lin + [m @ W @ m])


def study(n=10, G=1500, B=4096, regime="R", sigma0=0.15, seed=0):
    om, _ = O.synthetic_mixture(n, G, seed=seed, sigma0=sigma0)
    ev = O.build_eval_set(om)
    q = O.synthetic_queries(n, B, seed=seed + 1, regime=regime).astype(np.float64)
    t = O.synthetic_targets(B, seed=seed + 3).astype(np.float64)
    Linv = np.linalg.inv(ev.L)
    T = B // 256
    pred_ref = np.zeros((B, 3)); pred_f1 = np.zeros((B, 3)); pred_f2 = np.zeros((B, 3))
    for tt in range(T):
        sl = slice(tt * 256, (tt + 1) * 256)
        X = q[sl]; c = X.mean(0)
        Xc = X - c
        d = X[None] - ev.mean[:, None]                                   # [G,256,N]
        z = np.einsum("gij,gqj->gqi", Linv, d)
        s_ref = np.sum(z * z, -1)
        g_ref = np.exp(-0.5 * s_ref)
        pred_ref[sl] = g_ref.T @ ev.a
        Phi = quad_features(Xc)                                          # [256, F]
        Th = np.stack([theta(Linv[e], ev.mean[e] - c) for e in range(G)], 1)   # [F, G]
        s1 = split3_matmul(Phi, Th).astype(np.float64)                   # [256, G]
        pred_f1[sl] = np.exp(-0.5 * np.maximum(s1, 0)) @ ev.a
        Xh = np.concatenate([Xc, np.ones((256, 1))], 1)                  # [256, N+1]
        Aaug = np.concatenate([Linv, -np.einsum("gij,gj->gi", Linv, ev.mean - c)[:, :, None]], 2)  # [G,N,N+1]
        Z = split3_matmul(Xh, Aaug.reshape(G * n, n + 1).T).reshape(256, G, n).astype(np.float32)
        s2 = np.sum(Z * Z, -1, dtype=np.float32).astype(np.float64)
        pred_f2[sl] = np.exp(-0.5 * s2) @ ev.a
    rel = lambda a, b: float(np.linalg.norm(a - b) / np.linalg.norm(b))
    out = dict(regime=regime, sigma0=sigma0, pred_F1=rel(pred_f1, pred_ref), pred_F2=rel(pred_f2, pred_ref))
    # backward: S = sum coef z z^T, t = sum coef z  (exact, float64) vs per-tile fp32 moments (B1)
    loss, dpred, ell = O.loss_rel_l2(pred_ref, t)
    S_ref = np.zeros((G, n, n)); t_ref = np.zeros((G, n))
    M2 = np.zeros((G, n, n)); M1 = np.zeros((G, n)); M0 = np.zeros(G)
    for tt in range(T):
        sl = slice(tt * 256, (tt + 1) * 256)
        X = q[sl]; c = X.mean(0); Xc = X - c
        d = X[None] - ev.mean[:, None]
        z = np.einsum("gij,gqj->gqi", Linv, d)
        g = np.exp(-0.5 * np.sum(z * z, -1))
        coef = -g * (dpred[sl] @ ev.a.T).T                               # [G,256]
        S_ref += np.einsum("gq,gqi,gqj->gij", coef, z, z)
        t_ref += np.einsum("gq,gqi->gi", coef, z)
        # tensor-core moments of the centred queries (fp32 accumulate within the tile)
        Phi = quad_features(Xc).astype(np.float32)
        Mt = split3_matmul(coef.astype(np.float32), Phi).astype(np.float64)   # [G, F]
        P = n * (n + 1) // 2
        m2c = np.zeros((G, n, n))
        k = 0
        for i in range(n):
            for j in range(i + 1):
                m2c[:, i, j] = m2c[:, j, i] = Mt[:, k]; k += 1
        m1c = Mt[:, P:P + n]; m0 = Mt[:, P + n]
        # re-centre to global coordinates in float64: x = xc + c
        M2 += m2c + np.einsum("gi,j->gij", m1c, c) + np.einsum("i,gj->gij", c, m1c) + m0[:, None, None] * np.outer(c, c)
        M1 += m1c + m0[:, None] * c
        M0 += m0
    m = ev.mean
    D2 = M2 - np.einsum("gi,gj->gij", m, M1) - np.einsum("gi,gj->gij", M1, m) + M0[:, None, None] * np.einsum("gi,gj->gij", m, m)
    S_b1 = np.einsum("gia,gab,gjb->gij", Linv, D2, Linv)
    t_b1 = np.einsum("gia,ga->gi", Linv, M1 - M0[:, None] * m)
    out.update(S_B1=rel(S_b1, S_ref), t_B1=rel(t_b1, t_ref))
    # B1h (the K7-TC form): features of xhat = [x - 1/2; 1] (the z-GEMM's own features, no per-tile
    # centring), moments per 128-query block in 3xTF32/fp32, summed in float64, then
    # S~ = Ahat M Ahat^T and t~ = Ahat M[:, N] with Ahat = [L^-1 | L^-1 (1/2 - m)] in float64.
    Mh = np.zeros((G, n + 1, n + 1))
    for b0 in range(0, B, 128):
        sl = slice(b0, b0 + 128)
        X = q[sl]
        d = X[None] - ev.mean[:, None]
        z = np.einsum("gij,gqj->gqi", Linv, d)
        g = np.exp(-0.5 * np.sum(z * z, -1))
        coef = -g * (dpred[sl] @ ev.a.T).T
        Xh = np.concatenate([X - 0.5, np.ones((X.shape[0], 1))], 1)
        feats = np.stack([Xh[:, i] * Xh[:, j] for i in range(n + 1) for j in range(i + 1)], 1).astype(np.float32)
        Mt = split3_matmul(coef.astype(np.float32), feats).astype(np.float64)
        k = 0
        for i in range(n + 1):
            for j in range(i + 1):
                Mh[:, i, j] += Mt[:, k]
                if i != j:
                    Mh[:, j, i] += Mt[:, k]
                k += 1
    Ah = np.concatenate([Linv, np.einsum("gij,gj->gi", Linv, 0.5 - ev.mean)[:, :, None]], 2)
    S_h = np.einsum("gia,gab,gjb->gij", Ah, Mh, Ah)
    t_h = np.einsum("gia,ga->gi", Ah, Mh[:, :, n])
    out.update(S_B1h=rel(S_h, S_ref), t_B1h=rel(t_h, t_ref))
    return out


if __name__ == "__main__":
    for regime, s0 in (("R", 0.15), ("C", 0.15), ("R", 0.05), ("C", 0.05), ("R", 0.02), ("C", 0.02)):
        print(study(regime=regime, sigma0=s0), flush=True)
