"""The reference's module-level operations under their SPEC names (SPEC.md:63-101, 178-216, 253-281,
366-374), each executed by libndg.so kernels on the current CUDA device.

These are the drop-in surface a caller of `ndgauss` (gmm-core, culling and grad modules) uses; the
batched training step (`HotPath.fwd_bwd`) chains the same kernels without the per-call set-up. Inputs
may be numpy arrays or tensors; outputs are device tensors (float64 where the reference's quantity is
a float64 intermediate, float32 for predictions and gradients). Errors are the reference's classes
(errors.py:8-33). There is no CPU path: without libndg.so or a device every call raises.
"""
from __future__ import annotations

import numpy as np
import torch

from . import kernels as K
from .engine import (CandidateLists, GradientBuffer, HotPath, ProjectedBounds, ProjectionSet, TileBounds,
                     _p, _stream, adam_step, make_projection_set)
from .errors import InvalidParameterError
from .gmm import BRIGHTNESS, Mixture, n_chol, raw_width, tri

__all__ = ["activate_cholesky", "eval_gaussian", "eval_mixture", "compose_child", "make_projection_set",
           "project_components", "tile_bounds", "cull_tile", "brute_force_active", "loss_rel_l2", "backward",
           "finite_diff_grad", "adam_step"]


def _dev(device=None):
    if device is not None:
        return torch.device(device)
    if not torch.cuda.is_available():
        raise RuntimeError("ndgauss-b200 needs a CUDA device (no CPU fallback)")
    return torch.device("cuda", torch.cuda.current_device())


def _f32(x, dev):
    t = x if isinstance(x, torch.Tensor) else torch.from_numpy(np.asarray(x, dtype=np.float32))
    return t.to(device=dev, dtype=torch.float32).contiguous()


def _unpack(chol64, n):
    """packed row-major lower [..., P] -> dense [..., N, N]."""
    L = torch.zeros(chol64.shape[:-1] + (n, n), dtype=chol64.dtype, device=chol64.device)
    for i in range(n):
        for j in range(i + 1):
            L[..., i, j] = chol64[..., tri(i, j)]
    return L


def _pad_queries(q, tile):
    B = q.shape[0]
    pad = (-B) % tile
    if pad:
        q = torch.cat([q, q[-1:].expand(pad, q.shape[1])]) if B else torch.zeros(tile, q.shape[1], device=q.device)
    return q.contiguous(), B


def activate_cholesky(chol_raw, n_dims: int, device=None) -> torch.Tensor:
    """L[i,i] = exp(raw), L[i,j] = 2 sigmoid(raw) - 1 (i > j), float64 [..., N, N], via
    K1. A non-finite entry raises InvalidParameterError(component, entry) with `entry` the index into
    chol_raw and `component` the leading (flattened) index."""
    dev = _dev(device)
    n, P = int(n_dims), n_chol(int(n_dims))
    raw = _f32(chol_raw, dev)
    if raw.shape[-1] != P:
        raise ValueError(f"chol_raw must have length N(N+1)/2 = {P}")
    lead = raw.shape[:-1]
    raw = raw.reshape(-1, P)
    rows = torch.zeros(raw.shape[0], raw_width(n), dtype=torch.float32, device=dev)
    rows[:, n:n + P] = raw
    mix = Mixture(n, BRIGHTNESS, rows, torch.zeros_like(rows),
                  torch.zeros(rows.shape[0], dtype=torch.uint8, device=dev))
    hp = HotPath(n, device=dev)
    hp.reset_status()
    recs = hp.activate(mix)
    try:
        hp.check_status(mix)
    except InvalidParameterError as e:
        raise InvalidParameterError(f"non-finite chol_raw entry {e.entry - n}", component=e.component,
                                    block="chol", entry=e.entry - n) from None
    return _unpack(recs.chol64, n).reshape(lead + (n, n))


def eval_gaussian(g, x, device=None) -> torch.Tensor:
    """exp(-1/2 |z|^2) with L z = x - m (forward substitution) for one raw component
    row g [N + P + 4] at queries x [B, N]; returns float32 [B]. Runs the culling-off forward kernel on a
    one-component mixture with alpha = exp(0) = 1 and colour sigmoid(0) = 1/2, so g = 2 * pred exactly."""
    dev = _dev(device)
    row = _f32(g, dev).reshape(1, -1)
    x = _f32(x, dev)
    if x.ndim == 1:
        x = x[None]
    n = x.shape[1]
    if row.shape[1] != raw_width(n):
        raise ValueError(f"g must be a raw component row of length {raw_width(n)}")
    row = row.clone()
    row[0, n + n_chol(n):] = 0.0
    mix = Mixture(n, BRIGHTNESS, row, torch.zeros_like(row), torch.zeros(1, dtype=torch.uint8, device=dev))
    hp = HotPath(n, device=dev)
    q, B = _pad_queries(x, hp.tile)
    return 2.0 * hp.evaluate(mix, q, cull=False)[:B, 0]


def eval_mixture(mix: Mixture, x, active=None, *, tile_size: int = 256, k: int = 16, multiplier: float = 3.0,
                 projection_seed: int = 0) -> torch.Tensor:
    """SPEC.md:83-91 at every query x [B, N]: pred [B, 3] float32. `active`: None = cull
    (make_projection_set(N, k, projection_seed), multiplier), "all" = every live component,
    or a CandidateLists from cull_tile for x's tiles."""
    x = _f32(x, mix.device)
    hp = HotPath(mix.n_dims, k=k, multiplier=multiplier, tile_size=tile_size, projection_seed=projection_seed,
                 device=mix.device)
    q, B = _pad_queries(x, hp.tile)
    if isinstance(active, CandidateLists):
        hp.reset_status()
        recs = hp.activate(mix)
        recs.tc_conditioning()
        pred, _, _ = hp.forward(q, recs, active)
        hp.check_status(mix)
        return pred[:B]
    return hp.evaluate(mix, q, cull=active is None)[:B]


def compose_child(parent, child, device=None):
    """(m_c = L m_u + m_p, L U) for raw parent / child rows, float64 ([N], [N, N]), via K1."""
    dev = _dev(device)
    p, c = _f32(parent, dev).reshape(1, -1), _f32(child, dev).reshape(1, -1)
    R = p.shape[1]
    n = next(m for m in range(1, 17) if raw_width(m) == R)
    mix = Mixture(n, BRIGHTNESS, p, c, torch.ones(1, dtype=torch.uint8, device=dev), True)
    hp = HotPath(n, device=dev)
    hp.reset_status()
    recs = hp.activate(mix)
    hp.check_status(mix)
    return recs.mean64[1], _unpack(recs.chol64[1], n)


def project_components(mix: Mixture, ps: ProjectionSet, multiplier: float = 3.0) -> ProjectedBounds:
    """m_r = m.r, sigma_r = ||L^T r|| (FP64) for every evaluated Gaussian, [k, Gev]."""
    hp = HotPath(mix.n_dims, multiplier=multiplier, projections=ps, device=mix.device)
    hp.reset_status()
    recs = hp.activate(mix)
    pb = hp.project(recs)
    hp.check_status(mix)
    return pb


def tile_bounds(queries, ps: ProjectionSet, tile_size: int = 256) -> TileBounds:
    """per tile of tile_size contiguous queries and per vector, [min, max] of q.r."""
    q = _f32(queries, _dev())
    hp = HotPath(q.shape[1], projections=ps, tile_size=tile_size, device=q.device)
    return hp.tile_bounds(q)


def cull_tile(tb: TileBounds, pb: ProjectedBounds, multiplier: float | None = None) -> CandidateLists:
    """SPEC.md:198-206 for every tile of tb: culled iff for some vector the interval distance
    max(lo - m_r, m_r - hi, 0) exceeds multiplier * sigma_r (FP64, equality kept). Returns the active
    sets as CSR (`.offsets`, ascending `.idx`); candidate_lists() gives one index tensor per tile."""
    thr = pb.thr
    if multiplier is not None and float(multiplier) != pb.multiplier:
        thr = torch.where(pb.thr < 0, pb.thr, pb.sigma_r * float(multiplier))
    n = 1                                      # the cull itself does not depend on N
    hp = HotPath(n, k=int(tb.lo.shape[1]), tile_size=tb.tile_size, device=tb.lo.device)
    return hp.cull(tb, ProjectedBounds(pb.m_r, pb.sigma_r, thr, multiplier or pb.multiplier))


def brute_force_active(queries, mix: Mixture, epsilon: float, tile_size: int = 256):
    """per tile, the evaluated Gaussians with eval_gaussian >= epsilon at some tile
    query (FP64 on the device). Returns one ascending index tensor per tile."""
    q = _f32(queries, mix.device)
    hp = HotPath(mix.n_dims, tile_size=tile_size, device=mix.device)
    recs = hp.activate(mix)
    mask, counts = hp.brute_force_active(q, recs, epsilon)
    return _mask_lists(mask, recs.Gev)


def _mask_lists(mask, Gev):
    bits = torch.arange(32, device=mask.device, dtype=torch.int64)
    words = mask.to(torch.int64) & 0xFFFFFFFF
    full = ((words.unsqueeze(-1) >> bits) & 1).reshape(mask.shape[0], -1)[:, :Gev]
    return [torch.nonzero(r).flatten().to(torch.int32) for r in full]


def candidate_lists(cl: CandidateLists):
    """One ascending int32 index tensor per tile from a CSR."""
    off = cl.offsets.cpu().tolist()
    return [cl.idx[off[t]:off[t + 1]] for t in range(cl.T)]


def loss_rel_l2(pred, target, eps: float = 0.01, return_grad: bool = False):
    """mean over the 3B entries of (pred - target)^2 / (sg(pred)^2 + eps) in float64
    (fixed-order reduction); with return_grad also d loss / d pred [B, 3] (denominator detached, :291)."""
    dev = pred.device if isinstance(pred, torch.Tensor) else _dev()
    p, t = _f32(pred, dev).reshape(-1, 3), _f32(target, dev).reshape(-1, 3)
    if p.shape != t.shape:
        raise ValueError("pred and target batches must be congruent")
    B = p.shape[0]
    part = torch.empty(max(1, (B + 255) // 256), dtype=torch.float64, device=dev)
    dp = torch.empty_like(p) if return_grad else None
    K.call("ndg_loss_rel_l2", B, _p(p), _p(t), float(eps), max(1, B), _p(dp), _p(part), _stream())
    out = torch.empty(1, dtype=torch.float64, device=dev)
    K.call("ndg_loss_finalize", int(part.shape[0]), _p(part), _p(out), _stream())
    loss = float(out.cpu()[0]) if B else 0.0
    return (loss, dp) if return_grad else loss


def _batch(batch, dev):
    if isinstance(batch, (tuple, list)):
        q, t = batch
    else:
        q, t = batch.queries, batch.targets
    return _f32(q, dev), _f32(t, dev)


def backward(mix: Mixture, batch, active=None, eps: float = 0.01, *, tile_size: int = 256, k: int = 16,
             multiplier: float = 3.0, projection_seed: int = 0):
    """(loss, GradientBuffer) of loss_rel_l2 w.r.t. every raw parameter of every active
    component and live child (child -> parent cross terms included). `batch` = (queries, targets) or an
    object with .queries / .targets; `active` as for eval_mixture. A non-finite
    gradient raises NonFiniteGradientError(component, block, batch_index)."""
    q, t = _batch(batch, mix.device)
    if q.shape[0] % tile_size:
        raise ValueError("batch size must be a multiple of tile_size (SPEC.md:441)")
    hp = HotPath(mix.n_dims, k=k, multiplier=multiplier, tile_size=tile_size, eps=eps,
                 projection_seed=projection_seed, device=mix.device)
    res = hp.fwd_bwd(mix, q, t, cull=active is None,
                     candidates=active if isinstance(active, CandidateLists) else None)
    return res.loss, res.grads


def finite_diff_grad(mix: Mixture, batch, coordinate, h: float = 1e-4, eps: float = 0.01, points: int = 2) -> float:
    """(loss(theta + h) - loss(theta - h)) / (2h) for one raw coordinate
    (which, component, entry) -- which = "parent" | "child" -- with the forward re-run in float64,
    culling disabled and the rel-L2 denominator held at the unperturbed prediction.
    Evaluated by ndg_fd_f64 (only the perturbed Gaussians' change is summed, so the O(1) loss terms
    cancel exactly); points=4 gives the O(h^4) central stencil."""
    which, comp, entry = coordinate
    q, t = _batch(batch, mix.device)
    n, G = mix.n_dims, mix.G
    par, chi = mix.params.double().contiguous(), mix.child.double().contiguous()
    B = q.shape[0]
    pred = torch.empty(B, 3, dtype=torch.float64, device=mix.device)
    loss = torch.empty(1, dtype=torch.float64, device=mix.device)
    s = _stream()
    K.call("ndg_loss_f64", n, G, mix.amp_mode, 1, _p(par), _p(chi), _p(mix.flags), B, _p(q), _p(t), None, _p(pred),
           _p(loss), s)
    inv_den = (1.0 / (pred * pred + eps)).contiguous()
    cd = torch.tensor([[int(comp) + (G if which == "child" else 0), int(entry)]], dtype=torch.int32,
                      device=mix.device)
    fd = torch.empty(1, dtype=torch.float64, device=mix.device)
    K.call("ndg_fd_f64", n, G, mix.amp_mode, _p(par), _p(chi), _p(mix.flags), B, _p(q), _p(t), _p(pred), _p(inv_den),
           1, _p(cd), float(h), int(points), _p(fd), s)
    return float(fd.cpu()[0])
