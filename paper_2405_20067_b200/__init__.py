"""ndgauss-b200: the culled N-D Gaussian-mixture hot path of arXiv 2405.20067 on B200 (sm_100a).

Drop-in for the hot path of the reference package ``ndgauss`` (/root/reference/SPEC.md modules
gmm-core, culling, grad and the trainer's step; /root/reference/pkg): the same module-level
operations, types and exceptions, with every stage executed by hand-written CUDA kernels in
``libndg.so`` (C ABI: include/ndg.h). There is no CPU backend.

    >>> import paper_2405_20067_b200 as ndg
    >>> mix = ndg.Mixture.from_arrays(10, ndg.BRIGHTNESS, params)
    >>> hp = ndg.HotPath(10, k=16, multiplier=3.0, tile_size=256)
    >>> res = hp.fwd_bwd(mix, queries, targets)        # culled forward + rel-L2 loss + backward
"""
from .errors import (ConfigError, DegenerateSliceError, FileFormatError, InvalidParameterError,  # noqa: F401
                     NdgError, NonFiniteGradientError, TrainingAborted)
from .gmm import BRIGHTNESS, OPACITY, Mixture, n_chol, raw_slices, raw_width, tri  # noqa: F401
from .engine import (CandidateLists, EvalRecords, GradientBuffer, HotPath, ProjectedBounds,  # noqa: F401
                     ProjectionSet, StepResult, TileBounds, adam_step, alloc_gradients, kept_pairs_flops,
                     make_projection_set, new_adam_state)

__version__ = "0.1.0"


def eval_mixture(mix: Mixture, queries, *, tile_size: int = 256, k: int = 16, multiplier: float = 3.0,
                 projection_seed: int = 0, cull: bool = True):
    """Batched, culled eval_mixture at every query; returns pred [B, 3] on device."""
    hp = HotPath(mix.n_dims, k=k, multiplier=multiplier, tile_size=tile_size, projection_seed=projection_seed,
                 device=mix.device)
    return hp.evaluate(mix, queries, cull=cull)


def backward(mix: Mixture, queries, targets, *, eps: float = 0.01, tile_size: int = 256, k: int = 16,
             multiplier: float = 3.0, projection_seed: int = 0, cull: bool = True):
    """(loss, GradientBuffer) of the relative-L2 loss w.r.t. every raw parameter."""
    hp = HotPath(mix.n_dims, k=k, multiplier=multiplier, tile_size=tile_size, eps=eps,
                 projection_seed=projection_seed, device=mix.device)
    res = hp.fwd_bwd(mix, queries, targets, cull=cull)
    return res.loss, res.grads
