"""ndgauss-b200: the culled N-D Gaussian-mixture hot path of arXiv 2405.20067 on B200 (sm_100a).

Drop-in for the hot path of the reference package ``ndgauss`` (/root/reference/SPEC.md modules
gmm-core, culling, grad and the trainer's step; /root/reference/pkg): the same module-level
operations, types and exceptions, with every stage executed by hand-written CUDA kernels in
``libndg.so`` (C ABI: include/ndg.h). There is no CPU backend.

    >>> import paper_2405_20067_b200 as ndg
    >>> mix = ndg.Mixture.from_arrays(10, ndg.BRIGHTNESS, params)
    >>> hp = ndg.HotPath(10, k=16, multiplier=3.0, tile_size=256)
    >>> res = hp.fwd_bwd(mix, queries, targets)        # culled forward + rel-L2 loss + backward

The reference's module-level operations are exported under their SPEC names (api.py):
activate_cholesky, eval_gaussian, eval_mixture, compose_child, make_projection_set,
project_components, tile_bounds, cull_tile, brute_force_active, loss_rel_l2, backward,
finite_diff_grad, adam_step.
"""
from .errors import (ConfigError, DegenerateSliceError, FileFormatError, InvalidParameterError,  # noqa: F401
                     NdgError, NonFiniteGradientError, TrainingAborted)
from .gmm import BRIGHTNESS, OPACITY, Mixture, n_chol, raw_slices, raw_width, tri  # noqa: F401
from .engine import (CandidateLists, EvalRecords, GradientBuffer, GraphedEval, GraphedStep, HotPath, ProjectedBounds,  # noqa: F401
                     ProjectionSet, StepResult, TileBounds, adam_step, alloc_gradients, kept_pairs_flops,
                     make_projection_set, new_adam_state)

from .api import (activate_cholesky, backward, brute_force_active, candidate_lists, compose_child,  # noqa: F401
                  cull_tile, eval_gaussian, eval_mixture, finite_diff_grad, loss_rel_l2, project_components,
                  tile_bounds)

__version__ = "0.2.0"
