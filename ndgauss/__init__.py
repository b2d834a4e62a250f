"""`import ndgauss` shim: the reference package's name (/root/reference/pkg/pyproject.toml:6) mapped
onto the B200 implementation in paper_2405_20067_b200 (hot path only). The
module-level operations keep their SPEC names: activate_cholesky, eval_gaussian,
eval_mixture, compose_child, make_projection_set, project_components, tile_bounds, cull_tile,
brute_force_active, loss_rel_l2, backward, finite_diff_grad, adam_step."""
from paper_2405_20067_b200 import *  # noqa: F401,F403
from paper_2405_20067_b200 import __version__  # noqa: F401
from paper_2405_20067_b200.api import (activate_cholesky, adam_step, backward, brute_force_active,  # noqa: F401
                                       candidate_lists, compose_child, cull_tile, eval_gaussian, eval_mixture,
                                       finite_diff_grad, loss_rel_l2, make_projection_set, project_components,
                                       tile_bounds)
from . import errors, kernels  # noqa: F401
