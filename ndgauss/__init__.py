"""`import ndgauss` shim: the reference package's name (/root/reference/pkg/pyproject.toml:6) mapped
onto the B200 implementation in paper_2405_20067_b200 (hot path only)."""
from paper_2405_20067_b200 import *  # noqa: F401,F403
from paper_2405_20067_b200 import __version__, backward, eval_mixture  # noqa: F401
from . import errors, kernels  # noqa: F401
