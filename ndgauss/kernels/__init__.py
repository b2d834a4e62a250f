"""Reference slot `ndgauss.kernels` (pkg/setup.py:37, `_core`) -> the libndg.so ctypes binding."""
from paper_2405_20067_b200.kernels import LIB_PATH, SIGNATURES, call, layout, load  # noqa: F401
