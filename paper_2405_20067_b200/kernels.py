"""ctypes binding of libndg.so -- the slot the reference fills with ``ndgauss.kernels._core``
(/root/reference/pkg/setup.py:32-53).

Unlike the reference (which silently falls back to NumPy when the extension is missing,
pkg/setup.py:3-4, 14-29), there is exactly one backend: if libndg.so is absent or no CUDA device is
visible, every hot-path call raises. Every entry point is declared in include/ndg.h.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("NDG_LIB") or os.path.join(_HERE, "libndg.so")   # NDG_LIB: tuning builds only

_P = C.c_void_p
_I = C.c_int
_L = C.c_int64
_F = C.c_float
_D = C.c_double

# name -> argtypes, mirroring include/ndg.h one-to-one (tests/test_abi.py checks the export list)
SIGNATURES = {
    "ndg_abi_version": [],
    "ndg_last_error": [],
    "ndg_supported_dims": [_I],
    "ndg_raw_floats": [_I],
    "ndg_record_floats": [_I],
    "ndg_query_floats": [_I],
    "ndg_accum_doubles": [_I],
    "ndg_num_stats": [],
    "ndg_backward_chunk": [],
    "ndg_prologue": [_I, _L, _L, _I, _P, _P, _P, _P, _P, _P, _P, _P, _P],
    "ndg_project": [_I, _L, _P, _P, _P, _P, _I, _D, _P, _P, _P, _P],
    "ndg_tile_bounds": [_I, _L, _I, _P, _P, _I, _P, _P, _P],
    "ndg_cull_mask": [_L, _I, _L, _P, _P, _P, _P, _P, _P, _P],
    "ndg_cull_prefilter_workspace": [_L, _I],
    "ndg_cull_prefilter": [_L, _I, _L, _P, _P, _P, _P, _I, _P, _P, _P, _P],
    "ndg_scan_counts": [_L, _P, _P, _P, _P],
    "ndg_cull_compact": [_L, _L, _P, _P, _P, _P],
    "ndg_forward": [_I, _L, _I, _P, _P, _P, _I, _P, _P, _F, _L, _P, _P, _P, _P],
    "ndg_centre_records": [_I, _L, _P, _P, _P, _P],
    "ndg_loss_finalize": [_L, _P, _P, _P],
    "ndg_loss_rel_l2": [_L, _P, _P, _D, _L, _P, _P, _P],
    "ndg_work_items": [_L, _P, _P, _P],
    "ndg_bwd_bounds": [_I, _L, _P, _L, _P, _P, _P, _P],
    "ndg_backward": [_I, _L, _I, _P, _P, _I, _P, _P, _P, _L, _L, _P, _P, _P],
    "ndg_acc_dequant": [_I, _L, _L, _P, _P, _P],
    "ndg_backward_mma_supported": [_I],
    "ndg_backward_mma": [_I, _L, _I, _P, _P, _P, _P, _P, _L, _L, _P, _P, _P],
    "ndg_active_mask": [_I, _L, _I, _P, _P, _P, _P, _L, _D, _P, _P, _P],
    "ndg_nonfinite_query": [_I, _L, _I, _P, _P, _P, _L, _L, _L, _P, _P],
    "ndg_fd_f64": [_I, _I, _I, _P, _P, _P, _L, _P, _P, _P, _P, _I, _P, _D, _I, _P, _P],
    "ndg_backward_f64": [_I, _L, _L, _I, _P, _P, _P, _P, _P, _L, _P, _P, _P, _P, _P],
    "ndg_loss_f64": [_I, _I, _I, _I, _P, _P, _P, _L, _P, _P, _P, _P, _P, _P],
    "ndg_epilogue": [_I, _L, _L, _I, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P],
    "ndg_adam": [_I, _L, _P, _P, _P, _P, _P, _I, _F, _F, _F, _F, _F, _F, _F, _P],
    "ndg_adam_flags": [_I, _L, _P, _P, _P, _P, _P, _I, _I, _I, _F, _F, _F, _F, _F, _F, _F, _P],
    "ndg_tc_records": [_I, _L, _P, _P, _P, _P, _P, _P, _P],
    "ndg_forward_tc": [_I, _L, _I, _P, _P, _P, _P, _P, _F, _L, _P, _P, _P, _P],
    "ndg_sample_workspace": [_L],
    "ndg_sample_batch": [_I, _L, _I, _I, _I, C.c_uint64, C.c_uint64, _P, _P, _P],
    "ndg_shading_target": [_I, _L, _P, _P, _P, _P],
    "ndg_fp32_probe": [_P, _I, _I, _P],
    "ndg_fp32_probe_flops": [_I, _I],
    "ndg_tf32_probe": [_P, _I, _I, _P],
    "ndg_tf32_probe_flops": [_I, _I],
    "ndg_hmma_probe": [_P, _I, _I, _P],
    "ndg_hmma_probe_flops": [_I, _I],
}

ERRORS = {0: "NDG_OK", 1: "NDG_ERR_INVALID_PARAMETER", 2: "NDG_ERR_NONFINITE_GRADIENT",
          -1: "NDG_ERR_BAD_ARGUMENT", -2: "NDG_ERR_UNSUPPORTED_DIMS", -3: "NDG_ERR_CUDA"}

_lib = None


class KernelLibraryMissing(RuntimeError):
    pass


def load():
    """Load libndg.so (no CUDA call is made; safe on a CPU-only host)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise KernelLibraryMissing(
            f"{LIB_PATH} is not built -- run `python -c 'import __graft_entry__ as g; g.build()'` "
            "(there is no CPU fallback)")
    lib = C.CDLL(LIB_PATH)
    for name, argtypes in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.argtypes = argtypes
        fn.restype = {"ndg_last_error": C.c_char_p, "ndg_fp32_probe_flops": C.c_double,
                      "ndg_tf32_probe_flops": C.c_double, "ndg_hmma_probe_flops": C.c_double,
                      "ndg_cull_prefilter_workspace": C.c_int64,
                      "ndg_sample_workspace": C.c_int64}.get(name, C.c_int)
    _lib = lib
    return lib


class NdgLaunchError(RuntimeError):
    pass


# entry points that enqueue exactly one kernel of ours (bench.py reports the count as gpu_launches)
LAUNCHING = {"ndg_prologue", "ndg_project", "ndg_tile_bounds", "ndg_cull_mask", "ndg_cull_prefilter", "ndg_scan_counts",
             "ndg_cull_compact", "ndg_forward", "ndg_forward_tc", "ndg_tc_records", "ndg_loss_finalize", "ndg_loss_rel_l2", "ndg_backward", "ndg_backward_mma",
             "ndg_work_items", "ndg_bwd_bounds", "ndg_acc_dequant", "ndg_active_mask", "ndg_centre_records", "ndg_loss_f64", "ndg_backward_f64", "ndg_fd_f64", "ndg_nonfinite_query", "ndg_sample_batch", "ndg_shading_target", "ndg_epilogue", "ndg_adam", "ndg_adam_flags",
             "ndg_fp32_probe", "ndg_tf32_probe", "ndg_hmma_probe"}
# entry points that enqueue several kernels: ndg_cull_prefilter = init, stats, hist, plan, scatter, zero,
# pre-filtered cull and the dense cull (the plan makes one of the two paths exit at once)
MULTI_LAUNCH = {"ndg_cull_prefilter": 8, "ndg_sample_batch": 3}
launch_count = 0


def call(name: str, *args):
    """Invoke an entry point; a nonzero launch code raises with the library's error string."""
    global launch_count
    lib = load()
    rc = getattr(lib, name)(*args)
    if name in LAUNCHING:
        launch_count += MULTI_LAUNCH.get(name, 1)
    if rc != 0:
        msg = lib.ndg_last_error().decode(errors="replace")
        raise NdgLaunchError(f"{name} failed: {ERRORS.get(rc, rc)} {msg}")
    return rc


def layout(n: int) -> dict:
    lib = load()
    if not lib.ndg_supported_dims(n):
        raise ValueError(f"n_dims={n} not supported (1..16)")
    return dict(raw=lib.ndg_raw_floats(n), rec=lib.ndg_record_floats(n), qrec=lib.ndg_query_floats(n),
                acc=lib.ndg_accum_doubles(n), stats=lib.ndg_num_stats(), chunk=lib.ndg_backward_chunk())
