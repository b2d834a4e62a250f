"""ctypes front-end of oracle/ndg_oracle.c -- TEST INFRASTRUCTURE ONLY (checker + CPU baseline).

Mirrors oracle/ndg_oracle.py's step (same algorithm, float64, OpenMP). See the header of
oracle/ndg_oracle.c for the reference citations.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import time

import numpy as np

from . import ndg_oracle as O

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libndg_oracle.so")
_lib = None

_d = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
_f = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
_u8 = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")
_i64 = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
_i32 = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
_I, _L, _D = C.c_int, C.c_int64, C.c_double


def build(force: bool = False) -> str:
    """Compile the C oracle with the flags of the reference's intended _core (pkg/setup.py:41-42)
    plus -ffp-contract=off (sequential no-FMA culling arithmetic)."""
    src = os.path.join(_HERE, "ndg_oracle.c")
    if force or not os.path.exists(LIB_PATH) or os.path.getmtime(LIB_PATH) < os.path.getmtime(src):
        subprocess.check_call(["make", "-s", "-C", _HERE, "libndg_oracle.so"])
    return LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = C.CDLL(LIB_PATH)
        L.ndgo_max_threads.restype = _I
        L.ndgo_set_threads.argtypes = [_I]
        L.ndgo_eval_set.argtypes = [_I, _L, _L, _I, _d, _d, _u8, _u8, _d, _d, _d, _u8, _u8, _d, _d]
        L.ndgo_project.argtypes = [_I, _L, _d, _d, _u8, _u8, _d, _I, _D, _d, _d, _d]
        L.ndgo_tile_bounds.argtypes = [_I, _L, _I, _f, _d, _I, _d, _d]
        L.ndgo_cull_counts.argtypes = [_L, _I, _L, _d, _d, _d, _d, _i64]
        L.ndgo_cull_fill.argtypes = [_L, _I, _L, _d, _d, _d, _d, _i64, _i32]
        L.ndgo_forward.argtypes = [_I, _L, _I, _f, _d, _d, _d, _i64, _i32, _d]
        L.ndgo_loss.argtypes = [_L, _d, _f, _D, _L, _d, _d]
        L.ndgo_loss.restype = _D
        L.ndgo_backward.argtypes = [_I, _L, _I, _L, _f, _d, _d, _d, _d, _d, _i64, _i32, _d]
        L.ndgo_epilogue.argtypes = [_I, _L, _L, _I, _d, _d, _u8, _d, _d, _d, _d, _d, _d]
        _lib = L
    return _lib


def set_threads(n: int):
    lib().ndgo_set_threads(int(n))


def max_threads() -> int:
    return int(lib().ndgo_max_threads())


def eval_set(mix: O.OMixture, gev: int | None = None):
    L = lib()
    N, G = mix.n_dims, mix.G
    Gev = (2 * G if mix.any_child else G) if gev is None else gev
    mean = np.zeros((Gev, N))
    Lm = np.zeros((Gev, N, N))
    a = np.zeros((Gev, 3))
    live = np.zeros(Gev, np.uint8)
    degen = np.zeros(Gev, np.uint8)
    Lp = np.zeros((G, N, N))
    Uc = np.zeros((G, N, N))
    L.ndgo_eval_set(N, G, Gev, mix.amp_mode, np.ascontiguousarray(mix.params), np.ascontiguousarray(mix.child),
                    mix.has_child.astype(np.uint8), mix.frozen.astype(np.uint8), mean, Lm, a, live, degen, Lp, Uc)
    return dict(G=G, Gev=Gev, mean=mean, L=Lm, a=a, live=live, degen=degen, Lp=Lp, Uc=Uc)


def project(ev, R, mult):
    k, N = R.shape
    Gev = ev["Gev"]
    mr, sr, thr = (np.zeros((k, Gev)) for _ in range(3))
    lib().ndgo_project(N, Gev, ev["mean"], ev["L"], ev["live"], ev["degen"], np.ascontiguousarray(R), k,
                       float(mult), mr, sr, thr)
    return mr, sr, thr


def tile_bounds(q, R, tile):
    q = np.ascontiguousarray(q, np.float32)
    B, N = q.shape
    k = R.shape[0]
    T = B // tile
    lo, hi = np.zeros((T, k)), np.zeros((T, k))
    lib().ndgo_tile_bounds(N, B, tile, q, np.ascontiguousarray(R), k, lo, hi)
    return lo, hi


def cull_csr(lo, hi, mr, thr):
    T, k = lo.shape
    Gev = mr.shape[1]
    counts = np.zeros(T, np.int64)
    lib().ndgo_cull_counts(T, k, Gev, lo, hi, mr, thr, counts)
    offsets = np.zeros(T + 1, np.int64)
    offsets[1:] = np.cumsum(counts)
    idx = np.zeros(max(int(offsets[-1]), 1), np.int32)
    lib().ndgo_cull_fill(T, k, Gev, lo, hi, mr, thr, offsets, idx)
    return offsets, idx[:offsets[-1]]


def step(mix: O.OMixture, q, tgt, R, *, tile=256, mult=3.0, eps=0.01, cull=True, n_total=None, timings=None):
    """Full oracle step (same outputs as ndg_oracle.fwd_bwd)."""
    L = lib()
    q = np.ascontiguousarray(q, np.float32)
    tgt = np.ascontiguousarray(tgt, np.float32)
    B, N = q.shape
    T = B // tile
    t0 = time.perf_counter()
    ev = eval_set(mix)
    Gev = ev["Gev"]
    t1 = time.perf_counter()
    if cull:
        mr, sr, thr = project(ev, R, mult)
        t2 = time.perf_counter()
        lo, hi = tile_bounds(q, R, tile)
        offsets, idx = cull_csr(lo, hi, mr, thr)
    else:
        t2 = time.perf_counter()
        live = np.flatnonzero(ev["live"]).astype(np.int32)
        offsets = np.arange(T + 1, dtype=np.int64) * live.size
        idx = np.tile(live, T)
    idx = np.ascontiguousarray(idx, np.int32)
    t3 = time.perf_counter()
    pred = np.zeros((B, 3))
    L.ndgo_forward(N, B, tile, q, ev["mean"], ev["L"], ev["a"], offsets, idx if idx.size else np.zeros(1, np.int32),
                   pred)
    dpred = np.zeros((B, 3))
    ell = np.zeros(B)
    loss = L.ndgo_loss(B, pred, tgt, float(eps), int(n_total or B), dpred, ell)
    t4 = time.perf_counter()
    A = O.n_chol(N) + N + 6
    accum = np.zeros((Gev, A))
    L.ndgo_backward(N, B, tile, Gev, q, dpred, ell, ev["mean"], ev["L"], ev["a"], offsets,
                    idx if idx.size else np.zeros(1, np.int32), accum)
    t5 = time.perf_counter()
    R_ = O.raw_width(N)
    gp = np.zeros((mix.G, R_))
    gc = np.zeros((mix.G, R_))
    L.ndgo_epilogue(N, mix.G, Gev, mix.amp_mode, np.ascontiguousarray(mix.params), np.ascontiguousarray(mix.child),
                    ev["live"], ev["L"], ev["Lp"], ev["Uc"], accum, gp, gc)
    t6 = time.perf_counter()
    if timings is not None:
        timings.update(eval_set=t1 - t0, project=t2 - t1, bounds_cull=t3 - t2, forward_loss=t4 - t3,
                       backward=t5 - t4, epilogue=t6 - t5)
    P = O.n_chol(N)
    return dict(offsets=offsets, idx=idx, pred=pred, loss=loss, dpred=dpred, ell=ell, grad_parent=gp,
                grad_child=gc, stats=accum[:, P + N + 3:P + N + 6], accum=accum, ev=ev)
