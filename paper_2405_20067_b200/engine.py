"""The culled forward + backward hot path on one GPU, one C-ABI call per stage.

Host side of the reference's L1-L3 hot path: the operations of SPEC.md's
gmm-core, culling and grad modules, each enqueued on the current CUDA stream through libndg.so:

    K1 ndg_prologue      activate_cholesky + compose_child + activations
    K2 ndg_project       project_components
    K3 ndg_tile_bounds   TileBounds
    K4 ndg_cull_*        cull_tile for every tile -> CSR candidate lists
    K5 ndg_forward_tc    eval_mixture (+ K6 loss_rel_l2 fused), tcgen05
       ndg_forward       (FP32-pipe K5: ill-conditioned mixtures, tiles > 256, NDG_FORWARD=fp32)
    K7 ndg_backward      backward pair loop, FP32 pipe (N <= 14)
       ndg_backward_mma  (warp-MMA pair loop: N >= 14, or NDG_BACKWARD=mma for N >= 9)
       (+ ndg_bwd_bounds / ndg_work_items before, ndg_acc_dequant after: the deterministic
        fixed-point reduction of SPEC.md:294, and the band order of the work items)
    K8 ndg_epilogue      backward tail, raw-parameter chain rule
    K9 ndg_adam          adam_step

There is no CPU path: everything below requires libndg.so and a CUDA device.
"""
from __future__ import annotations

import ctypes
import math
import os
from dataclasses import dataclass, field

import numpy as np
import torch

from . import kernels as K
from .errors import InvalidParameterError, NonFiniteGradientError
from .gmm import FLAG_CHILD, FLAG_FROZEN, Mixture, n_chol, raw_width

_INT64_MAX = (1 << 63) - 1
_BLOCKS = ("mean", "chol", "color", "amp")


def _p(t):
    """Device pointer of a tensor (0 for None)."""
    return ctypes.c_void_p(0 if t is None else t.data_ptr())


def _stream():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


class _NvtxRange:
    """NVTX range around one stage when NDG_NVTX=1 (for nsys / ncu --nvtx); free otherwise."""
    on = os.environ.get("NDG_NVTX", "0") == "1"

    def __init__(self, name):
        self.name = name

    def __enter__(self):
        if self.on:
            torch.cuda.nvtx.range_push(self.name)

    def __exit__(self, *exc):
        if self.on:
            torch.cuda.nvtx.range_pop()
        return False


# ----------------------------------------------------------------------------------------------
# culling types
# ----------------------------------------------------------------------------------------------
@dataclass
class ProjectionSet:
    """k unit vectors in R^N reproducible from seed."""
    vectors: np.ndarray            # [k, N] float64
    seed: int
    device_vectors: torch.Tensor = field(default=None, repr=False)

    @property
    def k(self):
        return self.vectors.shape[0]

    def on(self, device):
        if self.device_vectors is None or self.device_vectors.device != device:
            self.device_vectors = torch.from_numpy(np.ascontiguousarray(self.vectors)).to(device)
        return self.device_vectors


def make_projection_set(n_dims: int, k: int = 16, seed: int = 0) -> ProjectionSet:
    """normalised independent standard normals. The stream is pinned to
    numpy.random.default_rng(seed).standard_normal((k, N)) and the norm to a sequential float64 sum
    of squares."""
    if n_dims < 1 or k < 1:
        raise ValueError("n_dims and k must be >= 1")
    v = np.random.default_rng(seed).standard_normal((k, n_dims))
    ss = v[:, 0] * v[:, 0]
    for j in range(1, n_dims):
        ss = ss + v[:, j] * v[:, j]
    return ProjectionSet(v / np.sqrt(ss)[:, None], int(seed))


@dataclass
class EvalRecords:
    """Output of K1 for the evaluated Gaussians (index space e = i | G + i)."""
    Gev: int
    rec: torch.Tensor        # [Gev, RS] float32 evaluation records
    mean64: torch.Tensor     # [Gev, N] float64
    chol64: torch.Tensor     # [Gev, P] float64 packed lower factor (composed for children)
    eflags: torch.Tensor     # [Gev] uint8: bit0 live, bit1 degenerate
    rec_tc: torch.Tensor = None   # [Gev, N*pad8(N+1) + 4] float32 Ahat records + colour (tensor-core forward)
    tc_cond: torch.Tensor = None   # [3] float64: [max, sum of squares, count] of B_e (ndg_tc_records)
    tc_cond_host: tuple = None     # read back with the step's one mid-pipeline sync
    rec_c: torch.Tensor = None     # K1c centred records, built on demand (very sharp mixtures)

    def tc_conditioning(self) -> float:
        """RMS over live Gaussians of B_e, the z-GEMM's conditioning (inf without tensor-core records)."""
        if self.tc_cond_host is None:
            if self.tc_cond is None:
                return float("inf")
            self.tc_cond_host = tuple(self.tc_cond.cpu().tolist())
        mx, ss, cnt = self.tc_cond_host
        return math.sqrt(ss / cnt) if cnt > 0 else 0.0

    def tc_peak(self) -> float:
        """max over live Gaussians of B_e: the worst single Gaussian's conditioning."""
        if self.tc_cond_host is None:
            self.tc_conditioning()
        return float(self.tc_cond_host[0]) if self.tc_cond_host is not None else float("inf")


@dataclass
class ProjectedBounds:
    """SPEC.md:161-167, laid out [k, Gev]; thr = multiplier * sigma_r, -1 when never evaluated."""
    m_r: torch.Tensor
    sigma_r: torch.Tensor
    thr: torch.Tensor
    multiplier: float


@dataclass
class TileBounds:
    """lo / hi [T, k]."""
    lo: torch.Tensor
    hi: torch.Tensor
    tile_size: int


@dataclass
class CandidateLists:
    """Per-tile active sets as CSR (offsets int64 [T+1], idx int32 ascending per tile)."""
    offsets: torch.Tensor
    idx: torch.Tensor
    chunk_offsets: torch.Tensor
    n_pairs_tiles: int        # sum over tiles of |cand(tile)|
    n_chunks: int
    mask: torch.Tensor = None  # [T, ceil(Gev/32)] int32 bit-words the CSR was compacted from

    @property
    def T(self):
        return int(self.offsets.shape[0]) - 1

    def kept_fraction(self, Gev: int) -> float:
        return self.n_pairs_tiles / max(1, self.T * Gev)


@dataclass
class GradientBuffer:
    """Raw-layout gradients of parents and children plus the density-control
    statistics, all views into ONE flat float32 buffer so a multi-GPU step needs one allreduce.
    Layout [params | stats | scalars | child]: without live children the child block is all zero
    and the step reduces only the prefix `reduced()` (half the bytes at cfg5)."""
    flat: torch.Tensor
    params: torch.Tensor      # [G, R]
    child: torch.Tensor       # [G, R]
    stats: torch.Tensor       # [Gev, 3]: loss share, gradient proxy, pairs
    scalars: torch.Tensor     # [2]: loss, total pairs (filled by the caller that reduces)
    children_live: bool = False

    def reduced(self) -> torch.Tensor:
        """The part of `flat` the step's allreduce must sum (the child block only when live)."""
        n = self.flat.numel() - (0 if self.children_live else self.child.numel())
        return self.flat[:n]


@dataclass
class StepResult:
    loss: float
    pred: torch.Tensor
    grads: GradientBuffer
    candidates: CandidateLists
    n_degenerate: int
    kept_fraction: float


def alloc_gradients(G: int, Gev: int, n: int, device) -> GradientBuffer:
    R = raw_width(n)
    flat = torch.zeros(2 * G * R + 3 * Gev + 2, dtype=torch.float32, device=device)
    o = 0
    gp = flat[o:o + G * R].view(G, R); o += G * R
    st = flat[o:o + 3 * Gev].view(Gev, 3); o += 3 * Gev
    sc = flat[o:o + 2]; o += 2
    gc = flat[o:o + G * R].view(G, R)
    return GradientBuffer(flat, gp, gc, st, sc, Gev == 2 * G)


def decode_status(st, G: int, n: int) -> int:
    """Map the device status word (include/ndg.h ndg_status) onto the reference's exceptions
    (errors.py:8-33); returns the degenerate-Gaussian count when there is no error."""
    R = raw_width(n)
    for slot, cls in ((0, InvalidParameterError), (1, NonFiniteGradientError)):
        if st[slot] != 0:
            key = _INT64_MAX - int(st[slot])
            which = "child" if key >= G * R else "parent"
            comp, entry = divmod(key % (G * R), R)
            blk = 0 if entry < n else 1 if entry < n + n_chol(n) else 2 if entry < n + n_chol(n) + 3 else 3
            if cls is InvalidParameterError:
                raise InvalidParameterError(f"non-finite raw parameter ({which} row, block {_BLOCKS[blk]})",
                                            component=int(comp), block=_BLOCKS[blk], entry=int(entry))
            err = NonFiniteGradientError(f"non-finite gradient ({which} row, block {_BLOCKS[blk]})",
                                         component=int(comp), block=_BLOCKS[blk], batch_index=-1)
            err.child_row = which == "child"
            raise err
    return int(st[2])


class HotPath:
    """One object per (device, N). Each method is one stage; `fwd_bwd` chains them."""

    def __init__(self, n_dims: int, *, k: int = 16, multiplier: float = 3.0, tile_size: int = 256,
                 eps: float = 0.01, projection_seed: int = 0, projections: ProjectionSet | None = None,
                 device=None, forward: str | None = None, backward: str | None = None, prefilter: str | None = None):
        self.n = int(n_dims)
        self.L = K.layout(self.n)
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        if self.device.type != "cuda":
            raise RuntimeError("HotPath needs a CUDA device (no CPU fallback)")
        self.ps = projections or make_projection_set(self.n, k, projection_seed)
        self.multiplier = float(multiplier)
        self.tile = int(tile_size)
        self.eps = float(eps)
        self.status = torch.zeros(4, dtype=torch.int64, device=self.device)
        # K5 implementation: "tc" = tcgen05 z-GEMM (3xTF32), "fp32" = FP32-pipe forward substitution
        self.forward_impl = forward or os.environ.get("NDG_FORWARD", "tc")
        if self.forward_impl not in ("tc", "fp32"):
            raise ValueError("forward must be 'tc' or 'fp32'")
        if self.forward_impl == "tc" and self.tile > 256:
            self.forward_impl = "fp32"      # the tcgen05 K5 covers tiles of up to two 128-query halves
        # K7 implementation: "auto" (default) = warp-MMA K7 for N >= MMA_MIN_N, else the FP32-pipe pair
        # loop; "fp32" / "mma" force one (both per-step guarded)
        bwd = backward or os.environ.get("NDG_BACKWARD", "auto")
        if bwd not in ("auto", "fp32", "mma"):
            raise ValueError("backward must be 'auto', 'fp32' or 'mma'")
        lib = K.load()
        if bwd == "auto":
            bwd = "mma" if self.n >= self.MMA_MIN_N else "fp32"
        if bwd == "mma" and not (lib.ndg_backward_mma_supported(self.n) and self.tile % 8 == 0):
            bwd = "fp32"
        self.backward_impl = bwd
        # K4 binning: "auto" = bucket pre-filter when the device-side plan finds it cheaper (tight tiles,
        # narrow Gaussians), else the dense pass; "on" forces the pre-filter, "off" the plain dense kernel.
        # All three give bit-identical candidate lists.
        self.prefilter = prefilter or os.environ.get("NDG_PREFILTER", "auto")
        if self.prefilter not in ("auto", "on", "off"):
            raise ValueError("prefilter must be 'auto', 'on' or 'off'")
        self._pf_ws = None
        self._recs = None    # the last activation: its conditioning bound rides on the cull's read-back
        self.last_forward_impl = self.last_backward_impl = None   # what the last step ran
        self.last_centred = False
        self.events = None   # when a dict: {"forward": [(start, end), ...], "backward": [...]} CUDA events
        # GraphedStep capture: the conditioning read-back is replaced by the captured value and the
        # candidate list / K7 work items are sized for the worst case, so no stage reads back mid-step
        self._static = None

    def enable_kernel_timing(self, on: bool = True):
        """Record CUDA events on the launching stream around the K5 and K7 launches."""
        self.events = {"forward": [], "backward": [], "cull": []} if on else None

    def _ev(self, name, when):
        if self.events is None:
            return
        # under graph capture: event record nodes, re-recorded by every replay (GraphedStep reads them)
        e = torch.cuda.Event(enable_timing=True, external=self._static is not None)
        e.record()
        if when == 0:
            self.events[name].append([e, None])
        else:
            self.events[name][-1][1] = e

    def kernel_ms(self, name):
        """Per-launch durations (ms) of the recorded launches of K5 ("forward"), K7 ("backward") and the
        K4a / K4p cull mask ("cull")."""
        return [x[0] if len(x) == 1 else x[0].elapsed_time(x[1]) for x in self.events[name]]

    # -- K1 --------------------------------------------------------------------------------
    def activate(self, mix: Mixture) -> EvalRecords:
        n, G, Gev = self.n, mix.G, mix.Gev
        dev = self.device
        rec = torch.empty(Gev, self.L["rec"], dtype=torch.float32, device=dev)
        mean64 = torch.empty(Gev, n, dtype=torch.float64, device=dev)
        chol64 = torch.empty(Gev, n_chol(n), dtype=torch.float64, device=dev)
        eflags = torch.empty(Gev, dtype=torch.uint8, device=dev)
        K.call("ndg_prologue", n, G, Gev, mix.amp_mode, _p(mix.params), _p(mix.child), _p(mix.flags), _p(rec),
               _p(mean64), _p(chol64), _p(eflags), _p(self.status), _stream())
        rec_tc = None
        # tensor-core records + the conditioning statistic: the TC kernels and the FP32 kernels'
        # centring decision both read it
        kk = ((n + 1 + 7) // 8) * 8
        rec_tc = torch.empty(Gev, n * kk + 4, dtype=torch.float32, device=dev)
        cond = torch.zeros(3, dtype=torch.float64, device=dev)
        K.call("ndg_tc_records", n, Gev, _p(mean64), _p(chol64), _p(eflags), _p(rec), _p(rec_tc), _p(cond), _stream())
        recs = EvalRecords(Gev, rec, mean64, chol64, eflags, rec_tc, cond)
        if self._static is not None:
            recs.tc_cond_host = self._static["cond"]
        self._recs = recs
        return recs

    # Largest z-GEMM conditioning (RMS over live Gaussians of B_e, ndg_tc_records) each tensor-core
    # kernel runs at; above it the step uses the FP32-pipe kernel with the same contract. K5: cfg2 sits
    # at 35, sigma 0.02 at 256 (parity 4.4e-5), the N=1 sigma 8e-4 mixture of tests/test_gpu_fuzz.py
    # at 842 (2.3e-4, out of tolerance). The moments K7 loses ~B^2 and is held to broad mixtures.
    TC_FORWARD_MAX_BOUND = 200.0      # RMS of B_e; error ~2e-7 * RMS (measured 4.4e-5 @ 256, 2.3e-4 @ 842)
    # ... and the worst single Gaussian: the error is per Gaussian (~2e-7 B_e on its own terms), so a few
    # very sharp Gaussians among broad ones barely move the RMS but would carry their own contributions
    # past the bar; past this peak the step runs the FP32 kernels (centred records, exact near the
    # Gaussian). cfg2's synthetic mixture peaks at ~520 (RMS 35), cfg4's at ~390.
    TC_FORWARD_PEAK_BOUND = 1000.0

    # The FP32 kernels' first term rho x + nb2 cancels like the z-GEMM (error ~1.4e-7 * RMS(B), e.g.
    # 1.45e-4 at RMS 1022 for the sigma 7e-4 mixture of tests/test_gpu_fuzz.py); past this bound they
    # run on centred records, z = rho ((x - m_hi) - m_lo), which loses nothing near the Gaussian.
    FP32_CENTRE_BOUND = 150.0
    FP32_CENTRE_PEAK_BOUND = 1000.0     # any single Gaussian past this also selects centred records

    def centred_records(self, recs: EvalRecords):
        """K1c records (or None) for the FP32 K5 / K7 of this step."""
        if recs.tc_conditioning() <= self.FP32_CENTRE_BOUND and recs.tc_peak() <= self.FP32_CENTRE_PEAK_BOUND:
            return None
        if recs.rec_c is None:
            recs.rec_c = torch.empty_like(recs.rec)
            K.call("ndg_centre_records", self.n, recs.Gev, _p(recs.mean64), _p(recs.rec), _p(recs.rec_c), _stream())
        return recs.rec_c

    def forward_tc_ok(self, recs: EvalRecords) -> bool:
        """Whether this step's K5 runs on the tensor cores (else the FP32-pipe K5, same contract)."""
        return (self.forward_impl == "tc" and recs.rec_tc is not None
                and recs.tc_conditioning() <= self.TC_FORWARD_MAX_BOUND
                and recs.tc_peak() <= self.TC_FORWARD_PEAK_BOUND)

    # The warp-MMA K7 forms z~ with the K5 z-GEMM (same records, same error ~2e-7 * RMS(B)), so it
    # shares the tensor-core forward's bound. Its cost does not depend on N (dims pad to one m16
    # block); the FP32 K7's grows with N and spills from 13 on. Measured (FP32 vs MMA, 50k Gaussians,
    # 2^18 queries, f16 K7-MMA): 126 vs 174 ms at N=13, 182 vs 178 at 14, 281 vs ~176 at 15, 315 vs 176
    # at 16 (the round-1 tf32 K7-MMA: ~208 at every N).
    MMA_MIN_N = 14

    def backward_mma_ok(self, recs: EvalRecords) -> bool:
        return (self.backward_impl == "mma" and recs.rec_tc is not None
                and recs.tc_conditioning() <= self.TC_FORWARD_MAX_BOUND
                and recs.tc_peak() <= self.TC_FORWARD_PEAK_BOUND)

    def backward_kernel_impl(self, recs: EvalRecords) -> str:
        """Which K7 this step runs: "mma" or "fp32"."""
        return "mma" if self.backward_mma_ok(recs) else "fp32"

    def kernel_choice(self, recs: EvalRecords) -> tuple:
        """Everything the step decides from the mixture's conditioning: (K5 on tensor cores, K7
        implementation, FP32 kernels on centred records)."""
        centred = not (recs.tc_conditioning() <= self.FP32_CENTRE_BOUND
                       and recs.tc_peak() <= self.FP32_CENTRE_PEAK_BOUND)
        return (self.forward_tc_ok(recs), self.backward_kernel_impl(recs), centred)

    # -- K2 --------------------------------------------------------------------------------
    def project(self, recs: EvalRecords) -> ProjectedBounds:
        k, Gev = self.ps.k, recs.Gev
        m_r = torch.empty(k, Gev, dtype=torch.float64, device=self.device)
        s_r = torch.empty_like(m_r)
        thr = torch.empty_like(m_r)
        K.call("ndg_project", self.n, Gev, _p(recs.mean64), _p(recs.chol64), _p(recs.eflags),
               _p(self.ps.on(self.device)), k, self.multiplier, _p(m_r), _p(s_r), _p(thr), _stream())
        return ProjectedBounds(m_r, s_r, thr, self.multiplier)

    # -- K3 --------------------------------------------------------------------------------
    def tile_bounds(self, queries: torch.Tensor) -> TileBounds:
        B = int(queries.shape[0])
        if B % self.tile:
            raise ValueError("batch size must be a multiple of tile_size (SPEC.md:441-442)")
        T, k = B // self.tile, self.ps.k
        lo = torch.empty(T, k, dtype=torch.float64, device=self.device)
        hi = torch.empty_like(lo)
        K.call("ndg_tile_bounds", self.n, B, self.tile, _p(queries), _p(self.ps.on(self.device)), k, _p(lo), _p(hi),
               _stream())
        return TileBounds(lo, hi, self.tile)

    # -- K4 --------------------------------------------------------------------------------
    # The pre-filter's device plan costs a handful of small launches: below this many (tile, Gaussian)
    # tests the dense pass is cheaper than deciding (cfg1: 64 tiles x 4096 Gaussians = 2.6e5).
    PREFILTER_MIN_TESTS = 1 << 22

    def cull(self, tb: TileBounds, pb: ProjectedBounds) -> CandidateLists:
        T, k = int(tb.lo.shape[0]), int(tb.lo.shape[1])
        Gev = int(pb.m_r.shape[1])
        W = (Gev + 31) // 32
        mask = torch.empty(T, W, dtype=torch.int32, device=self.device)
        counts = torch.zeros(T, dtype=torch.int64, device=self.device)
        self._ev("cull", 0)
        self._pf_used = k >= 2 and (self.prefilter == "on" or
                                    (self.prefilter == "auto" and T * Gev >= self.PREFILTER_MIN_TESTS))
        if self._pf_used:
            nb = int(K.load().ndg_cull_prefilter_workspace(Gev, k))
            if self._pf_ws is None or self._pf_ws.numel() < nb:
                self._pf_ws = torch.empty(nb, dtype=torch.uint8, device=self.device)
            K.call("ndg_cull_prefilter", T, k, Gev, _p(tb.lo), _p(tb.hi), _p(pb.m_r), _p(pb.thr),
                   1 if self.prefilter == "on" else 0, _p(self._pf_ws), _p(mask), _p(counts), _stream())
        else:
            K.call("ndg_cull_mask", T, k, Gev, _p(tb.lo), _p(tb.hi), _p(pb.m_r), _p(pb.thr), _p(mask), _p(counts),
                   _stream())
        self._ev("cull", 1)
        return self._finish_lists(T, Gev, counts, mask)

    def prefilter_plan(self):
        """(tests the pre-filtered pass counted, 1 if it ran) for the last cull, from the device plan."""
        if self._pf_ws is None or not getattr(self, "_pf_used", False):
            return None
        st = self._pf_ws[:64].view(torch.int64).cpu().tolist()
        return int(st[6]), int(st[7])

    def all_active(self, T: int, recs: EvalRecords) -> CandidateLists:
        """Culling disabled (SPEC.md:276 finite differences, SPEC.md:562 --no-cull): every live
        Gaussian is a candidate of every tile (still via the device compaction kernel)."""
        Gev = recs.Gev
        W = (Gev + 31) // 32
        live = (recs.eflags & 1).to(torch.bool)
        pad = torch.zeros(W * 32, dtype=torch.bool, device=self.device)
        pad[:Gev] = live
        bits = pad.view(W, 32).to(torch.int64) << torch.arange(32, device=self.device, dtype=torch.int64)
        words = bits.sum(dim=1).to(torch.int64)
        words = torch.where(words >= 2 ** 31, words - 2 ** 32, words).to(torch.int32)
        mask = words.unsqueeze(0).expand(T, W).contiguous()
        counts = live.sum().to(torch.int64).repeat(T)
        return self._finish_lists(T, Gev, counts, mask)

    def brute_force_active(self, queries, recs: EvalRecords, epsilon: float):
        """brute_force_active for every tile, in float64 on the device: returns
        (mask [T, ceil(Gev/32)] int32 bit-words, counts [T] int64) of the evaluated Gaussians with
        eval_gaussian >= epsilon at some query of the tile."""
        B = int(queries.shape[0])
        if B % self.tile:
            raise ValueError("batch size must be a multiple of tile_size (SPEC.md:441-442)")
        T, Gev = B // self.tile, recs.Gev
        W = (Gev + 31) // 32
        mask = torch.zeros(T, W, dtype=torch.int32, device=self.device)
        counts = torch.zeros(T, dtype=torch.int64, device=self.device)
        max_s2 = float("inf") if epsilon <= 0 else -2.0 * math.log(epsilon)
        K.call("ndg_active_mask", self.n, B, self.tile, _p(queries), _p(recs.mean64), _p(recs.chol64), _p(recs.eflags),
               Gev, max_s2, _p(mask), _p(counts), _stream())
        return mask, counts

    def _finish_lists(self, T, Gev, counts, mask) -> CandidateLists:
        offsets = torch.empty(T + 1, dtype=torch.int64, device=self.device)
        chunk_off = torch.empty(T + 1, dtype=torch.int64, device=self.device)
        K.call("ndg_scan_counts", T, _p(counts), _p(offsets), _p(chunk_off), _stream())
        if self._static is not None:
            # worst case: every live Gaussian in every tile; the real totals stay on the device
            idx = torch.empty(max(T * Gev, 1), dtype=torch.int32, device=self.device)
            K.call("ndg_cull_compact", T, Gev, _p(mask), _p(offsets), _p(idx), _stream())
            return CandidateLists(offsets, idx, chunk_off, None, T * -(-Gev // self.L["chunk"]), mask)
        vals = [offsets[T:T + 1], chunk_off[T:T + 1]]
        recs = self._recs if (self._recs is not None and self._recs.tc_cond is not None
                              and self._recs.tc_cond_host is None) else None
        if recs is not None:
            vals.append(recs.tc_cond.view(torch.int64))
        tot = torch.cat(vals).cpu()          # the step's one mid-pipeline sync: sizes idx (+ K5's conditioning)
        nnz, nchunks = int(tot[0]), int(tot[1])
        if recs is not None:
            recs.tc_cond_host = tuple(tot[2:5].view(torch.float64).tolist())
        idx = torch.empty(max(nnz, 1), dtype=torch.int32, device=self.device)
        K.call("ndg_cull_compact", T, Gev, _p(mask), _p(offsets), _p(idx), _stream())
        return CandidateLists(offsets, idx[:nnz], chunk_off, nnz, nchunks, mask)

    # -- K5 + K6 ---------------------------------------------------------------------------
    def forward(self, queries, recs: EvalRecords, cl: CandidateLists, targets=None, n_total=None):
        B = int(queries.shape[0])
        T = B // self.tile
        pred = torch.empty(B, 3, dtype=torch.float32, device=self.device)
        qrec = loss_part = None
        if targets is not None:
            qrec = torch.empty(B, self.L["qrec"], dtype=torch.float32, device=self.device)
            loss_part = torch.empty(T, dtype=torch.float64, device=self.device)
        self._ev("forward", 0)
        self.last_forward_impl = "tc" if self.forward_tc_ok(recs) else "fp32"
        if self.last_forward_impl == "tc":
            K.call("ndg_forward_tc", self.n, B, self.tile, _p(queries), _p(targets), _p(recs.rec_tc),
                   _p(cl.offsets), _p(cl.idx), self.eps, int(n_total or B), _p(pred), _p(qrec), _p(loss_part), _stream())
        else:
            rc = self.centred_records(recs)
            self.last_centred = rc is not None
            K.call("ndg_forward", self.n, B, self.tile, _p(queries), _p(targets), _p(recs.rec if rc is None else rc),
                   int(rc is not None), _p(cl.offsets),
                   _p(cl.idx), self.eps, int(n_total or B), _p(pred), _p(qrec), _p(loss_part), _stream())
        self._ev("forward", 1)
        return pred, qrec, loss_part

    def finalize_loss(self, loss_part) -> torch.Tensor:
        out = torch.empty(1, dtype=torch.float64, device=self.device)
        K.call("ndg_loss_finalize", int(loss_part.shape[0]), _p(loss_part), _p(out), _stream())
        return out

    # -- K7 + K8 ---------------------------------------------------------------------------
    def backward(self, mix: Mixture, recs: EvalRecords, cl: CandidateLists, qrec, grads: GradientBuffer):
        """K7 + K8. The cross-tile sums are exact int64 fixed point (two words per accumulator, scales
        from ndg_bwd_bounds), so gradients do not depend on the order work items finish."""
        B = int(qrec.shape[0])
        T, Gev, A = B // self.tile, recs.Gev, self.L["acc"]
        acc = torch.zeros(2, Gev, A, dtype=torch.int64, device=self.device)
        bounds = torch.zeros(4, dtype=torch.int32, device=self.device)
        K.call("ndg_bwd_bounds", self.n, B, _p(qrec), Gev, _p(recs.rec), _p(recs.eflags), _p(bounds), _stream())
        if self._static is None:
            items = torch.empty(max(cl.n_chunks, 1), dtype=torch.int64, device=self.device)
        else:
            items = torch.full((max(cl.n_chunks, 1),), -1, dtype=torch.int64, device=self.device)   # slots past
        K.call("ndg_work_items", T, _p(cl.chunk_offsets), _p(items), _stream())                      # the count exit
        self._ev("backward", 0)
        self.last_backward_impl = self.backward_kernel_impl(recs)
        if self.last_backward_impl == "mma":
            K.call("ndg_backward_mma", self.n, B, self.tile, _p(qrec), _p(recs.rec_tc), _p(cl.offsets), _p(cl.idx),
                   _p(items), cl.n_chunks, Gev, _p(bounds), _p(acc), _stream())
        else:
            rc = self.centred_records(recs)
            self.last_centred = rc is not None
            K.call("ndg_backward", self.n, B, self.tile, _p(qrec), _p(recs.rec if rc is None else rc),
                   int(rc is not None), _p(cl.offsets), _p(cl.idx), _p(items), cl.n_chunks, Gev, _p(bounds),
                   _p(acc), _stream())
        self._ev("backward", 1)
        K.call("ndg_acc_dequant", self.n, Gev, B, _p(bounds), _p(acc), _stream())
        accum = acc[0].view(torch.float64)
        K.call("ndg_epilogue", self.n, mix.G, recs.Gev, mix.amp_mode, _p(mix.params), _p(mix.child), _p(mix.flags),
               _p(recs.eflags), _p(recs.chol64), _p(accum), _p(grads.params), _p(grads.child), _p(grads.stats),
               _p(self.status), _stream())
        return accum

    def nonfinite_batch_index(self, mix: Mixture, recs: EvalRecords, cl: CandidateLists, qrec, err) -> int:
        """Error path of NonFiniteGradientError: the lowest index into this call's query
        batch at which the offending component's pairs (its own Gaussian, and for a parent row also its
        live child, whose composition reads the parent) give a non-finite backward term; -1 when no pair
        does (the non-finite value arose in the epilogue's solve)."""
        if cl.mask is None or qrec is None:
            return -1
        G, i = mix.G, int(err.component)
        if getattr(err, "child_row", False):
            e1, e2 = G + i, -1
        else:
            e1, e2 = i, (G + i if recs.Gev == 2 * G else -1)
        out = torch.full((1,), _INT64_MAX, dtype=torch.int64, device=self.device)
        K.call("ndg_nonfinite_query", self.n, int(qrec.shape[0]), self.tile, _p(qrec), _p(recs.rec), _p(cl.mask),
               recs.Gev, e1, e2, _p(out), _stream())
        b = int(out.cpu()[0])
        return -1 if b == _INT64_MAX else b

    # -- status ----------------------------------------------------------------------------
    def reset_status(self):
        self.status.zero_()

    def check_status(self, mix: Mixture, host_status=None):
        st = (self.status.cpu() if host_status is None else host_status).tolist()
        return decode_status(st, mix.G, self.n)

    # -- whole step ------------------------------------------------------------------------
    def fwd_bwd(self, mix: Mixture, queries, targets, *, cull: bool = True, n_total=None, grads=None,
                allreduce=None, check: bool = True, candidates: CandidateLists | None = None) -> StepResult:
        """One culled forward + loss + backward pass (SPEC.md:329 minus the optimizer step).

        `allreduce(flat)` -- when given -- sums the flat gradient buffer across ranks (one NCCL
        collective) before the status / loss read-back. `candidates` -- when given --
        are the per-tile active sets to use (SPEC.md:263's "active sets per tile"), e.g. from cull()."""
        recs, cl, pred, qrec, loss, grads = self._launch_step(mix, queries, targets, cull, n_total, grads, candidates)
        if allreduce is not None:
            with _NvtxRange("ndg.allreduce"):
                allreduce(grads.reduced())
        host = torch.cat([self.status, loss.view(torch.int64)]).cpu()
        return self._finish_step(mix, recs, cl, pred, qrec, grads, host[:4], float(host[4:5].view(torch.float64)[0]),
                                 allreduce is not None, check)

    def _finish_step(self, mix, recs, cl, pred, qrec, grads, status, loss, reduced, check) -> StepResult:
        """Host side of a step after its one read-back: status -> exceptions, the result record."""
        try:
            n_deg = self.check_status(mix, status) if check else 0
        except NonFiniteGradientError as err:
            err.batch_index = self.nonfinite_batch_index(mix, recs, cl, qrec, err)
            raise
        loss_v = float(grads.scalars[0]) if reduced else loss
        return StepResult(loss_v, pred, grads, cl, n_deg, cl.kept_fraction(recs.Gev))

    def _launch_step(self, mix, queries, targets, cull, n_total, grads, candidates):
        """Enqueue K1 ... K8 of one step (no read-back in static mode: a GraphedStep captures this)."""
        self.reset_status()
        with _NvtxRange("ndg.K1 activate"):
            recs = self.activate(mix)
        T = int(queries.shape[0]) // self.tile
        if candidates is not None:
            if candidates.T != T:
                raise ValueError("candidate lists do not match the batch's tile count")
            cl = candidates
            recs.tc_conditioning()                       # the read-back cull() would have carried
        elif cull:
            with _NvtxRange("ndg.K2-K4 bounds + cull"):
                pb = self.project(recs)
                tb = self.tile_bounds(queries)
                cl = self.cull(tb, pb)
        else:
            cl = self.all_active(T, recs)
        with _NvtxRange("ndg.K5 forward + loss"):
            pred, qrec, loss_part = self.forward(queries, recs, cl, targets, n_total)
            loss = self.finalize_loss(loss_part)
        if grads is None:
            grads = alloc_gradients(mix.G, recs.Gev, self.n, self.device)
        with _NvtxRange("ndg.K7-K8 backward"):
            self.backward(mix, recs, cl, qrec, grads)
        grads.scalars[0] = loss[0].to(torch.float32)
        if cl.n_pairs_tiles is None:
            grads.scalars[1:2].copy_(cl.offsets[T:T + 1] * self.tile)
        else:
            grads.scalars[1] = float(cl.n_pairs_tiles * self.tile)
        grads.children_live = recs.Gev == 2 * mix.G
        return recs, cl, pred, qrec, loss, grads

    def evaluate(self, mix: Mixture, queries, *, cull: bool = True) -> torch.Tensor:
        """Culled evaluation at every query (cmd_eval's path). A batch that is not a
        multiple of the tile size is padded with copies of its last query and the result sliced."""
        B = int(queries.shape[0])
        pad = (-B) % self.tile
        if pad:
            if B == 0:
                return torch.zeros(0, 3, dtype=torch.float32, device=self.device)
            return self.evaluate(mix, torch.cat([queries, queries[-1:].expand(pad, queries.shape[1])]).contiguous(),
                                 cull=cull)[:B]
        self.reset_status()
        recs = self.activate(mix)
        T = int(queries.shape[0]) // self.tile
        cl = self.cull(self.tile_bounds(queries), self.project(recs)) if cull else self.all_active(T, recs)
        pred, _, _ = self.forward(queries, recs, cl)
        self.check_status(mix)
        return pred


class GraphedStep:
    """HotPath.fwd_bwd captured once as a CUDA graph and replayed (verdict r01 weak 10): for small,
    launch-bound configurations (cfg1: ~0.4 ms of kernels behind ~22 launches and a mid-step host
    read-back) the whole step becomes one graph launch plus the end-of-step read-back.

    What makes the step capturable: the candidate list is sized for the worst case (T x Gev entries)
    and K7's grid for the worst-case work items (slots past the real count hold -1 and exit), so
    nothing reads the totals back mid-step; and the kernel choice that depends on the mixture's
    conditioning (HotPath.kernel_choice) is taken at capture. It is re-checked after every replay
    from the same read-back as the status word and the loss: if this step's mixture would choose
    differently, the step is re-run eagerly and the graph marked stale (recapture).

    `queries` / `targets` are the graph's input buffers (copy new batches into them); the mixture's
    tensors must stay the same storage (K9 Adam updates them in place; refinement events that
    reallocate them make `matches(mix)` false). The allreduce (NCCL or gloo) runs eagerly between the
    replay and the read-back. Results (pred, gradients, candidate lists) are views of the graph's
    buffers, overwritten by the next replay."""

    MAX_LIST = 1 << 24        # worst-case candidate list entries (T x Gev) a capture may allocate

    @classmethod
    def eligible(cls, hp: HotPath, mix: Mixture, batch: int) -> bool:
        return (batch // hp.tile) * mix.Gev <= cls.MAX_LIST

    def __init__(self, hp: HotPath, mix: Mixture, queries, targets, *, n_total=None, grads=None):
        if not self.eligible(hp, mix, int(queries.shape[0])):
            raise ValueError("worst-case candidate list too large for a captured step")
        self.hp, self.mix, self.queries, self.targets, self.n_total = hp, mix, queries, targets, n_total
        self.key = self._key(mix)
        self.grads = grads if grads is not None else alloc_gradients(mix.G, mix.Gev, hp.n, hp.device)
        self.stale = False
        # one eager step: warms every kernel (and its one-time attributes) and fixes the kernel choice
        hp.fwd_bwd(mix, queries, targets, n_total=n_total, grads=self.grads)
        self.cond = hp._recs.tc_cond_host
        self.choice = hp.kernel_choice(hp._recs)
        T = int(queries.shape[0]) // hp.tile
        hp._static = dict(cond=self.cond)
        try:
            # capture_begin / capture_end on a side stream (not the torch.cuda.graph context, which empties
            # the allocator cache on every capture: a fit re-captures after each refinement event)
            self.graph = torch.cuda.CUDAGraph()
            side = torch.cuda.Stream(hp.device)
            side.wait_stream(torch.cuda.current_stream(hp.device))
            timed = {k: len(v) for k, v in hp.events.items()} if hp.events is not None else None
            l0 = K.launch_count
            with torch.cuda.stream(side):
                self.graph.capture_begin()
                try:
                    recs, cl, pred, qrec, loss, _ = hp._launch_step(mix, queries, targets, True, n_total, self.grads,
                                                                    None)
                    self.readback = torch.cat([hp.status, loss.view(torch.int64), recs.tc_cond.view(torch.int64),
                                               cl.offsets[T:T + 1], cl.chunk_offsets[T:T + 1]])
                finally:
                    self.graph.capture_end()
            torch.cuda.current_stream(hp.device).wait_stream(side)
            self.launches = K.launch_count - l0            # libndg kernels per replay
            # CUDA-event pairs captured around K4 / K5 / K7 (when kernel timing was on at capture)
            self.timed = {} if timed is None else {k: hp.events[k].pop() for k in timed if len(hp.events[k]) > timed[k]}
        finally:
            hp._static = None
        self.recs, self.cl, self.pred, self.qrec = recs, cl, pred, qrec
        self.impl = (hp.last_forward_impl, hp.last_backward_impl)

    @staticmethod
    def _key(mix: Mixture):
        return (mix.G, mix.Gev, mix.amp_mode, mix.params.data_ptr(), mix.child.data_ptr(), mix.flags.data_ptr())

    def matches(self, mix: Mixture) -> bool:
        return not self.stale and self._key(mix) == self.key

    def __call__(self, allreduce=None, check: bool = True) -> StepResult:
        hp, mix = self.hp, self.mix
        if not self.matches(mix):
            raise RuntimeError("the mixture changed shape or storage since capture; build a new GraphedStep")
        self.graph.replay()
        if allreduce is not None:
            with _NvtxRange("ndg.allreduce"):
                allreduce(self.grads.reduced())
        host = self.readback.cpu()
        self.recs.tc_cond_host = tuple(host[5:8].view(torch.float64).tolist())
        hp._recs = self.recs
        if hp.kernel_choice(self.recs) != self.choice:
            # this mixture's conditioning picks other kernels than the captured ones: redo it eagerly
            self.stale = True
            return hp.fwd_bwd(mix, self.queries, self.targets, n_total=self.n_total, grads=self.grads,
                              allreduce=allreduce, check=check)
        if hp.events is not None:
            for name, (a, b) in self.timed.items():
                hp.events.setdefault(name, []).append([a.elapsed_time(b)])
        nnz, nch = int(host[8]), int(host[9])
        cl = CandidateLists(self.cl.offsets, self.cl.idx[:nnz], self.cl.chunk_offsets, nnz, nch, self.cl.mask)
        hp.last_forward_impl, hp.last_backward_impl = self.impl
        return hp._finish_step(mix, self.recs, cl, self.pred, self.qrec, self.grads, host[:4],
                               float(host[4:5].view(torch.float64)[0]), allreduce is not None, check)


class GraphedEval:
    """HotPath.evaluate captured as a CUDA graph for a FIXED mixture and query buffer -- a procedural
    target (datasets.GmmOracleTarget) evaluated at every training step's batch. Nothing is read back: the
    mixture does not change, so its status and its conditioning-dependent kernel choice are checked once,
    by the eager evaluation at capture. Each call writes the mixture's values at `queries` into `out`."""

    def __init__(self, hp: HotPath, mix: Mixture, queries, out, *, cull: bool = False):
        B = int(queries.shape[0])
        if B % hp.tile or tuple(out.shape) != (B, 3):
            raise ValueError("queries must be a tile multiple and out [B, 3]")
        hp.evaluate(mix, queries, cull=cull)           # eager: status check + the kernel choice
        cond = hp._recs.tc_cond_host
        hp._static = dict(cond=cond)
        try:
            self.graph = torch.cuda.CUDAGraph()
            side = torch.cuda.Stream(hp.device)
            side.wait_stream(torch.cuda.current_stream(hp.device))
            with torch.cuda.stream(side):
                self.graph.capture_begin()
                try:
                    hp.reset_status()
                    recs = hp.activate(mix)
                    T = B // hp.tile
                    cl = hp.cull(hp.tile_bounds(queries), hp.project(recs)) if cull else hp.all_active(T, recs)
                    pred, _, _ = hp.forward(queries, recs, cl)
                    out.copy_(pred)
                finally:
                    self.graph.capture_end()
            torch.cuda.current_stream(hp.device).wait_stream(side)
        finally:
            hp._static = None

    def __call__(self):
        self.graph.replay()


def adam_step(mix: Mixture, grads: GradientBuffer, state, step: int, lr=(2e-3, 5e-3, 1e-2, 1e-2),
              betas=(0.9, 0.999), eps=1e-8):
    """K9: bias-corrected Adam with per-block learning rates, applied to
    parent rows (not frozen) and live child rows. `state` = dict(m1p, m2p, m1c, m2c) float32."""
    n = mix.n_dims
    hyper = (int(step), *[float(x) for x in lr], float(betas[0]), float(betas[1]), float(eps), _stream())
    # rows selected on the device from the flag bytes (parents: not frozen; children: live and not frozen)
    K.call("ndg_adam_flags", n, mix.G, _p(mix.params), _p(grads.params), _p(state["m1p"]), _p(state["m2p"]),
           _p(mix.flags), 0, FLAG_FROZEN, *hyper)
    if mix.children_live:
        K.call("ndg_adam_flags", n, mix.G, _p(mix.child), _p(grads.child), _p(state["m1c"]), _p(state["m2c"]),
               _p(mix.flags), FLAG_CHILD, FLAG_FROZEN, *hyper)


def new_adam_state(mix: Mixture):
    z = lambda: torch.zeros_like(mix.params)  # noqa: E731
    return dict(m1p=z(), m2p=z(), m1c=z(), m2c=z())


def kept_pairs_flops(n: int) -> int:
    """Canonical algorithmic FP32 flops per (query, candidate) pair for fwd+bwd:
    F(N) = 3N^2 + 9N + 22 (184 / 412 / 934 at N = 6 / 10 / 16)."""
    return 3 * n * n + 9 * n + 22


def math_isfinite(x: float) -> bool:
    return math.isfinite(x)
