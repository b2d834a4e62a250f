"""Batch tiling and seeded synthetic inputs of the named shapes (reference module datasets,
/root/reference/SPEC.md:402-498; synthetic recipe SURVEY.md §8(d)).

Only what the hot path needs: the tile definition of sample_batch (queries sorted by the first
dimension, contiguous tiles of tile_size) and the synthetic mixture / query /
target generators the benchmark and the fit loop use. The generators are host-side NumPy (not on
the timed path); tests/test_cpu_infra.py checks they match the oracle's copies value for value.
"""
from __future__ import annotations

import math

import numpy as np

from .gmm import BRIGHTNESS, n_chol, raw_slices, raw_width, tri


def nn_sigma0(means, sample: int = 512, seed: int = 0) -> float:
    """Half the mean nearest-neighbour distance among the means, on a fixed subsample."""
    m = np.asarray(means, np.float64)
    G = m.shape[0]
    if G < 2:
        return 0.1
    rng = np.random.default_rng(seed)
    sel = rng.choice(G, size=min(G, sample), replace=False)
    d = []
    for i in sel:
        dd = np.sum((m - m[i]) ** 2, axis=1)
        dd[i] = np.inf
        d.append(math.sqrt(float(dd.min())))
    return 0.5 * float(np.mean(d))


def default_threshold(amp_mode: int) -> float:
    """Materialisation threshold t: 0.1 opacity / 0.01 brightness."""
    return 0.01 if amp_mode == BRIGHTNESS else 0.1


def amp_inverse(alpha, amp_mode: int):
    alpha = np.asarray(alpha, dtype=np.float64)
    return np.log(alpha) if amp_mode == BRIGHTNESS else np.log(alpha) - np.log1p(-alpha)


def synthetic_mixture(n: int, G: int, seed: int = 0, *, amp_mode: int = BRIGHTNESS, children: bool = False,
                      sigma0: float | None = None):
    """Seeded synthetic mixture; returns dict(params, child, has_child, frozen),
    float32 rows, and sigma0."""
    rng = np.random.default_rng(seed)
    ms, cs, cols, amp = raw_slices(n)
    R = raw_width(n)
    params = np.zeros((G, R))
    params[:, ms] = rng.random((G, n))
    s0 = nn_sigma0(params[:, ms]) if sigma0 is None else sigma0
    for i in range(n):
        for j in range(i + 1):
            if i == j:
                params[:, cs.start + tri(i, j)] = math.log(s0) + rng.uniform(-0.5, 0.5, G)
            else:
                params[:, cs.start + tri(i, j)] = rng.normal(0.0, s0, G)
    params[:, cols] = rng.normal(0.0, 1.0, (G, 3))
    params[:, amp] = rng.normal(math.log(0.1) if amp_mode == BRIGHTNESS else -2.0, 0.5, G)
    child = np.zeros((G, R))
    has_child = np.zeros(G, bool)
    if children:
        child[:, ms] = rng.normal(0.0, 0.3, (G, n))
        child[:, cs] = rng.normal(0.0, 0.1, (G, n_chol(n)))
        child[:, cols] = rng.normal(0.0, 1.0, (G, 3))
        child[:, amp] = amp_inverse(default_threshold(amp_mode) / 10.0, amp_mode) + rng.normal(0.0, 0.5, G)
        has_child[:] = True
    return dict(params=params.astype(np.float32), child=child.astype(np.float32), has_child=has_child,
                frozen=np.zeros(G, bool)), s0


def sort_into_tiles(q: np.ndarray, targets: np.ndarray | None = None):
    """Tile formation of sample_batch: stable sort by the first (position) dimension."""
    order = np.argsort(q[:, 0], kind="stable")
    return (q[order], None if targets is None else targets[order])


def synthetic_queries(n: int, B: int, seed: int = 1, *, regime: str = "R", tile_size: int = 256,
                      spread: float = 0.01) -> np.ndarray:
    """R: U[0,1)^N sorted by dim 0 (the reference sampler); C: coherent tiles (centre + N(0, spread^2));
    G: G-buffer-like queries on a 2-D manifold (gbuffer_queries)."""
    rng = np.random.default_rng(seed)
    if regime == "R":
        q = rng.random((B, n))
        q = q[np.argsort(q[:, 0], kind="stable")]
    elif regime == "C":
        T = B // tile_size
        centre = rng.random((T, 1, n))
        q = np.clip(centre + rng.normal(0.0, spread, (T, tile_size, n)), 0.0, 1.0).reshape(B, n)
    elif regime == "G":
        return gbuffer_queries(n, B, seed, tile_size)
    else:
        raise ValueError(f"unknown regime {regime!r}")
    return q.astype(np.float32)


def gbuffer_queries(n: int, B: int, seed: int = 1, tile_size: int = 256):
    """Regime G: G-buffer-like queries on a 2-D manifold in N-D. Pixels of a
    W x H image (W = 2^ceil(log2(B)/2)), grouped into square tiles of tile_size pixels (16 x 16 at 256):
    position (u, v, height(u, v)) | view direction to a fixed camera (mapped to [0,1]) | albedo(u, v) |
    roughness(u, v) | further smooth "variable" dims for N > 10; the first N features, float32. Tiles
    are tight in every dimension, so culling keeps only a few tens of Gaussians per tile and the
    binning (K4), not the pair loops, dominates the step."""
    rng = np.random.default_rng(seed)
    ph = rng.uniform(0.0, 1.0, 16)
    W = 1 << int(math.ceil(math.log2(max(B, 1)) / 2))
    H = B // W
    ts = int(round(math.sqrt(tile_size)))
    if ts * ts != tile_size or W % ts or H % ts or W * H != B:
        raise ValueError("regime G needs B = W * H with square tiles dividing the image")
    ty, tx, j, i = np.meshgrid(np.arange(H // ts), np.arange(W // ts), np.arange(ts), np.arange(ts), indexing="ij")
    px, py = (tx * ts + i).reshape(-1), (ty * ts + j).reshape(-1)
    u, v = (px + 0.5) / W, (py + 0.5) / H
    tau = 2.0 * np.pi
    h = 0.5 + 0.2 * np.sin(tau * (1.3 * u + ph[0])) * np.cos(tau * (0.9 * v + ph[1])) + 0.1 * np.sin(tau * (3.1 * u + 2.7 * v))
    cam = np.array([0.5, -0.8, 1.6])
    d = cam[None, :] - np.stack([u, v, h], 1)
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    feats = [u, v, h, 0.5 * (d[:, 0] + 1), 0.5 * (d[:, 1] + 1), 0.5 * (d[:, 2] + 1)]
    for c in range(3):
        feats.append(0.5 + 0.4 * np.sin(tau * (2.0 * u + ph[2 + c])) * np.cos(tau * (1.5 * v + ph[5 + c])))
    feats.append(0.5 + 0.45 * np.sin(tau * (u + v + ph[8])))
    k = 0
    while len(feats) < n:
        k += 1
        feats.append(0.5 + 0.4 * np.sin(tau * (k * u + (k + 1) * v + ph[9 + k % 7])))
    return np.stack(feats[:n], 1).astype(np.float32)


def gbuffer_mixture(n: int, G: int, seed: int = 0, *, sigma0: float = 0.005, amp_mode: int = BRIGHTNESS):
    """Mixture for regime G: means at the manifold features of G random pixels of a 1024 x 1024 image
    (gbuffer_queries' geometry), diagonal raw ln(sigma0) + U[-1/2, 1/2], off-diagonal raw N(0, sigma0^2),
    colour N(0, 1), amplitude as synthetic_mixture. Float32 rows."""
    rng = np.random.default_rng(seed)
    feats = gbuffer_queries(n, 1 << 20, seed=1)
    ms, cs, cols, amp = raw_slices(n)
    R = raw_width(n)
    params = np.zeros((G, R))
    params[:, ms] = feats[rng.integers(0, feats.shape[0], G)]
    for i in range(n):
        for j in range(i + 1):
            if i == j:
                params[:, cs.start + tri(i, j)] = math.log(sigma0) + rng.uniform(-0.5, 0.5, G)
            else:
                params[:, cs.start + tri(i, j)] = rng.normal(0.0, sigma0, G)
    params[:, cols] = rng.normal(0.0, 1.0, (G, 3))
    params[:, amp] = rng.normal(math.log(0.1) if amp_mode == BRIGHTNESS else -2.0, 0.5, G)
    return dict(params=params.astype(np.float32), child=np.zeros((G, R), np.float32), has_child=np.zeros(G, bool),
                frozen=np.zeros(G, bool))

def synthetic_targets(B: int, seed: int = 3) -> np.ndarray:
    return np.random.default_rng(seed).random((B, 3)).astype(np.float32)


# ------------------------------------------------------------------------------------------------
# device-side batch sampling and procedural targets
# ------------------------------------------------------------------------------------------------
class GmmOracleTarget:
    """gmm_oracle_target: a hidden mixture of the exact model family; targets are
    its exact (culling disabled) evaluation at the queries, on the GPU."""

    def __init__(self, seed: int, n_dims: int, n_components: int, amp_mode: int = BRIGHTNESS, device=None,
                 sigma0: float | None = None):
        import torch
        from .engine import HotPath
        from .gmm import Mixture
        self.n_dims = n_dims
        rows, self.sigma0 = synthetic_mixture(n_dims, n_components, seed=seed + 7919, amp_mode=amp_mode,
                                              sigma0=sigma0 if sigma0 is not None else 0.15)
        rows["params"][:, -1] = np.log(0.3) if amp_mode == BRIGHTNESS else 0.0
        self.mixture = Mixture.from_arrays(n_dims, amp_mode, **rows, device=device)
        self.hp = HotPath(n_dims, tile_size=256, device=self.mixture.device)
        self._torch = torch
        self._graph = None            # (key, GraphedEval) for the training loop's fixed batch buffers

    def __call__(self, queries):
        return self.hp.evaluate(self.mixture, queries, cull=False)

    def evaluate_into(self, queries, out):
        """The targets at `queries` into `out` without a host round trip: a GraphedEval captured for
        this (queries, out) buffer pair and replayed (the training loop draws every batch into the same
        buffers); other shapes / buffers fall back to the eager evaluation."""
        from .engine import GraphedEval
        key = (queries.data_ptr(), tuple(queries.shape), out.data_ptr())
        if queries.shape[0] % self.hp.tile:
            out.copy_(self(queries))
            return out
        if self._graph is None or self._graph[0] != key:
            self._graph = (key, GraphedEval(self.hp, self.mixture, queries, out, cull=False))
        self._graph[1]()
        return out


class ShadingToyTarget:
    """shading_toy_target: analytic shading-like function of
    position(3) | view direction(3) | albedo(3) | roughness(1) (first N of these roles, N in 4..10):
    a diffuse term smooth in position and modulated by albedo, plus a glossy cosine-power lobe around
    a position-dependent reflection direction whose exponent falls to its minimum at roughness 1.
    Evaluated by the `ndg_shading_target` kernel (csrc/ndg_sample.cu); the tests check it against the
    oracle's float64 restatement."""

    def __init__(self, seed: int, n_dims: int):
        if not 4 <= n_dims <= 10:
            raise ValueError("shading toy needs 4 <= N <= 10")
        rng = np.random.default_rng(seed)
        self.n_dims = n_dims
        self.freq = rng.uniform(1.0, 2.0, 3)
        self.phase = rng.uniform(0, 2 * np.pi, 3)
        self._params = {}

    def __call__(self, q, out=None):
        import ctypes

        import torch

        from . import kernels as K
        q = q.contiguous().float()
        p = self._params.get(q.device)
        if p is None:
            p = torch.tensor(np.concatenate([self.freq, self.phase]), dtype=torch.float32, device=q.device)
            self._params[q.device] = p
        if out is None:
            out = torch.empty(q.shape[0], 3, dtype=torch.float32, device=q.device)
        K.call("ndg_shading_target", self.n_dims, int(q.shape[0]), ctypes.c_void_p(q.data_ptr()),
               ctypes.c_void_p(p.data_ptr()), ctypes.c_void_p(out.data_ptr()),
               ctypes.c_void_p(torch.cuda.current_stream(q.device).cuda_stream))
        return out


class QuerySampler:
    """The stream of training batches: a counter-based generator (Philox4x32-10 keyed by seed, one draw
    index per batch) on the device, so its whole state is (seed, draw) -- checkpointed as two integers --
    and every rank of a data-parallel fit draws the same global batch."""

    def __init__(self, seed: int, draw: int = 0):
        self.seed, self.draw = int(seed) & ((1 << 64) - 1), int(draw)
        self._ws = None

    def state(self) -> dict:
        return dict(seed=self.seed, draw=self.draw)

    def set_state(self, st: dict):
        self.seed, self.draw = int(st["seed"]), int(st["draw"])

    def queries(self, n_dims: int, batch_size: int, tile_size: int, device, rank: int = 0, world: int = 1, out=None):
        """The next global batch, this rank's strided tiles of it (into `out` when given)."""
        import ctypes

        import torch

        from . import kernels as K
        T = batch_size // tile_size
        mine = len(range(rank, T, world))
        if out is None:
            q = torch.empty(mine * tile_size, n_dims, dtype=torch.float32, device=device)
        else:
            if tuple(out.shape) != (mine * tile_size, n_dims) or out.dtype != torch.float32 or not out.is_contiguous():
                raise ValueError("out must be a contiguous float32 [local batch, n_dims] tensor")
            q = out
        nb = int(K.load().ndg_sample_workspace(batch_size))
        if self._ws is None or self._ws.numel() * 8 < nb or self._ws.device != q.device:
            self._ws = torch.empty((nb + 7) // 8, dtype=torch.int64, device=device)
        K.call("ndg_sample_batch", n_dims, batch_size, tile_size, rank, world, ctypes.c_uint64(self.seed),
               ctypes.c_uint64(self.draw), ctypes.c_void_p(self._ws.data_ptr()), ctypes.c_void_p(q.data_ptr()),
               ctypes.c_void_p(torch.cuda.current_stream(q.device).cuda_stream))
        self.draw += 1
        return q


class FileDataset:
    """A tensor-file source: fixed queries [M, N] and targets [M, 3] resident in
    HBM. sample_batch draws random slices without replacement within an epoch (a fresh device-side
    permutation per epoch, seeded by (seed, epoch); a batch that runs past the end takes the rest and
    continues in the reshuffled next epoch), sorts the slice by the first (position) dimension into
    tiles, and -- when perturb_sigma > 0 -- adds clamped Gaussian noise of that scale to the
    direction-tagged dimensions of the queries only (perturb_directions). Its whole
    state is (seed, epoch, position, draw): four integers in the checkpoint."""

    def __init__(self, queries, targets, roles=None, *, seed: int = 0, perturb_sigma: float = 0.0, device=None):
        import torch
        q = torch.as_tensor(np.ascontiguousarray(queries, np.float32))
        t = torch.as_tensor(np.ascontiguousarray(targets, np.float32))
        if q.ndim != 2 or t.shape != (q.shape[0], 3):
            raise ValueError("queries [M, N] and targets [M, 3] required")
        if perturb_sigma < 0:
            raise ValueError("perturb_sigma must be >= 0")
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.q, self.t = q.to(self.device), t.to(self.device)
        self.n_dims, self.count = int(q.shape[1]), int(q.shape[0])
        self.roles = list(roles) if roles is not None else [3] * self.n_dims
        self.dir_dims = [i for i, r in enumerate(self.roles) if r == 1]          # formats.ROLES["direction"]
        self.seed, self.perturb_sigma = int(seed), float(perturb_sigma)
        self.epoch, self.pos, self.draw = 0, 0, 0
        self._perm = None

    @classmethod
    def from_ndgt(cls, path, **kw):
        from .formats import read_ndgt
        q, t, roles = read_ndgt(path)
        return cls(q, t, roles, **kw)

    def state(self) -> dict:
        return dict(seed=self.seed, epoch=self.epoch, pos=self.pos, draw=self.draw)

    def set_state(self, st: dict):
        self.seed, self.epoch, self.pos, self.draw = (int(st["seed"]), int(st["epoch"]), int(st["pos"]),
                                                      int(st["draw"]))
        self._perm = None

    _TAGS = {"epoch": 1, "perturb": 2, "init": 3}

    def _generator(self, tag: str, value: int = 0):
        """A device generator seeded by splitmix64 of (seed, tag, value): deterministic across processes."""
        import torch
        x = 0
        for v in (self.seed, self._TAGS[tag], value):
            x = (x ^ (v & 0xFFFFFFFFFFFFFFFF)) + 0x9E3779B97F4A7C15 & 0xFFFFFFFFFFFFFFFF
            x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9 & 0xFFFFFFFFFFFFFFFF
            x = (x ^ (x >> 27)) * 0x94D049BB133111EB & 0xFFFFFFFFFFFFFFFF
            x ^= x >> 31
        g = torch.Generator(device=self.device)
        g.manual_seed(x & ((1 << 63) - 1))
        return g

    def _permutation(self):
        import torch
        if self._perm is None or self._perm[0] != self.epoch:
            self._perm = (self.epoch, torch.randperm(self.count, generator=self._generator("epoch", self.epoch),
                                                     device=self.device))
        return self._perm[1]

    def _next_indices(self, B: int):
        import torch
        parts, need = [], B
        while need:
            take = min(need, self.count - self.pos)
            parts.append(self._permutation()[self.pos:self.pos + take])
            self.pos += take
            need -= take
            if self.pos == self.count:                     # epoch wrap: reshuffle
                self.epoch, self.pos = self.epoch + 1, 0
        return parts[0] if len(parts) == 1 else torch.cat(parts)

    def points(self, count: int):
        """`count` dataset points (initial means): the first of a seeded permutation."""
        import torch
        perm = torch.randperm(self.count, generator=self._generator("init"), device=self.device)
        return self.q[perm[:min(count, self.count)]]

    def batch(self, batch_size: int, tile_size: int, rank: int = 0, world: int = 1, out=None):
        import torch
        idx = self._next_indices(batch_size)
        q = self.q[idx]
        if self.perturb_sigma > 0 and self.dir_dims:
            d = torch.tensor(self.dir_dims, device=self.device)
            noise = torch.randn(batch_size, len(self.dir_dims), generator=self._generator("perturb", self.draw),
                                device=self.device) * self.perturb_sigma
            q[:, d] = (q[:, d] + noise).clamp_(0.0, 1.0)
        self.draw += 1
        order = torch.sort(q[:, 0], stable=True).indices      # tiles from spatially sorted queries
        T = batch_size // tile_size
        order = order.view(T, tile_size)[rank::world].reshape(-1)
        if out is None:
            return q[order].contiguous(), self.t[idx[order]].contiguous()
        torch.index_select(q, 0, order, out=out[0])
        torch.index_select(self.t, 0, idx[order], out=out[1])
        return out


def sample_batch(target, n_dims: int, batch_size: int, tile_size: int, sampler, device, rank: int = 0,
                 world: int = 1, out=None):
    """SPEC.md:440-448 on the device: fresh uniform queries, sorted by the first (position) dimension
    into contiguous tiles, exact targets. batch_size must be a multiple of tile_size. `sampler` is a
    QuerySampler (or an int seed for a one-off batch); the sort is generated, not performed
    (csrc/ndg_sample.cu: the sorted first coordinates are uniform order statistics).

    Data-parallel (world > 1): every rank draws the same GLOBAL batch and keeps its strided tiles (global
    tile i -> rank i mod world, parallel.shard_tiles), evaluating the target only there -- so the union
    over ranks is exactly the 1-GPU batch and the summed gradients equal the 1-GPU step's.
    `out` = (queries, targets) buffers to fill (e.g. a GraphedStep's inputs)."""
    if batch_size % tile_size:
        raise ValueError("batch_size must be a multiple of tile_size (SPEC.md:441)")
    T = batch_size // tile_size
    if world > 1 and T < world:
        raise ValueError(f"{T} tiles cannot give each of {world} ranks one (batch_size / tile_size >= world)")
    if isinstance(target, FileDataset):                     # file source: its own epoch / slice state
        return target.batch(batch_size, tile_size, rank, world, out=out)
    if not isinstance(sampler, QuerySampler):
        sampler = QuerySampler(int(sampler))
    if out is None:
        q = sampler.queries(n_dims, batch_size, tile_size, device, rank, world)
        return q, target(q).contiguous()
    q = sampler.queries(n_dims, batch_size, tile_size, device, rank, world, out=out[0])
    if isinstance(target, ShadingToyTarget):
        target(q, out=out[1])
    elif isinstance(target, GmmOracleTarget):
        target.evaluate_into(q, out[1])
    else:
        out[1].copy_(target(q))
    return out
