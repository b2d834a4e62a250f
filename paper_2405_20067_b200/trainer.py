"""Fit loop with optimizer-controlled refinement (reference module trainer).

One iteration: sample batch → tile → cull → forward → loss → backward → Adam, i.e. one
`HotPath.fwd_bwd` (K1-K8, plus the single NCCL all_reduce when data-parallel) and one `adam_step`
(K9) on the device. Refinement events run between iterations ("single threaded between
iterations") every `phase_length` iterations after `warmup_phases` phases, on the device (tensor ops
on the SoA rows; the composed child factors come from K1): check_materialize → materialize →
spawn_children, and components whose activated amplitude stayed below t/100 for a
whole phase are frozen out. New rows and children start with zeroed Adam moments
(SPEC.md:322).

Frozen components are compacted out of the working set: their rows move to an archive and the K1-K8
passes, Adam and the allreduce only see live rows. Every row keeps an id (its position in the
reference's ordered mixture: original rows first, materialized rows appended in event order), and
`full_mixture()` / `full_state()` merge the archive back in id order for checkpoints and results, so
the saved mixture is the one the uncompacted loop would hold (frozen rows in place, flagged).
"""
from __future__ import annotations

import math
import time
from dataclasses import dataclass, field

import numpy as np
import torch

from . import datasets as D
from .engine import GraphedStep, HotPath, adam_step, new_adam_state
from .errors import NonFiniteGradientError, TrainingAborted
from .gmm import BRIGHTNESS, FLAG_CHILD, FLAG_FROZEN, Mixture, n_chol, raw_slices, raw_width, tri


@dataclass
class TrainConfig:
    """SPEC.md:309-318 with the ledger defaults."""
    iterations: int = 1000
    phase_length: int = 300
    warmup_phases: int = 1
    materialize_threshold: float | None = None      # default: 0.1 opacity / 0.01 brightness
    lr_mean: float = 2e-3
    lr_chol: float = 5e-3
    lr_color: float = 1e-2
    lr_amp: float = 1e-2
    beta1: float = 0.9
    beta2: float = 0.999
    adam_eps: float = 1e-8
    batch_size: int = 1 << 16
    tile_size: int = 256
    seed: int = 0
    k: int = 16
    multiplier: float = 3.0
    loss_eps: float = 0.01
    cull: bool = True
    n_components: int = 256
    amp_mode: int = BRIGHTNESS
    graph: bool = True          # replay the step as a CUDA graph when the worst-case list is small (GraphedStep)

    def threshold(self) -> float:
        return self.materialize_threshold if self.materialize_threshold is not None else \
            D.default_threshold(self.amp_mode)


@dataclass
class MetricsRow:
    """metrics.csv row: iteration,loss,n_components,culled_fraction,ms_per_iter."""
    iteration: int
    loss: float
    n_components: int
    culled_fraction: float
    ms_per_iter: float


@dataclass
class TrainResult:
    mixture: Mixture
    metrics: list = field(default_factory=list)
    events: list = field(default_factory=list)


# ------------------------------------------------------------------------------------------------
# activation helpers for the refinement events (host, float64, between iterations)
# ------------------------------------------------------------------------------------------------
def _sigmoid(x):
    return 1.0 / (1.0 + np.exp(-x))


def _activate(chol_raw, n):
    L = np.zeros(chol_raw.shape[:-1] + (n, n))
    for i in range(n):
        for j in range(i + 1):
            r = chol_raw[..., tri(i, j)]
            L[..., i, j] = np.exp(r) if i == j else 2.0 * _sigmoid(r) - 1.0
    return L


def spawn_rows(n, count, mode, t, rng):
    """spawn_children: U = I, m_u = 0, color_raw in +-0.1, activated amp = t/10."""
    ms, cs, cols, amp = raw_slices(n)
    rows = np.zeros((count, raw_width(n)), np.float32)
    rows[:, cols] = rng.uniform(-0.1, 0.1, (count, 3))
    rows[:, amp] = D.amp_inverse(t / 10.0, mode)
    return rows


def initial_mixture(cfg: TrainConfig, n_dims: int, points: torch.Tensor, device) -> Mixture:
    """Means from dataset points, per-dimension sigma = half the mean nearest-neighbour distance,
    zero off-diagonals; neutral colour; amplitude 0.5 of the brightness scale."""
    pts = points[: cfg.n_components].double().cpu().numpy()
    s0 = D.nn_sigma0(pts)
    ms, cs, cols, amp = raw_slices(n_dims)
    rows = np.zeros((cfg.n_components, raw_width(n_dims)), np.float32)
    rows[:, ms] = pts
    for i in range(n_dims):
        rows[:, cs.start + tri(i, i)] = math.log(max(s0, 1e-3))
    rows[:, amp] = D.amp_inverse(0.5 if cfg.amp_mode == BRIGHTNESS else 0.5, cfg.amp_mode)
    return Mixture.from_arrays(n_dims, cfg.amp_mode, rows, device=device)


class Trainer:
    """Holds the device state of one fit: mixture, Adam moments, freeze counters, hot path."""

    def __init__(self, cfg: TrainConfig, target, n_dims: int, *, mixture: Mixture | None = None, device=None,
                 allreduce=None, rank: int = 0, world: int = 1):
        self.cfg, self.target, self.n = cfg, target, n_dims
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        # the batch stream (counter-based, device-side) is seeded identically on every rank: each draws
        # the same global batch and keeps its own tiles (datasets.sample_batch), so the ranks' tiles
        # partition the 1-GPU batch
        self.sampler = D.QuerySampler(cfg.seed * 1000003 + 1)
        self.rng = np.random.default_rng(cfg.seed)
        self.allreduce, self.rank, self.world = allreduce, rank, world
        if mixture is None and isinstance(target, D.FileDataset):
            mixture = initial_mixture(cfg, n_dims, target.points(cfg.n_components), self.device)
        elif mixture is None:
            # initial means from data points: a one-off draw, identical on every rank; the
            # first coordinate of a sorted draw is ordered, so pick the points by a seeded permutation
            q0 = D.QuerySampler(cfg.seed).queries(n_dims, max(cfg.tile_size, cfg.n_components), 1, self.device)
            perm = np.random.default_rng(cfg.seed).permutation(q0.shape[0])
            mixture = initial_mixture(cfg, n_dims, q0[torch.from_numpy(perm).to(self.device)], self.device)
        self.mix = mixture
        self.ids = torch.arange(self.mix.G, dtype=torch.int64, device=self.device)
        self.next_id = self.mix.G
        self.archive = None           # frozen rows compacted out of the working set (params, child, flags, ids)
        self.hp = HotPath(n_dims, k=cfg.k, multiplier=cfg.multiplier, tile_size=cfg.tile_size, eps=cfg.loss_eps,
                          projection_seed=cfg.seed, device=self.device)
        self.state = new_adam_state(self.mix)
        self.low_count = torch.zeros(self.mix.G, dtype=torch.int32, device=self.device)
        self.step_no = 0
        self.last_allreduce_bytes = 0
        self.phase_stats = None       # [Gev, 3] float64 on the device: the phase's density statistics
        self.last_good = self.mix.clone()
        self._gs = None               # the captured step of the current working set (GraphedStep)
        self._gbuf = None             # its static (queries, targets) buffers
        self._n_frozen = int(((self.mix.flags & FLAG_FROZEN) != 0).sum())   # host mirror (changes at events)

    # -- one iteration -----------------------------------------------------------------------
    def iteration(self) -> MetricsRow:
        cfg = self.cfg
        t0 = time.perf_counter()
        try:
            res = self._step()
        except NonFiniteGradientError as err:                       # a training abort
            self.mix = self.last_good.clone()
            self._gs = None
            raise TrainingAborted(f"non-finite gradient at iteration {self.step_no} ({self._batch_name()}; "
                                  f"component {err.component}, block {err.block}, batch index {err.batch_index})",
                                  iteration=self.step_no) from err
        self.last_allreduce_bytes = res.grads.reduced().numel() * 4 if self.allreduce is not None else 0
        if not math.isfinite(res.loss):
            self.mix = self.last_good.clone()
            self._gs = None
            raise TrainingAborted(f"non-finite loss at iteration {self.step_no} ({self._batch_name()})",
                                  iteration=self.step_no)
        self.step_no += 1
        st = res.grads.stats.double()
        if self.phase_stats is None or self.phase_stats.shape != st.shape:
            self.phase_stats = torch.zeros_like(st)
        self.phase_stats += st
        adam_step(self.mix, res.grads, self.state, self.step_no,
                  lr=(cfg.lr_mean, cfg.lr_chol, cfg.lr_color, cfg.lr_amp), betas=(cfg.beta1, cfg.beta2),
                  eps=cfg.adam_eps)
        amp_col = raw_width(self.n) - 1
        alpha = self.mix.params[:, amp_col]
        alpha = torch.exp(alpha) if cfg.amp_mode == BRIGHTNESS else torch.sigmoid(alpha)
        low = alpha < cfg.threshold() / 100.0
        self.low_count = torch.where(low, self.low_count + 1, torch.zeros_like(self.low_count))
        ms = (time.perf_counter() - t0) * 1e3
        return MetricsRow(self.step_no, res.loss, int(self.live_components()), 1.0 - res.kept_fraction, ms)

    def _batch_name(self) -> str:
        """The offending batch of an abort: the state that regenerates it."""
        if isinstance(self.target, D.FileDataset):
            st = self.target.state()
            return f"file batch {st['draw'] - 1}, epoch {st['epoch']}"
        return f"batch draw {self.sampler.draw - 1} of sampler seed {self.sampler.seed}"

    def _step(self):
        """sample_batch + fwd_bwd (+ the allreduce). Small working sets (worst-case candidate list <= 2^24)
        replay one CUDA graph per step (engine.GraphedStep, byte-identical to the eager step), captured
        again whenever a refinement event replaced the working set; the batch is drawn straight into its
        input buffers."""
        cfg = self.cfg
        T = cfg.batch_size // cfg.tile_size
        B_local = len(range(self.rank, T, self.world)) * cfg.tile_size
        if not (cfg.graph and cfg.cull and GraphedStep.eligible(self.hp, self.mix, B_local)):
            q, tg = D.sample_batch(self.target, self.n, cfg.batch_size, cfg.tile_size, self.sampler, self.device,
                                   self.rank, self.world)
            return self.hp.fwd_bwd(self.mix, q, tg, cull=cfg.cull, n_total=cfg.batch_size, allreduce=self.allreduce)
        if self._gbuf is None:
            self._gbuf = (torch.empty(B_local, self.n, dtype=torch.float32, device=self.device),
                          torch.empty(B_local, 3, dtype=torch.float32, device=self.device))
        qs, ts = self._gbuf
        D.sample_batch(self.target, self.n, cfg.batch_size, cfg.tile_size, self.sampler, self.device, self.rank,
                       self.world, out=(qs, ts))
        if self._gs is None or not self._gs.matches(self.mix):
            self._gs = GraphedStep(self.hp, self.mix, qs, ts, n_total=cfg.batch_size)
        return self._gs(allreduce=self.allreduce)

    # -- resume state (resume is bit-identical) ----------------------------
    def rng_state(self) -> dict:
        """Everything random that the future of the fit depends on: the batch stream's (seed, draw)
        (identical on every rank; for a file source its (seed, epoch, position, draw)) and the full numpy
        PCG64 state of the spawn RNG."""
        st = dict(seed=self.cfg.seed, sampler=self.sampler.state(), numpy=self.rng.bit_generator.state)
        if isinstance(self.target, D.FileDataset):
            st["dataset"] = self.target.state()
        return st

    def set_rng_state(self, st: dict):
        if isinstance(st.get("sampler"), dict):
            self.sampler.set_state(st["sampler"])
        if isinstance(st.get("dataset"), dict) and isinstance(self.target, D.FileDataset):
            self.target.set_state(st["dataset"])
        if isinstance(st.get("numpy"), dict):
            self.rng.bit_generator.state = st["numpy"]

    def live_components(self) -> int:
        return self.mix.G - self._n_frozen         # frozen rows are archived at events (host mirror, no sync)

    # -- refinement events ---------------------------------------------
    def density_summary(self) -> dict:
        """The phase's density-control statistics (north_star; gathered inside K7, summed over the
        phase's iterations on the device): totals, the components no tile query reached (zero pairs)
        and the components carrying the largest loss share. Reported with every refinement event."""
        if self.phase_stats is None:
            return {}
        ps = self.phase_stats.cpu().numpy()
        G = self.mix.G
        parent = ps[:G]
        out = dict(loss_share=float(ps[:, 0].sum()), grad_proxy=float(ps[:, 1].sum()), pairs=float(ps[:, 2].sum()),
                   unreached_components=int(np.count_nonzero(parent[:, 2] == 0)),
                   top_loss_share=[int(i) for i in np.argsort(-parent[:, 0], kind="stable")[:8]])
        if ps.shape[0] == 2 * G:
            out["child_loss_share"] = float(ps[G:, 0].sum())
        return out

    def phase_event(self):
        """One refinement boundary: freeze-out, check_materialize + materialize, spawn_children. The
        event record carries the phase's density statistics (density_summary)."""
        stats = self.density_summary()
        self.phase_stats = None
        ev = self.materialize_step()
        ev["spawned"] = self.spawn_step()
        ev["n_components"] = self.mix.G + (0 if self.archive is None else int(self.archive["ids"].numel()))
        ev["live_components"] = self.mix.G
        ev["density_stats"] = stats
        self.last_good = self.mix.clone()
        return ev

    # -- working set <-> the reference's ordered mixture ---------------------------------------------
    def _compact(self):
        """Move frozen rows (out of optimisation and evaluation) to the archive."""
        fr = (self.mix.flags & FLAG_FROZEN) != 0
        if not bool(fr.any()):
            self._n_frozen = 0
            return 0
        keep = ~fr
        moved = dict(params=self.mix.params[fr], child=self.mix.child[fr], flags=self.mix.flags[fr], ids=self.ids[fr])
        self.archive = moved if self.archive is None else {k: torch.cat([self.archive[k], moved[k]])
                                                            for k in moved}
        fl = self.mix.flags[keep].contiguous()
        self.mix = Mixture(self.n, self.cfg.amp_mode, self.mix.params[keep].contiguous(),
                           self.mix.child[keep].contiguous(), fl, bool(((fl & FLAG_CHILD) != 0).any()))
        self.state = {k: v[keep].contiguous() for k, v in self.state.items()}
        self.low_count = self.low_count[keep].contiguous()
        self.ids = self.ids[keep].contiguous()
        self._n_frozen = 0
        return int(fr.sum())

    def _merged(self, active: dict, archived: dict):
        if self.archive is None:
            return active
        order = torch.argsort(torch.cat([self.ids, self.archive["ids"]]))
        return {k: torch.cat([active[k], archived[k]])[order].contiguous() for k in active}

    def full_mixture(self) -> Mixture:
        """The whole ordered mixture: live rows and the archived frozen rows (flagged), in id order."""
        m = self._merged(dict(params=self.mix.params, child=self.mix.child, flags=self.mix.flags),
                         self.archive or {})
        fl = m["flags"]
        return Mixture(self.n, self.cfg.amp_mode, m["params"], m["child"], fl,
                       bool((((fl & FLAG_CHILD) != 0) & ((fl & FLAG_FROZEN) == 0)).any()))

    def full_state(self):
        """(Adam moments, low-amplitude counters) over the whole ordered mixture; archived rows: zeros."""
        na = 0 if self.archive is None else int(self.archive["ids"].numel())
        z = lambda v: torch.zeros((na,) + tuple(v.shape[1:]), dtype=v.dtype, device=v.device)  # noqa: E731
        st = self._merged(dict(self.state), {k: z(v) for k, v in self.state.items()})
        lc = self._merged(dict(lc=self.low_count), dict(lc=z(self.low_count)))["lc"]
        return st, lc

    def resume(self, ckpt: dict):
        """Continue from a checkpoint: iteration, Adam moments, freeze counters and RNG
        state over the saved ordered mixture (this Trainer was built on it), then compact."""
        self.step_no = int(ckpt["iteration"])
        for k in ("m1p", "m2p", "m1c", "m2c"):
            self.state[k] = torch.from_numpy(np.ascontiguousarray(ckpt[k])).to(self.device)
        self.low_count = torch.from_numpy(np.ascontiguousarray(ckpt["low_count"])).to(self.device)
        self.set_rng_state(ckpt.get("rng", {}))
        self._compact()
        self.last_good = self.mix.clone()

    def materialize_step(self):
        """Freeze-out, then check_materialize and materialize
        (SPEC.md:356-364): each selected child becomes a standalone component with the composed mean
        and factor (K1's float64 m_c = L m_u + m_p and L U), activations inverted with off-diagonal
        clamping to +-(1 - 1e-6); its parent loses the child. All on the device."""
        cfg, n = self.cfg, self.n
        t = cfg.threshold()
        ms, cs, cols, amp = raw_slices(n)
        mix = self.mix
        G = mix.G
        flags = mix.flags.clone()
        newly_frozen = (self.low_count >= cfg.phase_length) & ((flags & FLAG_FROZEN) == 0)
        flags = torch.where(newly_frozen, (flags | FLAG_FROZEN) & ~FLAG_CHILD, flags)
        has_child = (flags & FLAG_CHILD) != 0
        camp = mix.child[:, amp].double()
        alpha = torch.exp(camp) if cfg.amp_mode == BRIGHTNESS else torch.sigmoid(camp)
        sel = torch.nonzero(has_child & (alpha >= t)).flatten()
        k = int(sel.numel())
        clamped = 0
        if k:
            recs = self.hp.activate(mix)                 # composed child rows e = G + i, float64
            e = G + sel
            new_rows = torch.zeros(k, raw_width(n), dtype=torch.float64, device=self.device)
            new_rows[:, ms] = recs.mean64[e]
            L = recs.chol64[e]
            raw = torch.empty_like(L)
            lim = 1.0 - 1e-6
            for i in range(n):
                for j in range(i + 1):
                    v = L[:, tri(i, j)]
                    if i == j:
                        raw[:, tri(i, j)] = torch.log(v)
                    else:
                        vc = v.clamp(-lim, lim)
                        clamped += int((vc != v).sum())
                        s_ = (vc + 1.0) / 2.0
                        raw[:, tri(i, j)] = torch.log(s_) - torch.log1p(-s_)
            new_rows[:, cs] = raw
            new_rows[:, cols] = mix.child[sel][:, cols].double()
            new_rows[:, amp] = mix.child[sel][:, amp].double()
            flags[sel] = flags[sel] & ~FLAG_CHILD
            zf = torch.zeros(k, raw_width(n), dtype=torch.float32, device=self.device)
            params = torch.cat([mix.params, new_rows.float()])
            child = torch.cat([mix.child, zf])
            flags = torch.cat([flags, torch.zeros(k, dtype=torch.uint8, device=self.device)])
            self.state = {key: torch.cat([v, zf]) for key, v in self.state.items()}   # zero moments
            self.low_count = torch.cat([self.low_count, torch.zeros(k, dtype=torch.int32, device=self.device)])
            self.ids = torch.cat([self.ids, torch.arange(self.next_id, self.next_id + k, dtype=torch.int64,
                                                         device=self.device)])
            self.next_id += k
        else:
            params, child = mix.params, mix.child
        self.mix = Mixture(n, cfg.amp_mode, params.contiguous(), child.contiguous(), flags.contiguous(),
                           bool((((flags & FLAG_CHILD) != 0) & ((flags & FLAG_FROZEN) == 0)).any()))
        self.low_count.zero_()
        self._compact()
        return dict(iteration=self.step_no, materialized=k, frozen=int(newly_frozen.sum()), clamped=int(clamped))

    def spawn_step(self) -> int:
        """spawn_children: every live component without a child gets one (U = I,
        m_u = 0, colour in +-0.1 raw from the checkpointed spawn RNG, activated amplitude t/10) with
        zeroed moments."""
        cfg, n = self.cfg, self.n
        mix = self.mix
        needs = ((mix.flags & FLAG_CHILD) == 0) & ((mix.flags & FLAG_FROZEN) == 0)
        cnt = int(needs.sum())
        if cnt:
            rows = torch.from_numpy(spawn_rows(n, cnt, cfg.amp_mode, cfg.threshold(), self.rng)).to(self.device)
            child = mix.child.clone()
            child[needs] = rows
            for key in ("m1c", "m2c"):
                self.state[key][needs] = 0.0
            flags = torch.where(needs, mix.flags | FLAG_CHILD, mix.flags)
            self.mix = Mixture(n, cfg.amp_mode, mix.params, child, flags.contiguous(), True)
        return cnt


def train(cfg: TrainConfig, target, n_dims: int, *, mixture: Mixture | None = None, device=None, allreduce=None,
          rank: int = 0, world: int = 1, callback=None) -> TrainResult:
    """SPEC.md:326-334. Returns the final mixture, one MetricsRow per iteration and the refinement
    events. 0 iterations returns the initial mixture unchanged."""
    tr = Trainer(cfg, target, n_dims, mixture=mixture, device=device, allreduce=allreduce, rank=rank, world=world)
    out = TrainResult(tr.mix)
    for it in range(cfg.iterations):
        row = tr.iteration()
        out.metrics.append(row)
        if callback:
            callback(tr, row)
        if (it + 1) % cfg.phase_length == 0 and (it + 1) // cfg.phase_length >= cfg.warmup_phases:
            out.events.append(tr.phase_event())
    out.mixture = tr.full_mixture()
    return out


def held_out_rel_l2(mix: Mixture, target, n_dims: int, n: int = 1 << 14, seed: int = 12345, tile_size: int = 256):
    """Relative L2 of the mixture against the target on fresh held-out queries."""
    q, tg = D.sample_batch(target, n_dims, n, tile_size, D.QuerySampler(seed), mix.device)
    hp = HotPath(n_dims, tile_size=tile_size, device=mix.device)
    pred = hp.evaluate(mix, q, cull=True)
    return float(torch.linalg.norm(pred - tg) / torch.linalg.norm(tg))
