#!/usr/bin/env python
"""Benchmark of the culled N-D Gaussian-mixture fwd+bwd step (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--regime R|C]

Workload (BASELINE.json configs[1], the metric's configuration): 10-D mixture of 100k Gaussians,
2^20 queries per GPU per step, tiles of 256 queries sorted by dim 0 (regime R, the reference
sampler SPEC.md:443), k = 16 projection vectors, multiplier 3, relative-L2 loss eps 0.01.
A step = K1 prologue, K2 projections, K3 tile bounds, K4 binning, K5+K6 forward+loss,
K7 backward, K8 epilogue, [NCCL allreduce of the flat gradient buffer when N > 1], K9 Adam.
`value` = queries processed by all ranks / max-over-ranks device time of K steps (CUDA events),
inputs resident in HBM, L2 flushed (256 MiB write) before every timed step.
`e2e` = the same step through the public API with pinned-host inputs copied in every step and the
loss read back. Rank 0 prints one JSON line.

--impl reference times the reference's CPU path on the host cores: the reference ships no
runnable implementation, so this is oracle/ndg_oracle.c -- the C/OpenMP
restatement of SPEC.md standing in for the reference's intended `_core` (pkg/setup.py:36-43) --
on a bounded sample of the same workload (whole tiles x all Gaussians, every stage parallel within a
tile so all host threads are busy); its rate is the sample's queries over its measured wall time.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "culled query evals/sec (fwd+bwd) at 10-D, 1/2/4/8 B200; % of FP32/HBM roofline"
NOMINAL_FP32_TFLOPS = 2 * 128 * 148 * 1.965e9 / 1e12     # 74.4, datasheet-class (not measured)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--regime", choices=["R", "C", "G"], default="R")
    ap.add_argument("--n-dims", type=int, default=10)
    ap.add_argument("--gaussians", type=int, default=100_000)
    ap.add_argument("--batch", type=int, default=1 << 20, help="queries per GPU per step")
    ap.add_argument("--tile", type=int, default=256)
    ap.add_argument("--k", type=int, default=16)
    ap.add_argument("--children", action="store_true", help="every component carries a live child (Gev = 2G)")
    ap.add_argument("--graph", choices=["auto", "on", "off"], default="auto",
                    help="replay the step as one CUDA graph (auto: when the worst-case candidate list is <= 2^24)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-secondary", action="store_true", help="skip the regime-C secondary measurement")
    ap.add_argument("--cpu-seconds", type=float, default=12.0, help="target CPU sample duration")
    return ap.parse_args()


def config_label(a) -> str:
    """BASELINE.json config this workload matches (configs[i] -> "cfg{i+1}"), else "custom"."""
    table = {(6, 4096, 16384): "cfg1", (10, 100_000, 1 << 20): "cfg2", (16, 500_000, 1 << 22): "cfg4",
             (10, 1_000_000, 1 << 19): "cfg5 (per-GPU shard of 2^22 at 8 GPUs)"}
    return table.get((a.n_dims, a.gaussians, a.batch), "custom")


def workload_name(a, regime):
    return (f"{config_label(a)}: {a.n_dims}-D synthetic shading-shaped mixture, {a.gaussians} Gaussians"
            f"{' (+live children)' if a.children else ''}, {a.batch} queries/GPU/step, tile {a.tile}, "
            f"k={a.k}, multiplier 3, regime {regime} "
            f"({ {'R': 'U[0,1)^N sorted by dim 0', 'C': 'coherent tiles, spread 0.01', 'G': 'G-buffer-like: 2-D manifold, 16x16-pixel tiles, mixture seeded on the manifold, sigma0 0.005'}[regime] })")


# ------------------------------------------------------------------------------------------------
# CPU baseline (oracle/ndg_oracle.c, all host threads, bounded sample)
# ------------------------------------------------------------------------------------------------
def _sample_tiles(q, t, tile, S):
    """S whole tiles spread evenly over the batch (tile i*T/S), gathered contiguously."""
    import numpy as np
    T = q.shape[0] // tile
    sel = (np.arange(S) * T) // S
    rows = (sel[:, None] * tile + np.arange(tile)[None, :]).reshape(-1)
    return np.ascontiguousarray(q[rows]), np.ascontiguousarray(t[rows])


def cpu_sample(a, mix_np, q, t, R, target_s, steps=1, warmup=0):
    """Time the C/OpenMP restatement (oracle/ndg_oracle.c, every host thread) on a bounded sample of
    the workload: S whole tiles spread over the batch x ALL Gaussians, one full step each (activation,
    projections, tile bounds, cull, forward, loss, backward, epilogue). Every stage is parallel WITHIN
    a tile (queries for the forward, Gaussian blocks for the cull and the backward), so one tile
    already keeps every thread busy. The reported rate is the sample's own queries / its measured
    wall time -- no extrapolation -- with the per-Gaussian fixed costs paid once per sampled step."""
    import numpy as np

    from oracle import c_oracle as CO
    from oracle import ndg_oracle as O

    CO.build()
    # torchrun exports OMP_NUM_THREADS=1 to every rank; the baseline runs on rank 0 alone and uses
    # every host core it is allowed on
    CO.set_threads(len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1))
    threads = CO.max_threads()
    om = O.OMixture(a.n_dims, 0, mix_np["params"].astype(np.float64), mix_np["child"].astype(np.float64),
                    mix_np["has_child"], mix_np["frozen"])
    T = q.shape[0] // a.tile

    def run(S):
        qs, ts = _sample_tiles(q, t, a.tile, S)
        t0, c0 = time.perf_counter(), time.process_time()
        CO.step(om, qs, ts, R, tile=a.tile, n_total=q.shape[0])
        return time.perf_counter() - t0, time.process_time() - c0

    w1, _ = run(1)
    S = int(max(1, min(T, round(target_s / max(w1, 1e-6)))))
    walls, cpus = [], []
    for i in range(warmup + steps):
        w, c = run(S)
        if i >= warmup:
            walls.append(w)
            cpus.append(c)
    wall = statistics.median(walls)
    util = sum(cpus) / max(sum(walls), 1e-9) / threads
    return dict(value=S * a.tile / wall, step_s=wall, walls=walls, tiles=S, threads=threads, utilization=util,
                queries=S * a.tile,
                sample=f"{S} of {T} tiles (every {T // S}th, {S * a.tile} queries) x all {om.G} Gaussians per step, "
                       f"full step (activation .. epilogue) on {threads} threads; value = sampled queries / measured "
                       f"wall time (no extrapolation); measured CPU utilisation {util:.2f}")


def reference_arm(a, rank, world):
    """--impl reference: the reference's CPU path (C restatement, all host threads), rank 0 only.
    A step is one bounded sample of the workload (cpu_sample), sized so W + K steps take a few
    minutes; ms_per_step is that sample's measured wall time."""
    if rank != 0:
        return
    from oracle import ndg_oracle as O
    from paper_2405_20067_b200 import datasets as D
    mix_np, _ = D.synthetic_mixture(a.n_dims, a.gaussians, seed=0, children=a.children)
    q = D.synthetic_queries(a.n_dims, a.batch, seed=1, regime=a.regime, tile_size=a.tile)
    t = D.synthetic_targets(a.batch, seed=3)
    R = O.make_projection_set(a.n_dims, a.k, 2)
    per = max(2.0, min(a.cpu_seconds, 150.0 / max(1, a.steps + a.warmup)))
    info = cpu_sample(a, mix_np, q, t, R, per, steps=a.steps, warmup=a.warmup)
    v = info["value"]
    line = dict(metric=METRIC, value=v, unit="queries/s", n_gpus=world, steps=a.steps, warmup=a.warmup,
                ms_per_step=info["step_s"] * 1e3, higher_is_better=True, scaling="weak", vs_baseline=None,
                dtype="f64", data="synthetic", impl="reference",
                config=dict(workload=workload_name(a, a.regime), n_dims=a.n_dims, gaussians=a.gaussians,
                            batch_per_gpu=a.batch, tile=a.tile, k=a.k, multiplier=3.0, regime=a.regime,
                            queries_per_timed_step=info["queries"]),
                cpu_baseline=dict(value=v, unit="queries/s", cores=info["threads"], kind="port",
                                  sample=info["sample"], cpu=_cpu_model(), utilization=info["utilization"],
                                  per_step_values=[round(info["queries"] / w, 3) for w in info["walls"]]),
                e2e=dict(value=v, unit="queries/s", h2d_bytes_per_step=0, d2h_bytes_per_step=0),
                note="reference ships no runnable implementation (SURVEY.md §0); timed: oracle/ndg_oracle.c "
                     "(C/OpenMP restatement of SPEC.md, stand-in for the absent compiled _core)")
    print(json.dumps(line), flush=True)


def _cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


# ------------------------------------------------------------------------------------------------
# clocks during the timed region
# ------------------------------------------------------------------------------------------------
class ClockSampler:
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    """nvidia-smi polling every 100 ms, started BEFORE the warm-up: its NVML start-up stalls the driver for
    tens of ms, which inflated short host-latency-bound timed regions when it was launched inside them.
    Rows are stamped on arrival; stop() keeps those that arrived inside [begin(), end()] (or, for a timed
    region shorter than the poll period, the first row after begin())."""

    def __init__(self, gpu_index):
        import threading
        self.rows, self.t0, self.t1 = [], None, None
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                       "-i", str(gpu_index), "-lms", "100"], stdout=subprocess.PIPE,
                                      stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.p = None
            return
        self.th = threading.Thread(target=self._read, daemon=True)
        self.th.start()
        deadline = time.monotonic() + 10.0
        while not self.rows and time.monotonic() < deadline and self.p.poll() is None:
            time.sleep(0.02)                      # wait until NVML is up and sampling

    def _read(self):
        for line in self.p.stdout:
            if line.count(",") >= 8:
                self.rows.append((time.monotonic(), line.strip().split(",")))

    def begin(self):
        self.t0 = time.monotonic()

    def end(self):
        self.t1 = time.monotonic()

    def stop(self):
        if self.p is None:
            return dict(sm_mhz=None, sm_max_mhz=None, reasons=["nvidia-smi unavailable"])
        if self.t1 is not None and not any(t >= self.t0 for t, _ in self.rows):
            time.sleep(0.25)                      # region shorter than the poll period: take the next row
        self.p.terminate()
        try:
            self.p.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.p.kill()
        self.th.join(timeout=5)
        t0 = self.t0 if self.t0 is not None else 0.0
        t1 = self.t1 if self.t1 is not None else float("inf")
        inside = [r for t, r in self.rows if t0 <= t <= t1]
        rows = inside or [r for t, r in self.rows if t >= t0][:1]
        if not rows:
            return dict(sm_mhz=None, sm_max_mhz=None, reasons=["no samples"])
        sm = [float(r[1]) for r in rows]
        mx = max(float(r[2]) for r in rows)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[j] for r in rows for j in range(4) if r[5 + j].strip() == "Active"})
        return dict(sm_mhz=statistics.median(sm), sm_max_mhz=mx, reasons=reasons, samples=len(rows),
                    power_w_max=max(float(r[3]) for r in rows if r[3].strip() not in ("", "[N/A]")))


# ------------------------------------------------------------------------------------------------
# our arm
# ------------------------------------------------------------------------------------------------
def fp32_peak(torch, K, dev):
    """Measured FFMA rate of this GPU (TFLOP/s) -- the roofline denominator for K5 / K7."""
    out = torch.empty(256, device=dev)
    blocks, iters = 148 * 8, 4096
    s = torch.cuda.current_stream()
    import ctypes
    for _ in range(2):
        K.call("ndg_fp32_probe", ctypes.c_void_p(out.data_ptr()), blocks, iters, ctypes.c_void_p(s.cuda_stream))
    best = 0.0
    for _ in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        K.call("ndg_fp32_probe", ctypes.c_void_p(out.data_ptr()), blocks, iters, ctypes.c_void_p(s.cuda_stream))
        b.record()
        b.synchronize()
        best = max(best, K.load().ndg_fp32_probe_flops(blocks, iters) / (a.elapsed_time(b) * 1e-3) / 1e12)
    return best


def tf32_peak(torch, K, dev):
    """Measured dense TF32 tcgen05 rate (TFLOP/s) -- the tensor roofline of the TC forward."""
    import ctypes
    out = torch.empty(256, device=dev)
    s = torch.cuda.current_stream()
    blocks, iters = 148, 20000
    K.call("ndg_tf32_probe", ctypes.c_void_p(out.data_ptr()), blocks, iters, ctypes.c_void_p(s.cuda_stream))
    best = 0.0
    for _ in range(3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        K.call("ndg_tf32_probe", ctypes.c_void_p(out.data_ptr()), blocks, iters, ctypes.c_void_p(s.cuda_stream))
        b.record()
        b.synchronize()
        best = max(best, K.load().ndg_tf32_probe_flops(blocks, iters) / (a.elapsed_time(b) * 1e-3) / 1e12)
    return best


def hmma_peak(torch, K, dev):
    """Measured mma.sync m16n8k8 tf32 rate (TFLOP/s) -- the tensor roofline of the warp-MMA K7."""
    import ctypes
    out = torch.empty(512, device=dev)
    s = torch.cuda.current_stream()
    blocks, iters = 148, 4000
    K.call("ndg_hmma_probe", ctypes.c_void_p(out.data_ptr()), blocks, iters, ctypes.c_void_p(s.cuda_stream))
    best = 0.0
    for _ in range(3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        K.call("ndg_hmma_probe", ctypes.c_void_p(out.data_ptr()), blocks, iters, ctypes.c_void_p(s.cuda_stream))
        b.record()
        b.synchronize()
        best = max(best, K.load().ndg_hmma_probe_flops(blocks, iters) / (a.elapsed_time(b) * 1e-3) / 1e12)
    return best


def run_regime(a, regime, torch, ndg, D, K, dist, rank, world, dev, steps, warmup, measure_e2e):
    import numpy as np

    from paper_2405_20067_b200 import parallel as P
    if regime == "G":
        mix_np, s0 = D.gbuffer_mixture(a.n_dims, a.gaussians, seed=0), 0.005
    else:
        mix_np, s0 = D.synthetic_mixture(a.n_dims, a.gaussians, seed=0, children=a.children)
    # one global batch of a.batch * world queries; rank r keeps global tiles r, r + world, ... (weak
    # scaling: a.batch queries per GPU)
    q = D.synthetic_queries(a.n_dims, a.batch * world, seed=1, regime=regime, tile_size=a.tile)
    t = D.synthetic_targets(a.batch * world, seed=3)
    if world > 1:
        q, t, _ = P.shard_queries(q, t, a.tile, rank, world)
        q, t = np.ascontiguousarray(q), np.ascontiguousarray(t)
    mix = ndg.Mixture.from_arrays(a.n_dims, ndg.BRIGHTNESS, **mix_np, device=dev)
    hp = ndg.HotPath(a.n_dims, k=a.k, multiplier=3.0, tile_size=a.tile, projection_seed=2, device=dev)
    qd = torch.from_numpy(q).to(dev)
    td = torch.from_numpy(t).to(dev)
    grads = ndg.alloc_gradients(mix.G, mix.Gev, a.n_dims, dev)
    state = ndg.new_adam_state(mix)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    n_total = a.batch * world
    allreduce = P.make_allreduce() if world > 1 else None
    it = [0]
    # small, launch-bound steps (worst-case candidate list <= 2^24 entries, e.g. cfg1) replay one CUDA
    # graph of K1..K8 (engine.GraphedStep); qd / td are then its input buffers
    gs = None
    if a.graph == "on" or (a.graph == "auto" and ndg.GraphedStep.eligible(hp, mix, qd.shape[0])):
        hp.enable_kernel_timing(True)                   # capture the K4 / K5 / K7 event pairs too
        gs = ndg.GraphedStep(hp, mix, qd, td, n_total=n_total, grads=grads)
        hp.enable_kernel_timing(False)

    def step(queries, targets):
        it[0] += 1
        if gs is not None:
            if queries is not qd:
                qd.copy_(queries, non_blocking=True)
                td.copy_(targets, non_blocking=True)
            res = gs(allreduce=allreduce)
        else:
            res = hp.fwd_bwd(mix, queries, targets, n_total=n_total, grads=grads, allreduce=allreduce)
        ndg.adam_step(mix, grads, state, step=it[0])
        return res

    clocks = ClockSampler(int(os.environ.get("LOCAL_RANK", 0))) if rank == 0 else None
    for _ in range(warmup):
        res = step(qd, td)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    hp.enable_kernel_timing(True)
    launches0 = K.launch_count
    step_ms, kept, pairs = [], [], []
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    if clocks:
        clocks.begin()
    for _ in range(steps):
        flush.zero_()                                   # L2 flush, outside the timed interval
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        res = step(qd, td)
        e1.record()
        e1.synchronize()
        step_ms.append(e0.elapsed_time(e1))
        kept.append(res.kept_fraction)
        pairs.append(res.candidates.n_pairs_tiles * a.tile)
    torch.cuda.synchronize()
    if clocks:
        clocks.end()
    if world > 1:
        dist.barrier()
    launches = K.launch_count - launches0 + (gs.launches * steps if gs is not None else 0)
    clk = clocks.stop() if clocks else None
    fwd_ms = statistics.mean(hp.kernel_ms("forward"))
    bwd_ms = statistics.mean(hp.kernel_ms("backward"))
    cull_ms = statistics.mean(hp.kernel_ms("cull"))
    plan = hp.prefilter_plan()
    hp.enable_kernel_timing(False)
    total_ms = sum(step_ms)
    if world > 1:
        tt = torch.tensor([total_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        total_ms = float(tt)
    out = dict(total_ms=total_ms, ms_per_step=total_ms / steps, value=a.batch * world * steps / (total_ms * 1e-3),
               kept=statistics.mean(kept), pairs=statistics.mean(pairs), fwd_ms=fwd_ms, bwd_ms=bwd_ms,
               cull_ms=cull_ms, prefilter_ran=bool(plan and plan[1]),
               allreduce_bytes=int(grads.reduced().numel()) * 4,
               launches=launches, clocks=clk, loss=res.loss, sigma0=s0, fwd_impl=hp.last_forward_impl,
               bwd_impl=hp.last_backward_impl, graph=gs is not None and not gs.stale)

    # K4 alone, dense pass vs bucket pre-filter (same tile and projected bounds; identical masks)
    recs = hp.activate(mix)
    tb, pb = hp.tile_bounds(qd), hp.project(recs)
    ab = {}
    for mode in ("off", "on"):
        hk = ndg.HotPath(a.n_dims, k=a.k, multiplier=3.0, tile_size=a.tile, projection_seed=2, device=dev,
                         prefilter=mode)
        hk.enable_kernel_timing(True)
        for _ in range(3 + 10):
            hk.cull(tb, pb)
        torch.cuda.synchronize()
        ab["dense" if mode == "off" else "prefilter"] = statistics.median(hk.kernel_ms("cull")[3:])
    out["cull_ab"] = ab

    if measure_e2e:
        qh = torch.from_numpy(q).pin_memory()
        th = torch.from_numpy(t).pin_memory()
        e2e_ms = []
        for i in range(warmup + steps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            flush.zero_()
            e0.record()
            if gs is not None:                         # H2D straight into the graph's input buffers
                qd.copy_(qh, non_blocking=True)
                td.copy_(th, non_blocking=True)
                res = step(qd, td)
            else:
                qd2 = qh.to(dev, non_blocking=True)
                td2 = th.to(dev, non_blocking=True)
                res = step(qd2, td2)                   # fwd_bwd reads the loss back to the host
            e1.record()
            e1.synchronize()
            if i >= warmup:
                e2e_ms.append(e0.elapsed_time(e1))
        tot = sum(e2e_ms)
        if world > 1:
            tt = torch.tensor([tot], dtype=torch.float64, device=dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            tot = float(tt)
        out["e2e"] = dict(value=a.batch * world * steps / (tot * 1e-3), unit="queries/s",
                          h2d_bytes_per_step=int(q.nbytes + t.nbytes), d2h_bytes_per_step=8 + 32,
                          ms_per_step=tot / steps)
    return out, (mix_np, q, t, hp.ps.vectors)


def our_arm(a, rank, world):
    import torch
    dist = None
    # bind the rank's GPU before the process group, so NCCL's communicator and barriers use it
    local = int(os.environ.get("LOCAL_RANK", 0)) % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        # NDG_DIST_BACKEND=gloo only for plumbing checks with several ranks on one GPU (NCCL refuses that)
        dist.init_process_group(os.environ.get("NDG_DIST_BACKEND", "nccl"))
    dev = torch.device("cuda", local)
    import paper_2405_20067_b200 as ndg
    from paper_2405_20067_b200 import datasets as D
    from paper_2405_20067_b200 import kernels as K

    peak = fp32_peak(torch, K, dev)
    tpeak = tf32_peak(torch, K, dev)
    main, (mix_np, q, t, R) = run_regime(a, a.regime, torch, ndg, D, K, dist, rank, world, dev, a.steps, a.warmup,
                                         not a.no_e2e)
    secondary = None
    if not a.no_secondary:
        secondary = {}
        for other in [r for r in ("R", "C", "G") if r != a.regime]:
            s, _ = run_regime(a, other, torch, ndg, D, K, dist, rank, world, dev, max(3, a.steps // 2), 3, False)
            secondary[f"regime_{other}"] = dict(
                value=s["value"], unit="queries/s", ms_per_step=s["ms_per_step"], kept_fraction=s["kept"],
                pairs_per_step=s["pairs"], workload=workload_name(a, other),
                kernels_ms=dict(cull=s["cull_ms"], forward=s["fwd_ms"], backward=s["bwd_ms"]),
                cull_impl="bucket pre-filter (K4p)" if s["prefilter_ran"] else "dense (K4a)",
                fp32_frac_step=s["pairs"] * ndg.kept_pairs_flops(a.n_dims) / (s["ms_per_step"] * 1e-3) / 1e12 / peak)
            if "cull_ab" in s:
                secondary[f"regime_{other}"]["cull_ab_ms"] = s["cull_ab"]
    if rank != 0:
        if dist:
            dist.barrier()
            dist.destroy_process_group()
        return
    n = a.n_dims
    f_fwd, f_bwd = n * n + 3 * n + 8, 2 * n * n + 6 * n + 14
    pairs = main["pairs"]
    kern = {
        "forward": dict(ms=main["fwd_ms"], tflops=pairs * f_fwd / (main["fwd_ms"] * 1e-3) / 1e12),
        "backward": dict(ms=main["bwd_ms"], tflops=pairs * f_bwd / (main["bwd_ms"] * 1e-3) / 1e12),
    }
    for v in kern.values():
        v["frac_of_measured_fp32"] = v["tflops"] / peak
        v["share_of_step"] = v["ms"] / main["ms_per_step"]
    if main["fwd_impl"] == "tc":
        # the tensor-core K5 does not run its algorithmic flops on the FP32 pipe: keep its FP32-equivalent
        # rate under an explicit name and report it against the tensor peak below
        kern["forward"]["fp32_equivalent_tflops"] = kern["forward"].pop("tflops")
        kern["forward"].pop("frac_of_measured_fp32")
    kern_cull = dict(ms=main["cull_ms"], share_of_step=main["cull_ms"] / main["ms_per_step"],
                     impl="bucket pre-filter (K4p)" if main["prefilter_ran"] else "dense (K4a)",
                     ab_ms=main["cull_ab"])
    if main["fwd_impl"] == "tc":
        # tensor-core forward: the z-GEMM is 2 * (N+1) * N flops per pair (algorithmic); 3xTF32 issues it three
        # times (hi.hi + hi.lo + lo.hi) for float32 accuracy
        alg_f = 2 * (n + 1) * n
        t_alg = pairs * alg_f / (main["fwd_ms"] * 1e-3) / 1e12
        kern["forward"].update(impl="tcgen05 kind::tf32 (3xTF32)", tensor_peak_measured=tpeak,
                               tensor_flops_per_pair_algorithmic=alg_f, tensor_tflops_algorithmic=t_alg,
                               frac_of_measured_tf32_algorithmic=t_alg / tpeak,
                               tensor_flops_per_pair_issued=3 * alg_f, tensor_tflops_issued=3 * t_alg,
                               frac_of_measured_tf32_issued=3 * t_alg / tpeak)
    if main["bwd_impl"] == "mma":
        # warp-MMA K7 (f16 form): per Gaussian and 16 queries, 10 m16n8k16 MMAs issued (z-GEMM: 2 n-tiles x 3
        # products; S-GEMM: 2 column blocks x 2) = 2560 tensor flops per pair on the padded 16-dim block
        hpeak = hmma_peak(torch, K, dev)
        mm_f = 10 * 2 * 16 * 8 * 16 // 16
        m_tf = pairs * mm_f / (main["bwd_ms"] * 1e-3) / 1e12
        kern["backward"].update(impl="mma.sync m16n8k16 f16 (hi/lo split, 3 products)", tensor_tflops=m_tf, tensor_peak_measured=hpeak,
                                frac_of_measured_hmma=m_tf / hpeak, tensor_flops_per_pair=mm_f)
    dom = max(kern, key=lambda k: kern[k]["ms"])
    traffic = None
    try:
        tr = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json")))
        traffic = tr.get(f"{dom}:N{n}:G{a.gaussians}:B{a.batch}:{a.regime}")
    except (OSError, ValueError):
        pass
    step_tflops = pairs * ndg.kept_pairs_flops(n) / (main["ms_per_step"] * 1e-3) / 1e12
    if dom == "forward" and main["fwd_impl"] == "tc":
        f = kern["forward"]
        roof = dict(bound="tensor", kernel=dom, achieved=f["tensor_tflops_algorithmic"], peak=tpeak, unit="TFLOP/s",
                    frac=f["frac_of_measured_tf32_algorithmic"], traffic=traffic,
                    peak_source="measured tcgen05 kind::tf32 probe on this GPU",
                    bound_note="the dominant kernel is the tcgen05 K5: achieved counts the algorithmic z-GEMM "
                               "(2(N+1)N flops per pair) once; 3xTF32 issues it three times (kernels.forward)",
                    flops_per_pair=dict(forward=f_fwd, backward=f_bwd, step=ndg.kept_pairs_flops(n)),
                    step_fp32_equivalent_tflops=step_tflops)
    else:
        roof = (dict(bound="tensor", kernel=dom, achieved=kern[dom]["tensor_tflops"],
             peak=kern[dom]["tensor_peak_measured"], unit="TFLOP/s",
             frac=kern[dom]["frac_of_measured_hmma"], traffic=traffic,
             peak_source="measured mma.sync m16n8k16 f16 probe (ndg_hmma_probe) on this GPU: the legacy "
                         "warp-level tensor path this kernel issues, not the tcgen05 peak",
             bound_note="the dominant kernel is the warp-MMA K7 (N >= 14): achieved counts its padded "
                        "split-f16 MMA flops (2560 per pair); the kernel is issue-bound (the per-query scalars "
                        "and operand splits between the MMAs), see DESIGN.md; its FP32-equivalent rate is in "
                        "kernels.backward",
             flops_per_pair=dict(forward=f_fwd, backward=f_bwd, step=ndg.kept_pairs_flops(n),
                                 backward_tensor=kern[dom]["tensor_flops_per_pair"]),
             step_fp32_equivalent_tflops=step_tflops)
        if dom == "backward" and main["bwd_impl"] == "mma" else
        dict(bound="fp32", kernel=dom, achieved=kern[dom]["tflops"], peak=peak, unit="TFLOP/s",
            frac=kern[dom]["tflops"] / peak, traffic=traffic,
            peak_source="measured FFMA probe (ndg_fp32_probe) on this GPU; MEASURED_PEAKS.json has no "
                        "FP32 entry",
            bound_note="the dominant kernel (K7 backward) runs on the FP32 SIMT pipe: its DRAM traffic "
                       "(`traffic`, ncu, ~2x its algorithmic bytes) is <1% of the HBM roof and it issues "
                       "no tensor-core work, so neither 'hbm' nor 'tensor' applies; the K5 forward's "
                       "tensor roofline is in kernels.forward",
            peak_nominal=NOMINAL_FP32_TFLOPS, frac_of_nominal=kern[dom]["tflops"] / NOMINAL_FP32_TFLOPS,
            flops_per_pair=dict(forward=f_fwd, backward=f_bwd, step=ndg.kept_pairs_flops(n)),
            step_fp32_equivalent_tflops=step_tflops,
            step_note="the step's rate counts K5's tensor-core z-GEMM as FP32-equivalent flops; the "
                      "roofline figure of the step is `frac` (its dominant kernel, K7)"))
    line = dict(
        metric=METRIC, value=main["value"], unit="queries/s", n_gpus=world, steps=a.steps, warmup=a.warmup,
        ms_per_step=main["ms_per_step"], higher_is_better=True, scaling="weak", vs_baseline=None, dtype="f32",
        data="synthetic (seeded NumPy PCG64 mixture / queries / targets of the named shape)",
        config=dict(workload=workload_name(a, a.regime), n_dims=n, gaussians=a.gaussians,
                    evaluated_gaussians=a.gaussians * (2 if a.children else 1), batch_per_gpu=a.batch,
                    global_batch=a.batch * world, tile=a.tile, k=a.k, multiplier=3.0, regime=a.regime,
                    kept_fraction=main["kept"], pairs_per_step=pairs, sigma0=main["sigma0"],
                    allreduce_payload_bytes_per_step=main["allreduce_bytes"],
                    step_launch=("one CUDA-graph replay of K1..K8 per step (engine.GraphedStep; worst-case-sized "
                                 "candidate list, no mid-step read-back) + K9 Adam" if main["graph"] else
                                 "eager: one C-ABI launch per stage, one mid-step read-back sizing the candidate list"),
                    l2="flushed before every timed step (256 MiB write, outside the timed interval)",
                    parallelism=f"dp{world} (one global batch of {a.batch * world} queries, strided tiles per "
                                f"rank, mixture replicated, 1 {(dist.get_backend() if dist else 'nccl').upper()} "
                                f"allreduce/step of the flat gradient buffer)"),
        roofline=roof,
        kernels=dict(kern, cull=kern_cull), gpu_launches=main["launches"], clocks=main["clocks"], loss=main["loss"],
    )
    if "e2e" in main:
        line["e2e"] = main["e2e"]
    if secondary:
        line["secondary"] = secondary
    if world == 1 and not a.no_cpu_baseline:
        info = cpu_sample(a, mix_np, q, t, R, a.cpu_seconds)
        line["cpu_baseline"] = dict(value=info["value"], unit="queries/s", cores=info["threads"],
                                    kind="port", sample=info["sample"], cpu=_cpu_model(),
                                    sample_seconds=info["step_s"], utilization=info["utilization"])
    print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


def main():
    a = parse()
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    if a.impl == "reference":
        reference_arm(a, rank, world)
    else:
        our_arm(a, rank, world)


if __name__ == "__main__":
    main()
