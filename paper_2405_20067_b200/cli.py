"""Command-line surface of the reference, hot-path commands only:

    ndgauss fit  --config PATH --out DIR [--resume CKPT]
    ndgauss eval --ckpt PATH (--queries PATH | --grid SPEC) --out DIR [--ref PATH] [--no-cull]
    ndgauss bench-cull --config PATH --out CSV
    ndgauss gradcheck [--seed S]

fit writes metrics.csv (iteration,loss,n_components,culled_fraction,ms_per_iter) and a checkpoint
every phase and at the end; exit 0 on completion, 2 on a config error, 3 on TrainingAborted
(SPEC.md:514-515). eval writes the predictions as an NDGT file (and PFM/PPM for a 2-D grid slice)
and reports rel-L2 / PSNR against --ref. --grid SPEC = "d0,d1:W,H[:v]" evaluates the
2-D slice over dims d0, d1 at W x H points with the other dims fixed at v (default 0.5).
bench-cull (the paper's culling ablation) sweeps k x multiplier x tile size over a
seeded synthetic workload ([bench] config section) and writes one CSV row per point: cull fraction,
false culls = (tile, Gaussian) pairs brute_force_active at the 3-sigma level epsilon = exp(-4.5)
(float64, on the device) that the cull dropped, max |pred_culled - pred_brute|, and
the wall-clock of culled vs brute-force evaluation. Multiplier >= 3 rows have no false culls by
Cauchy-Schwarz; multiplier 1 rows show the paper's artifact regime. (The culled tail still moves pred
by up to exp(-m^2/2) * sum |a| of the dropped Gaussians, so max_abs_err is reported, not bounded by
1e-6: DESIGN.md §5.)
gradcheck compares the analytic gradients with central finite differences of a
float64 evaluator (paper_2405_20067_b200/gradcheck.py); exit 0 iff every coordinate's relative error
(1e-6 absolute floor) is < 1e-4. --fp32 checks the float32 product kernels instead,
under the relaxed block-relative 1e-4 rule, and says so in its output.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import sys

import numpy as np

from . import formats as nio
from .errors import ConfigError, FileFormatError, NdgError, TrainingAborted


def _target(cfg: dict, n_dims: int, device):
    from . import datasets as D
    data = cfg.get("data", {})
    kind = data.get("target", "shading")
    if kind == "shading":
        return D.ShadingToyTarget(int(data.get("target_seed", 0)), n_dims)
    if kind == "gmm":
        return D.GmmOracleTarget(int(data.get("target_seed", 0)), n_dims, int(data.get("target_components", 8)),
                                 device=device)
    if kind == "file":                       # an NDGT tensor file
        if "path" not in data:
            raise ConfigError("data.target = file needs data.path", field="path")
        ds = D.FileDataset.from_ndgt(str(data["path"]), seed=int(data.get("target_seed", 0)),
                                     perturb_sigma=float(data.get("perturb_sigma", 0.0)), device=device)
        if ds.n_dims != n_dims:
            raise ConfigError(f"data.n_dims = {n_dims} but {data['path']} holds {ds.n_dims}-D queries",
                              field="n_dims")
        return ds
    raise ConfigError(f"unknown target {kind!r}", field="target")


def _state_of(tr, cfg_raw):
    m = tr.full_mixture()            # the ordered mixture: frozen rows (compacted out of the loop) in place
    st, low = tr.full_state()
    return dict(n_dims=m.n_dims, amp_mode=m.amp_mode, iteration=tr.step_no, adam_step=tr.step_no,
                config=cfg_raw, dataset=cfg_raw.get("data", {}),
                rng=tr.rng_state(),
                params=m.params.cpu().numpy(), child=m.child.cpu().numpy(), flags=m.flags.cpu().numpy(),
                m1p=st["m1p"].cpu().numpy(), m2p=st["m2p"].cpu().numpy(),
                m1c=st["m1c"].cpu().numpy(), m2c=st["m2c"].cpu().numpy(),
                low_count=low.cpu().numpy())


def _dist_setup():
    """torchrun: one process per GPU (RANK / LOCAL_RANK / WORLD_SIZE from the environment), NCCL
    process group (NDG_DIST_BACKEND=gloo for plumbing checks); returns (rank, world, allreduce)."""
    import torch
    world = int(os.environ.get("WORLD_SIZE", 1))
    if world <= 1:
        return 0, 1, None
    import torch.distributed as dist

    from .parallel import make_allreduce
    local = int(os.environ.get("LOCAL_RANK", 0)) % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    if not dist.is_initialized():
        dist.init_process_group(os.environ.get("NDG_DIST_BACKEND", "nccl"))
    return dist.get_rank(), world, make_allreduce()


def cmd_fit(args) -> int:
    """SPEC.md:511-519. Under torchrun every rank runs this: the mixture and optimizer state are
    replicated, each rank evaluates its strided tiles of the one global batch (datasets.sample_batch)
    and the step's gradients are summed by ONE allreduce; rank 0 writes
    metrics.csv and the checkpoints. --resume continues bit-identically: the checkpoint
    carries the torch sampling-generator state and the full numpy PCG64 state, and metrics.csv is
    appended to."""
    import torch
    from .gmm import FLAG_CHILD, FLAG_FROZEN, Mixture
    from .trainer import Trainer
    try:
        cfg_raw = nio.parse_config(open(args.config).read())
        cfg = nio.train_config_from(cfg_raw)
    except ConfigError as e:
        print(f"config error: {e}", file=sys.stderr)
        return 2
    rank, world, allreduce = _dist_setup()
    if cfg.batch_size % cfg.tile_size or cfg.batch_size // cfg.tile_size < world:
        print(f"config error: batch_size must be a multiple of tile_size with at least one tile per rank "
              f"({world} ranks)", file=sys.stderr)
        return 2
    n = int(cfg_raw.get("data", {}).get("n_dims", 10))
    if rank == 0:
        os.makedirs(args.out, exist_ok=True)
    dev = torch.device("cuda", torch.cuda.current_device())
    target = _target(cfg_raw, n, dev)
    mix = None
    st = None
    if args.resume:
        st = nio.load_checkpoint(args.resume)
        fl = st["flags"]
        mix = Mixture.from_arrays(st["n_dims"], st["amp_mode"], st["params"], st["child"], (fl & FLAG_CHILD) != 0,
                                  (fl & FLAG_FROZEN) != 0, device=dev)
    tr = Trainer(cfg, target, n, mixture=mix, device=dev, allreduce=allreduce, rank=rank, world=world)
    if st is not None:
        tr.resume(st)
    metrics = None
    if rank == 0:
        path = os.path.join(args.out, "metrics.csv")
        fresh = st is None or not os.path.exists(path)
        metrics = open(path, "w" if fresh else "a")
        if fresh:
            metrics.write("iteration,loss,n_components,culled_fraction,ms_per_iter\n")
    ckpt = os.path.join(args.out, "checkpoint.ndgc")

    def save():
        if rank == 0:
            nio.save_checkpoint(ckpt, _state_of(tr, cfg_raw))

    try:
        start = tr.step_no
        for it in range(start, cfg.iterations):
            row = tr.iteration()
            if metrics:
                metrics.write(f"{row.iteration},{row.loss:.9g},{row.n_components},{row.culled_fraction:.6f},"
                              f"{row.ms_per_iter:.3f}\n")
            if it == start and world > 1 and rank == 0:
                print(f"data-parallel fit: {world} ranks, allreduce payload {tr.last_allreduce_bytes} bytes/step",
                      file=sys.stderr)
            if (it + 1) % cfg.phase_length == 0:
                if (it + 1) // cfg.phase_length >= cfg.warmup_phases:
                    ev = tr.phase_event()
                    if rank == 0:       # refinement events with the phase's density statistics
                        with open(os.path.join(args.out, "events.jsonl"), "a") as fe:
                            fe.write(json.dumps(ev, sort_keys=True) + "\n")
                    if world > 1 and rank == 0:
                        print(f"phase event at {it + 1}: {tr.mix.G} components, children live "
                              f"{tr.mix.children_live}", file=sys.stderr)
                save()
    except TrainingAborted as e:
        save()
        print(f"training aborted: {e}", file=sys.stderr)
        return 3
    finally:
        if metrics:
            metrics.close()
    save()
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
    return 0


def _grid_queries(spec: str, n: int):
    parts = spec.split(":")
    d0, d1 = (int(x) for x in parts[0].split(","))
    w, h = (int(x) for x in parts[1].split(","))
    fixed = float(parts[2]) if len(parts) > 2 else 0.5
    ys, xs = np.meshgrid((np.arange(h) + 0.5) / h, (np.arange(w) + 0.5) / w, indexing="ij")
    q = np.full((h * w, n), fixed, np.float32)
    q[:, d0] = xs.ravel()
    q[:, d1] = ys.ravel()
    return q, (h, w)


def cmd_eval(args) -> int:
    import torch
    from .engine import HotPath
    from .gmm import FLAG_CHILD, FLAG_FROZEN, Mixture
    try:
        st = nio.load_checkpoint(args.ckpt)
    except (OSError, FileFormatError) as e:
        print(f"cannot read checkpoint: {e}", file=sys.stderr)
        return 2
    n = st["n_dims"]
    dev = torch.device("cuda", torch.cuda.current_device())
    fl = st["flags"]
    # inference mixture: children are not evaluated
    mix = Mixture.from_arrays(n, st["amp_mode"], st["params"], st["child"], np.zeros_like(fl, bool),
                              (fl & FLAG_FROZEN) != 0, device=dev)
    shape = None
    if args.grid:
        q, shape = _grid_queries(args.grid, n)
    else:
        q, _, _ = nio.read_ndgt(args.queries)
        if q.shape[1] != n:
            print("dimension mismatch between checkpoint and queries", file=sys.stderr)
            return 2
    os.makedirs(args.out, exist_ok=True)
    B = q.shape[0]
    tile = int(st["config"].get("culling", {}).get("tile_size", 256))
    pad = (-B) % tile
    qq = np.concatenate([q, np.repeat(q[-1:], pad, 0)]) if (pad and B) else q
    pred = np.zeros((0, 3), np.float32)
    if B:
        hp = HotPath(n, tile_size=tile, device=dev)
        pred = hp.evaluate(mix, torch.from_numpy(np.ascontiguousarray(qq)).to(dev), cull=not args.no_cull)
        pred = pred.cpu().numpy()[:B]
    nio.write_ndgt(os.path.join(args.out, "pred.ndgt"), q, pred)
    if shape is not None:
        img = pred.reshape(shape[0], shape[1], 3)
        nio.write_pfm(os.path.join(args.out, "slice.pfm"), img)
        nio.write_ppm(os.path.join(args.out, "slice.ppm"), img)
    if args.ref and B:
        _, ref, _ = nio.read_ndgt(args.ref)
        err = float(np.linalg.norm(pred - ref) / max(np.linalg.norm(ref), 1e-30))
        mse = float(np.mean((pred - ref) ** 2))
        psnr = 10.0 * math.log10(max(float(ref.max()), 1e-30) ** 2 / max(mse, 1e-30))
        print(f"rel_l2={err:.6g} psnr={psnr:.3f}")
    return 0


_POPCOUNT = None


def _popcount(words) -> int:
    """Number of set bits in an int32 tensor (byte lookup table)."""
    import torch
    global _POPCOUNT
    if _POPCOUNT is None or _POPCOUNT.device != words.device:
        _POPCOUNT = torch.tensor([bin(i).count("1") for i in range(256)], dtype=torch.int64, device=words.device)
    return int(_POPCOUNT[words.contiguous().view(torch.uint8).long()].sum())


def cmd_bench_cull(args) -> int:
    import time
    import torch
    from . import datasets as D
    from .engine import HotPath
    from .gmm import Mixture
    try:
        cfg = nio.parse_config(open(args.config).read())
    except ConfigError as e:
        print(f"config error: {e}", file=sys.stderr)
        return 2
    b = cfg.get("bench", {})
    aslist = lambda v, d: [v] if isinstance(v, (int, float)) else (list(v) if v is not None else d)  # noqa: E731
    n = int(cfg.get("data", {}).get("n_dims", 10))
    G, B = int(b.get("gaussians", 10000)), int(b.get("queries", 1 << 16))
    regime, seed, reps = str(b.get("regime", "C")), int(b.get("seed", 0)), int(b.get("reps", 3))
    eps = float(b.get("epsilon", math.exp(-4.5)))
    ks = [int(x) for x in aslist(b.get("k_list"), [4, 8, 16, 32])]
    mults = [float(x) for x in aslist(b.get("multiplier_list"), [1, 2, 3, 4])]
    tiles = [int(x) for x in aslist(b.get("tile_list"), [64, 256])]
    dev = torch.device("cuda", torch.cuda.current_device())
    if regime == "G":      # G-buffer-like inference workload: mixture seeded on the query manifold
        mix_np = D.gbuffer_mixture(n, G, seed=seed, sigma0=float(b.get("sigma0", 0.005)))
    else:
        mix_np, _ = D.synthetic_mixture(n, G, seed=seed, sigma0=b.get("sigma0"))
    mix = Mixture.from_arrays(n, 0, **mix_np, device=dev)
    qd = torch.from_numpy(D.synthetic_queries(n, B, seed=seed + 1, regime=regime)).to(dev)

    def timed(fn):
        fn()                                   # warm-up (also builds the per-N kernel attributes)
        ts = []
        for _ in range(reps):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            out = fn()
            torch.cuda.synchronize()
            ts.append(time.perf_counter() - t0)
        return out, 1e3 * sorted(ts)[len(ts) // 2]

    rows = []
    for tile in tiles:
        if B % tile:
            print(f"queries ({B}) must be a multiple of every tile size ({tile})", file=sys.stderr)
            return 2
        hb = HotPath(n, tile_size=tile, device=dev)
        pred_ref, ms_brute = timed(lambda: hb.evaluate(mix, qd, cull=False))
        recs = hb.activate(mix)
        T = B // tile
        live_pairs = T * int((recs.eflags & 1).sum())
        active, acount = hb.brute_force_active(qd, recs, eps)
        n_active = int(acount.sum())
        for mult in mults:
            for k in ks:
                hp = HotPath(n, k=k, multiplier=mult, tile_size=tile, projection_seed=seed + 2, device=dev)
                pred, ms_cull = timed(lambda: hp.evaluate(mix, qd, cull=True))
                cl = hp.cull(hp.tile_bounds(qd), hp.project(recs))
                false_culls = _popcount(active & ~cl.mask)
                err = float((pred - pred_ref).abs().max()) if B else 0.0
                rows.append(dict(k=k, multiplier=mult, tile_size=tile, cull_fraction=1.0 - cl.n_pairs_tiles / max(1, live_pairs),
                                 kept_pairs=cl.n_pairs_tiles * tile, active_pairs=n_active * tile, false_culls=false_culls,
                                 max_abs_err=err, ms_culled=ms_cull, ms_brute=ms_brute, speedup=ms_brute / ms_cull))
    cols = list(rows[0].keys()) if rows else []
    with open(args.out, "w") as f:
        f.write(",".join(cols) + "\n")
        for r in rows:
            f.write(",".join(f"{r[c]:.6g}" if isinstance(r[c], float) else str(r[c]) for c in cols) + "\n")
    return 0


def cmd_gradcheck(args) -> int:
    from . import gradcheck
    return 0 if gradcheck.run(seed=args.seed, per_n=args.per_n, analytic="fp32" if args.fp32 else "f64") else 1


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="ndgauss")
    sub = ap.add_subparsers(dest="cmd", required=True)
    f = sub.add_parser("fit")
    f.add_argument("--config", required=True)
    f.add_argument("--out", required=True)
    f.add_argument("--resume")
    e = sub.add_parser("eval")
    e.add_argument("--ckpt", required=True)
    g = e.add_mutually_exclusive_group(required=True)
    g.add_argument("--queries")
    g.add_argument("--grid")
    e.add_argument("--out", required=True)
    e.add_argument("--ref")
    e.add_argument("--no-cull", action="store_true")
    bc = sub.add_parser("bench-cull")
    bc.add_argument("--config", required=True)
    bc.add_argument("--out", required=True)
    gc = sub.add_parser("gradcheck")
    gc.add_argument("--seed", type=int, default=0)
    gc.add_argument("--per-n", type=int, default=100, help="random mixtures per (N, amplitude mode)")
    gc.add_argument("--fp32", action="store_true",
                    help="check the float32 product kernels under the relaxed block-relative rule instead of "
                         "SPEC.md:572's per-coordinate rule on the float64 analytic path")
    args = ap.parse_args(argv)
    try:
        return {"fit": cmd_fit, "eval": cmd_eval, "bench-cull": cmd_bench_cull,
                "gradcheck": cmd_gradcheck}[args.cmd](args)
    except NdgError as err:
        print(f"error: {err}", file=sys.stderr)
        return 1


if __name__ == "__main__":
    sys.exit(main())
