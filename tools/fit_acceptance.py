"""The SPEC's fit-quality acceptance runs on one GPU, through the product trainer:

  recovery  fit a hidden 8-component gmm_oracle_target in N=6 starting from 32 components for 10k
            iterations; held-out relative L2 must fall below 1e-2.
  shading   fit shading_toy_target in N=10 with the default config for 20k iterations; held-out PSNR
            must exceed 30 dB, and the refinement phases should raise the component count while
            the best-so-far validation loss falls.

Prints one JSON object with the curves (held-out metric every `--every` iterations, component counts,
refinement events) and the pass/fail of each criterion.
"""
import argparse, json, math, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2405_20067_b200 import datasets as D
from paper_2405_20067_b200 import trainer as T
from paper_2405_20067_b200.engine import HotPath

ap = argparse.ArgumentParser()
ap.add_argument("--which", choices=["recovery", "shading", "both"], default="both")
ap.add_argument("--every", type=int, default=1000)
ap.add_argument("--recovery-iters", type=int, default=10000)
ap.add_argument("--shading-iters", type=int, default=20000)
a = ap.parse_args()
torch.cuda.set_device(0)
dev = torch.device("cuda", 0)


def held_out(mix, target, n, count=1 << 14):
    q, tg = D.sample_batch(target, n, count, 256, D.QuerySampler(12345), dev)
    pred = HotPath(n, device=dev).evaluate(mix, q, cull=True)
    rel = float(torch.linalg.norm(pred - tg) / torch.linalg.norm(tg))
    mse = float(torch.mean((pred - tg) ** 2))
    peak = float(tg.max())
    return rel, 10.0 * math.log10(max(peak, 1e-30) ** 2 / max(mse, 1e-30))


def run(name, cfg, target, n):
    curve = []

    def cb(tr, row):
        if (row.iteration + 1) % a.every == 0:
            rel, psnr = held_out(tr.mix, target, n)
            curve.append(dict(iteration=row.iteration + 1, held_out_rel_l2=rel, psnr_db=psnr,
                              n_components=row.n_components, loss=row.loss))
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = T.train(cfg, target, n, callback=cb)
    torch.cuda.synchronize()
    rel, psnr = held_out(res.mixture, target, n)
    return dict(seconds=time.perf_counter() - t0, final_held_out_rel_l2=rel, final_psnr_db=psnr,
                curve=curve, events=res.events)


out = {}
if a.which in ("recovery", "both"):
    tgt = D.GmmOracleTarget(0, 6, 8, device=dev)
    cfg = T.TrainConfig(iterations=a.recovery_iters, n_components=32, seed=0)
    r = run("recovery", cfg, tgt, 6)
    r["pass"] = r["final_held_out_rel_l2"] < 1e-2
    out["recovery_N6_8hidden_32init"] = r
if a.which in ("shading", "both"):
    tgt = D.ShadingToyTarget(0, 10)
    cfg = T.TrainConfig(iterations=a.shading_iters, seed=0)
    r = run("shading", cfg, tgt, 10)
    comps = [c["n_components"] for c in r["curve"]]
    best, best_after_phase = float("inf"), []
    for c in r["curve"]:
        best = min(best, c["held_out_rel_l2"])
        best_after_phase.append(best)
    r["pass_psnr"] = r["final_psnr_db"] > 30.0
    r["components_grow"] = comps == sorted(comps) and comps[-1] > comps[0]
    r["best_loss_falls"] = best_after_phase[-1] < best_after_phase[0]
    out["shading_N10_default"] = r
print(json.dumps(out))
