"""cfg3 (BASELINE.json configs[2]): 10-D fit loop with density control over 1k steps, culling on vs
off. Reports steps/s, final loss, held-out rel-L2 and the refinement events for both runs."""
import argparse, json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2405_20067_b200 import datasets as D
from paper_2405_20067_b200 import trainer as T

ap = argparse.ArgumentParser()
ap.add_argument("--iterations", type=int, default=1000)
ap.add_argument("--batch", type=int, default=1 << 16)
ap.add_argument("--components", type=int, default=4096)
ap.add_argument("--target", default="shading")
a = ap.parse_args()
torch.cuda.set_device(0)
out = {}
for cull in (True, False):
    tgt = D.ShadingToyTarget(0, 10) if a.target == "shading" else D.GmmOracleTarget(0, 10, 64)
    cfg = T.TrainConfig(iterations=a.iterations, phase_length=300, n_components=a.components, batch_size=a.batch,
                        cull=cull, seed=0)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = T.train(cfg, tgt, 10)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    losses = [m.loss for m in res.metrics]
    out["cull_on" if cull else "cull_off"] = dict(
        steps_per_s=a.iterations / dt, seconds=dt, first_loss=losses[0], final_loss=sum(losses[-20:]) / 20,
        held_out_rel_l2=T.held_out_rel_l2(res.mixture, tgt, 10), events=res.events,
        mean_culled_fraction=sum(m.culled_fraction for m in res.metrics) / len(res.metrics),
        loss_curve=[round(l, 5) for l in losses[::50]])
print(json.dumps(dict(config=vars(a), **out)))
