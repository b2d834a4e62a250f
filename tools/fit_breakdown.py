"""Where a fit iteration's time goes (cfg3 shape by default): wall clock per iteration against the
CUDA-event time of the culling (K4), forward (K5) and backward (K7) kernels. Tuning aid."""
import argparse, json, os, statistics, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2405_20067_b200 import datasets as D
from paper_2405_20067_b200 import trainer as T

ap = argparse.ArgumentParser()
ap.add_argument("--iterations", type=int, default=200)
ap.add_argument("--batch", type=int, default=1 << 16)
ap.add_argument("--components", type=int, default=4096)
ap.add_argument("--n-dims", type=int, default=10)
ap.add_argument("--children", action="store_true")
a = ap.parse_args()
torch.cuda.set_device(0)
tgt = D.ShadingToyTarget(0, a.n_dims)
cfg = T.TrainConfig(iterations=a.iterations, phase_length=10 ** 9, n_components=a.components, batch_size=a.batch, seed=0)
tr = T.Trainer(cfg, tgt, a.n_dims)
tr.hp.enable_kernel_timing(True)          # before the first iteration: the captured step records them too
if a.children:
    tr.spawn_step()
for _ in range(20):
    tr.iteration()
torch.cuda.synchronize()
tr.hp.events = {k: [] for k in tr.hp.events}
t0 = time.perf_counter()
for _ in range(a.iterations):
    tr.iteration()
torch.cuda.synchronize()
wall = (time.perf_counter() - t0) * 1e3 / a.iterations
k = {n: statistics.mean(tr.hp.kernel_ms(n)) for n in ("cull", "forward", "backward")}
print(json.dumps(dict(config=vars(a), Gev=tr.mix.Gev, wall_ms_per_iter=wall, kernels_ms=k,
                      kernel_share=sum(k.values()) / wall)))
