"""K4 dense cull timing on one workload (select the library with NDG_LIB). Tuning aid."""
import argparse, json, os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2405_20067_b200 as ndg
from paper_2405_20067_b200 import datasets as D

ap = argparse.ArgumentParser()
ap.add_argument("--n-dims", type=int, default=10)
ap.add_argument("--gaussians", type=int, default=100_000)
ap.add_argument("--batch", type=int, default=1 << 20)
ap.add_argument("--reps", type=int, default=20)
a = ap.parse_args()
torch.cuda.set_device(0)
mix_np, _ = D.synthetic_mixture(a.n_dims, a.gaussians, seed=0)
mix = ndg.Mixture.from_arrays(a.n_dims, 0, **mix_np)
q = torch.from_numpy(D.synthetic_queries(a.n_dims, a.batch, seed=1)).cuda()
hp = ndg.HotPath(a.n_dims, projection_seed=2, prefilter="off")
recs = hp.activate(mix)
tb, pb = hp.tile_bounds(q), hp.project(recs)
hp.enable_kernel_timing(True)
for _ in range(a.reps):
    hp.cull(tb, pb)
torch.cuda.synchronize()
ms = hp.kernel_ms("cull")[3:]
print(json.dumps(dict(lib=os.path.basename(os.environ.get("NDG_LIB", "libndg.so")), n=a.n_dims, G=a.gaussians,
                      B=a.batch, cull_ms=statistics.median(ms))))
