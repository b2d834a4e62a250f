"""Kernel A/B micro-benchmark: times K5 (forward) and K7 (backward) alone at a bench workload for
one libndg build (select with NDG_LIB=path). Prints one JSON line. Tuning aid, not the bench."""
import argparse, json, os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2405_20067_b200 as ndg
from paper_2405_20067_b200 import datasets as D

ap = argparse.ArgumentParser()
ap.add_argument("--n-dims", type=int, default=10)
ap.add_argument("--gaussians", type=int, default=100_000)
ap.add_argument("--batch", type=int, default=1 << 20)
ap.add_argument("--regime", default="R")
ap.add_argument("--iters", type=int, default=3)
ap.add_argument("--children", action="store_true")
a = ap.parse_args()
torch.cuda.set_device(0)
mix_np, _ = D.synthetic_mixture(a.n_dims, a.gaussians, seed=0, children=a.children)
q = D.synthetic_queries(a.n_dims, a.batch, seed=1, regime=a.regime)
t = D.synthetic_targets(a.batch, seed=3)
mix = ndg.Mixture.from_arrays(a.n_dims, 0, **mix_np)
hp = ndg.HotPath(a.n_dims, projection_seed=2)
qd, td = torch.from_numpy(q).cuda(), torch.from_numpy(t).cuda()
res = hp.fwd_bwd(mix, qd, td, check=False)
hp.enable_kernel_timing(True)
for _ in range(a.iters):
    res = hp.fwd_bwd(mix, qd, td, check=False)
torch.cuda.synchronize()
n = a.n_dims
pairs = res.candidates.n_pairs_tiles * 256
f = statistics.median(hp.kernel_ms("forward")); b = statistics.median(hp.kernel_ms("backward"))
g = res.grads.flat.double()
print(json.dumps(dict(lib=os.path.basename(os.environ.get("NDG_LIB", "libndg.so")), fwd=hp.last_forward_impl, bwd=hp.last_backward_impl, regime=a.regime, n=n,
      fwd_ms=f, bwd_ms=b, fwd_tflops=pairs * (n*n+3*n+8) / f / 1e9, bwd_tflops=pairs * (2*n*n+6*n+14) / b / 1e9,
      kept=res.kept_fraction, loss=res.loss, grad_checksum=float(g.abs().sum()), pred_sum=float(res.pred.double().sum()))))
