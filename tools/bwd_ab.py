"""A/B of two K7 implementations on one workload: block-relative gradient differences between
backward=<--other> ("mma") and backward="fp32" (same forward), plus K7 timings.
Tuning aid, not a test."""
import argparse, json, os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2405_20067_b200 as ndg
from paper_2405_20067_b200 import datasets as D
from paper_2405_20067_b200.gmm import n_chol

ap = argparse.ArgumentParser()
ap.add_argument("--n-dims", type=int, default=10)
ap.add_argument("--gaussians", type=int, default=20000)
ap.add_argument("--batch", type=int, default=1 << 16)
ap.add_argument("--regime", default="R")
ap.add_argument("--sigma0", type=float, default=None)
ap.add_argument("--iters", type=int, default=2)
ap.add_argument("--other", choices=["mma"], default="mma")
a = ap.parse_args()
torch.cuda.set_device(0)
kw = {} if a.sigma0 is None else dict(sigma0=a.sigma0)
mix_np, _ = D.synthetic_mixture(a.n_dims, a.gaussians, seed=0, **kw)
q = D.synthetic_queries(a.n_dims, a.batch, seed=1, regime=a.regime)
t = D.synthetic_targets(a.batch, seed=3)
mix = ndg.Mixture.from_arrays(a.n_dims, 0, **mix_np)
qd, td = torch.from_numpy(q).cuda(), torch.from_numpy(t).cuda()
out = {}
for impl in ("fp32", a.other):
    hp = ndg.HotPath(a.n_dims, projection_seed=2, backward=impl)
    res = hp.fwd_bwd(mix, qd, td, check=False)
    hp.enable_kernel_timing(True)
    for _ in range(a.iters):
        res = hp.fwd_bwd(mix, qd, td, check=False)
    torch.cuda.synchronize()
    out[impl] = dict(ms=statistics.median(hp.kernel_ms("backward")), g=res.grads.params.double().cpu().numpy(),
                     st=res.grads.stats.double().cpu().numpy(), impl=hp.backward_impl)
n = a.n_dims
blocks = dict(mean=slice(0, n), chol=slice(n, n + n_chol(n)), color=slice(n + n_chol(n), n + n_chol(n) + 3),
              amp=slice(n + n_chol(n) + 3, n + n_chol(n) + 4))
rel = lambda x, y: float(np.linalg.norm(x - y) / max(np.linalg.norm(y), 1e-300))
o = a.other
errs = {k: rel(out[o]["g"][:, s], out["fp32"]["g"][:, s]) for k, s in blocks.items()}
errs.update({f"stat{j}": rel(out[o]["st"][:, j], out["fp32"]["st"][:, j]) for j in range(3)})
print(json.dumps({"n": n, "G": a.gaussians, "B": a.batch, "regime": a.regime, f"impl_{o}": out[o]["impl"],
                  "fp32_ms": out["fp32"]["ms"], f"{o}_ms": out[o]["ms"], "rel": errs}))
