"""Debugging aid: one fuzz-style case through both K7s stage by stage; prints the Gaussians whose K7-MMA
accumulators were flagged (NaN after dequant) or differ most from the FP32 K7's."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from oracle import ndg_oracle as O
import paper_2405_20067_b200 as ndg

N, tile, B, G, seed, children, amp_mode, regime = (int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]),
                                                   int(sys.argv[5]), sys.argv[6] == "1", int(sys.argv[7]), sys.argv[8])
om, _ = O.synthetic_mixture(N, G, seed=seed, children=children, amp_mode=amp_mode)
q = O.synthetic_queries(N, B, seed=seed + 1, regime=regime, tile_size=tile)
t = O.synthetic_targets(B, seed=seed + 3)
mix = ndg.Mixture.from_arrays(N, amp_mode, om.params, om.child, om.has_child, om.frozen)
qd, td = torch.from_numpy(q).cuda(), torch.from_numpy(t).cuda()
acc = {}
for impl in ("fp32", "mma"):
    hp = ndg.HotPath(N, tile_size=tile, projection_seed=seed + 2, forward="fp32", backward=impl, prefilter="off")
    hp.reset_status()
    recs = hp.activate(mix)
    cl = hp.cull(hp.tile_bounds(qd), hp.project(recs))
    pred, qrec, lp = hp.forward(qd, recs, cl, td)
    grads = ndg.alloc_gradients(mix.G, recs.Gev, N, "cuda")
    a = hp.backward(mix, recs, cl, qrec, grads).cpu().numpy()
    acc[impl] = a
    print(impl, hp.last_backward_impl, "nan rows:", np.nonzero(np.isnan(a).any(1))[0][:20])
a, b = acc["mma"], acc["fp32"]
bad = np.nonzero(np.isnan(a).any(1))[0]
for e in bad[:3]:
    print("e", e, "mma", a[e][:12], "\nfp32", b[e][:12])
ok = ~np.isnan(a).any(1)
d = np.abs(a[ok] - b[ok]).max(1) / (np.abs(b[ok]).max(1) + 1e-30)
print("max rel row diff (finite rows):", d.max() if d.size else None)
