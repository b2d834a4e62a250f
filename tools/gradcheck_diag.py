"""Arbitrates a gradcheck disagreement: product analytic gradient vs float64 finite differences
(ndg_loss_f64) vs the float64 oracle's analytic gradient, for one mixture. Debugging aid."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from oracle import ndg_oracle as O
from paper_2405_20067_b200 import gradcheck as GC, datasets as D
from paper_2405_20067_b200.gmm import Mixture
from paper_2405_20067_b200.engine import HotPath

n, amp, j = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
seed = 0 + 1000 * n + 97 * amp + j
G, B = 6, 256
e, where, nc, br, sp = GC.check_mixture(n, G, seed, amp)
print("gradcheck worst", e, where)
mix_np, _ = D.synthetic_mixture(n, G, seed=seed, amp_mode=amp, children=True, sigma0=0.2)
q = D.synthetic_queries(n, B, seed=seed + 1, regime="R", tile_size=B)
t = D.synthetic_targets(B, seed=seed + 3)
om = O.OMixture(n, amp, mix_np["params"], mix_np["child"], mix_np["has_child"], mix_np["frozen"])
ref = O.fwd_bwd(om, q, t, O.make_projection_set(n, 16, 0), tile_size=B, cull=False)
mix = Mixture.from_arrays(n, amp, **mix_np)
hp = HotPath(n, tile_size=B)
res = hp.fwd_bwd(mix, torch.from_numpy(q).cuda(), torch.from_numpy(t).cuda(), cull=False)
blk, r, c = where
gpu = (res.grads.params if blk == "parent" else res.grads.child).cpu().numpy()[r, c]
orc = (ref["grad_parent"] if blk == "parent" else ref["grad_child"])[r, c]
fdv = O.finite_diff_grad(om, q, t, blk, r, c, h=1e-4)
print("gpu analytic", gpu, "oracle analytic", orc, "oracle FD", fdv)
gp = res.grads.params.cpu().numpy(); rp = ref["grad_parent"]
print("block rel parent", np.linalg.norm(gp - rp) / np.linalg.norm(rp))
# per-coordinate view of the failing component: analytic vs the float64 evaluator's FD vs oracle FD
import paper_2405_20067_b200.gradcheck as GCm
R = gp.shape[1]
base = np.concatenate([mix_np["params"], mix_np["child"]]).astype(np.float64)
rows = [r if blk == "parent" else G + r]
coords = [(rows[0], cc) for cc in range(R)]
h = 1e-4
var = np.repeat(base[None], 2 * len(coords), axis=0)
for k, (rr, cc) in enumerate(coords):
    var[2 * k, rr, cc] += h
    var[2 * k + 1, rr, cc] -= h
dev = torch.device("cuda", 0)
var_d = torch.from_numpy(var).to(dev)
par, chi = var_d[:, :G].contiguous(), var_d[:, G:].contiguous()
qd, td = torch.from_numpy(q).to(dev), torch.from_numpy(t).to(dev)
pred = torch.empty(B, 3, dtype=torch.float64, device=dev)
loss = torch.empty(len(var), dtype=torch.float64, device=dev)
from paper_2405_20067_b200 import kernels as K
s_ = torch.cuda.current_stream().cuda_stream
bd = torch.from_numpy(base).to(dev)
bp, bc = bd[:G].contiguous(), bd[G:].contiguous()
K.call("ndg_loss_f64", n, G, amp, 1, bp.data_ptr(), bc.data_ptr(), mix.flags.data_ptr(), B, qd.data_ptr(), td.data_ptr(), None, pred.data_ptr(), loss.data_ptr(), s_)
print("base pred max diff vs oracle:", float(np.abs(pred.cpu().numpy() - ref["pred"]).max()))
inv = (1.0 / (pred * pred + 0.01)).contiguous()
K.call("ndg_loss_f64", n, G, amp, len(var), par.data_ptr(), chi.data_ptr(), mix.flags.data_ptr(), B, qd.data_ptr(), td.data_ptr(), inv.data_ptr(), None, loss.data_ptr(), s_)
lv = loss.cpu().numpy()
g_an = (gp if blk == "parent" else res.grads.child.cpu().numpy())[r]
for k, (rr, cc) in enumerate(coords):
    fdk = (lv[2 * k] - lv[2 * k + 1]) / (2 * h)
    print(cc, f"{g_an[cc]: .6e} {fdk: .6e} {O.finite_diff_grad(om, q, t, blk, r, cc, h=1e-4): .6e}")
