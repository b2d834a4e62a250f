"""Small culled fwd+bwd steps that exercise every pipeline kernel once, for compute-sanitizer
(racecheck / synccheck / memcheck, one tool per run): K1-K4, the tcgen05 K5 (warp-specialised,
mbarrier rings, TMEM double buffers), the FP32 K5, the FP32 K7 and the warp-MMA K7 (per-warp smem
scratch), the fixed-point reduction kernels and K8/K9. Not a test; the sanitizer's exit code is."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2405_20067_b200 as ndg  # noqa: E402
from paper_2405_20067_b200 import datasets as D  # noqa: E402

torch.cuda.set_device(0)
for n, G, B, fwd, bwd, children in ((10, 300, 1024, "tc", "fp32", True), (16, 200, 512, "tc", "mma", True),
                                    (6, 300, 512, "fp32", "fp32", False), (12, 100, 512, "fp32", "mma", False)):
    rows, _ = D.synthetic_mixture(n, G, seed=1, children=children)
    mix = ndg.Mixture.from_arrays(n, 0, **rows)
    q = torch.from_numpy(D.synthetic_queries(n, B, seed=2, regime="C")).cuda()
    t = torch.from_numpy(D.synthetic_targets(B, seed=3)).cuda()
    hp = ndg.HotPath(n, projection_seed=2, forward=fwd, backward=bwd)
    res = hp.fwd_bwd(mix, q, t)
    state = ndg.new_adam_state(mix)
    ndg.adam_step(mix, res.grads, state, 1)
    torch.cuda.synchronize()
    print(n, fwd, hp.last_forward_impl, bwd, hp.last_backward_impl, res.loss, flush=True)
print("ok")
