"""Re-run one seeded fuzz case (tests/test_gpu_fuzz.py) by index and print the K5 conditioning and the
per-block errors against the oracle. Debugging aid: NDG_FUZZ_CASES / NDG_FUZZ_SEED select the sweep."""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import test_gpu_fuzz as T
from oracle import ndg_oracle as O
import paper_2405_20067_b200 as ndg

name = sys.argv[1]
for c in T._cases():
    if "N{N}-t{tile}-B{B}-G{G}-{fwd}-{bwd}".format(**c) == name:
        break
else:
    raise SystemExit("no such case")
print(c)
om, s0 = O.synthetic_mixture(c["N"], c["G"], seed=c["seed"], children=c["children"], amp_mode=c["amp_mode"], sigma0=c["sigma0"])
q = O.synthetic_queries(c["N"], c["B"], seed=c["seed"] + 1, regime=c["regime"], tile_size=c["tile"])
t = O.synthetic_targets(c["B"], seed=c["seed"] + 3)
mix = ndg.Mixture.from_arrays(c["N"], c["amp_mode"], om.params, om.child, om.has_child, om.frozen)
for fwd in ("tc", "fp32"):
    hp = ndg.HotPath(c["N"], tile_size=c["tile"], projection_seed=c["seed"] + 2, forward=fwd, backward=c["bwd"])
    res = hp.fwd_bwd(mix, torch.from_numpy(q).cuda(), torch.from_numpy(t).cuda())
    ref = O.fwd_bwd(om, q, t, hp.ps.vectors, tile_size=c["tile"])
    rel = lambda a, b: float(np.linalg.norm(np.asarray(a, np.float64) - b) / max(np.linalg.norm(b), 1e-300))
    ms, cs, cols, amp = O.raw_slices(c["N"])
    out = {"sigma0": float(s0), "ran": hp.last_forward_impl, "pred": rel(res.pred.cpu().numpy(), ref["pred"])}
    if fwd == "tc":
        out["cond_rms"] = hp._recs.tc_conditioning()
        out["cond_max"] = hp._recs.tc_cond_host[0]
    for tag, got, want in (("parent", res.grads.params, ref["grad_parent"]), ("child", res.grads.child, ref["grad_child"])):
        g = got.cpu().numpy()
        for nm, sl in (("mean", ms), ("chol", cs), ("color", cols), ("amp", slice(amp, amp + 1))):
            out[f"{tag}.{nm}"] = rel(g[:, sl], want[:, sl])
    print(fwd, out)
