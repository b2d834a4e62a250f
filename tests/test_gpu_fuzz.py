"""Seeded random sweep of the whole hot path against the float64 oracle: dimension, mixture size,
tile size (including non-powers of two, tiles smaller than one 128-query MMA half and tiles larger
than the tensor-core forward's 256), children, amplitude mode, query regime and every implementation
of K5 (tcgen05, FP32) and K7 (FP32, warp-MMA for N >= 9, tcgen05 moments for N <= 12). Same bars as test_gpu_parity.py (CSR bit-exact, 1e-4 block-relative).
NDG_FUZZ_CASES / NDG_FUZZ_SEED widen the sweep (default 24 cases)."""
import os

import numpy as np
import pytest
import torch

from oracle import ndg_oracle as O

pytestmark = pytest.mark.gpu
RTOL = 1e-4


def _cases(n_cases=int(os.environ.get("NDG_FUZZ_CASES", "24")), seed=int(os.environ.get("NDG_FUZZ_SEED", "20261018"))):
    rng = np.random.default_rng(seed)
    out = []
    for i in range(n_cases):
        N = int(rng.integers(1, 17))
        tile = int(rng.choice([32, 64, 96, 128, 200, 256, 512]))
        T = int(rng.integers(1, 5))
        G = int(rng.integers(1, 400))
        fwd = str(rng.choice(["tc", "fp32"]))
        bwds = ["fp32"] + (["mma"] if N >= 9 else [])
        bwd = str(rng.choice(bwds))
        out.append(dict(N=N, tile=tile, B=tile * T, G=G, children=bool(rng.integers(0, 2)),
                        amp_mode=int(rng.integers(0, 2)), regime=str(rng.choice(["R", "C"])), fwd=fwd, bwd=bwd,
                        sigma0=None, seed=int(rng.integers(0, 1000)),
                        prefilter=str(rng.choice(["auto", "on", "off"]))))
    return out


def _rel(a, b, floor=1e-30):
    """Block-relative error; blocks whose reference norm is below `floor` are compared absolutely against
    the floor. The fwd_bwd cases use floor = 1e-12 x the step's gradient scale (sum over the batch of
    |dL/dpred|_1 + |ell|): a block that small belongs to Gaussians that no query reaches (g ~ e^-60 at
    every pair, e.g. a single 15-D Gaussian 9 sigma from all queries), whose numerically-zero gradients
    float32 resolves only to the z-GEMM's conditioning (error ~ |z~| B_e 2e-7 per pair) -- twelve orders
    below anything Adam (eps 1e-8) can act on."""
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), floor))


@pytest.mark.parametrize("case", _cases(), ids=lambda c: "N{N}-t{tile}-B{B}-G{G}-{fwd}-{bwd}-pf{prefilter}".format(**c))
def test_fuzz_fwd_bwd(cuda, case):
    import paper_2405_20067_b200 as ndg
    c = case
    om, _ = O.synthetic_mixture(c["N"], c["G"], seed=c["seed"], children=c["children"], amp_mode=c["amp_mode"],
                                sigma0=c["sigma0"])
    q = O.synthetic_queries(c["N"], c["B"], seed=c["seed"] + 1, regime=c["regime"], tile_size=c["tile"])
    t = O.synthetic_targets(c["B"], seed=c["seed"] + 3)
    mix = ndg.Mixture.from_arrays(c["N"], c["amp_mode"], om.params, om.child, om.has_child, om.frozen)
    hp = ndg.HotPath(c["N"], tile_size=c["tile"], projection_seed=c["seed"] + 2, forward=c["fwd"], backward=c["bwd"],
                     prefilter=c["prefilter"])
    res = hp.fwd_bwd(mix, torch.from_numpy(q).cuda(), torch.from_numpy(t).cuda())
    ref = O.fwd_bwd(om, q, t, hp.ps.vectors, tile_size=c["tile"])
    assert np.array_equal(res.candidates.offsets.cpu().numpy(), ref["offsets"])
    assert np.array_equal(res.candidates.idx.cpu().numpy(), ref["idx"])
    assert _rel(res.pred.cpu().numpy(), ref["pred"]) < RTOL
    assert abs(res.loss - ref["loss"]) <= RTOL * max(abs(ref["loss"]), 1e-30)
    ms, cs, cols, amp = O.raw_slices(c["N"])
    floor = max(1e-30, 1e-12 * float(np.abs(ref["dpred"]).sum() + np.abs(ref["ell"]).sum()))
    for tag, got, want in (("parent", res.grads.params, ref["grad_parent"]), ("child", res.grads.child, ref["grad_child"])):
        if tag == "child" and not c["children"]:
            continue
        g = got.cpu().numpy()
        for name, sl in (("mean", ms), ("chol", cs), ("color", cols), ("amp", slice(amp, amp + 1))):
            assert _rel(g[:, sl], want[:, sl], floor) < RTOL, f"{tag}.{name}"
    st = res.grads.stats.cpu().numpy()
    for j in range(2):
        assert _rel(st[:, j], ref["stats"][:, j], floor) < RTOL, f"stat {j}"
    assert np.array_equal(st[:, 2], ref["stats"][:, 2]), "pair counts"
