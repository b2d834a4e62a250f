"""Edge cases of the round-2 paths on the GPU: the bucket pre-filter and the fixed-point backward on
tiny, empty and degenerate inputs (one tile, one Gaussian, every component frozen, Gev not a multiple
of 32), all against the oracle."""
import numpy as np
import pytest
import torch

from oracle import ndg_oracle as O

pytestmark = pytest.mark.gpu


def _mix(om):
    import paper_2405_20067_b200 as ndg
    return ndg.Mixture.from_arrays(om.n_dims, om.amp_mode, om.params, om.child, om.has_child, om.frozen)


@pytest.mark.parametrize("G,B,mode", [(1, 256, "on"), (33, 256, "on"), (33, 512, "off"), (100, 768, "on")])
def test_tiny_problems_match_oracle(cuda, G, B, mode):
    import paper_2405_20067_b200 as ndg
    om, _ = O.synthetic_mixture(6, G, seed=G, children=G > 1)
    q = O.synthetic_queries(6, B, seed=2, regime="C")
    t = O.synthetic_targets(B, seed=3)
    hp = ndg.HotPath(6, projection_seed=2, prefilter=mode)
    hp.PREFILTER_MIN_TESTS = 0
    res = hp.fwd_bwd(_mix(om), torch.from_numpy(q).cuda(), torch.from_numpy(t).cuda())
    ref = O.fwd_bwd(om, q, t, hp.ps.vectors)
    assert np.array_equal(res.candidates.offsets.cpu().numpy(), ref["offsets"])
    assert np.array_equal(res.candidates.idx.cpu().numpy(), ref["idx"])
    g, r = res.grads.params.cpu().numpy(), ref["grad_parent"]
    assert np.linalg.norm(g - r) <= 1e-4 * max(np.linalg.norm(r), 1e-30)


def test_every_component_frozen(cuda):
    """No live Gaussian: empty candidate lists from both K4 passes, zero prediction and gradients."""
    import paper_2405_20067_b200 as ndg
    om, _ = O.synthetic_mixture(4, 50, seed=1)
    om.frozen[:] = True
    q = O.synthetic_queries(4, 512, seed=2)
    t = O.synthetic_targets(512, seed=3)
    for mode in ("on", "off"):
        hp = ndg.HotPath(4, projection_seed=2, prefilter=mode)
        hp.PREFILTER_MIN_TESTS = 0
        res = hp.fwd_bwd(_mix(om), torch.from_numpy(q).cuda(), torch.from_numpy(t).cuda())
        assert res.candidates.n_pairs_tiles == 0
        gr = res.grads
        assert float(res.pred.abs().max()) == 0.0
        assert all(float(x.abs().max()) == 0.0 for x in (gr.params, gr.child, gr.stats))
        assert res.loss == pytest.approx(O.fwd_bwd(om, q, t, hp.ps.vectors)["loss"], rel=1e-6)


def test_far_gaussian_contributes_exact_zero(cuda):
    """A Gaussian culled from every tile gets exactly zero gradient through the fixed-point
    reduction, and a live one next to it is unaffected."""
    import paper_2405_20067_b200 as ndg
    om, _ = O.synthetic_mixture(3, 2, seed=4, sigma0=0.05)
    om.params[1, :3] = [30.0, 30.0, 30.0]                   # far outside the unit cube
    q = O.synthetic_queries(3, 512, seed=5)
    t = O.synthetic_targets(512, seed=6)
    hp = ndg.HotPath(3, projection_seed=2)
    res = hp.fwd_bwd(_mix(om), torch.from_numpy(q).cuda(), torch.from_numpy(t).cuda())
    g = res.grads.params.cpu().numpy()
    assert np.all(g[1] == 0.0) and np.any(g[0] != 0.0)
    ref = O.fwd_bwd(om, q, t, hp.ps.vectors)
    assert np.linalg.norm(g[0] - ref["grad_parent"][0]) <= 1e-4 * np.linalg.norm(ref["grad_parent"][0])


def test_epilogue_warp_and_thread_forms_agree_bitwise(cuda, tmp_path):
    """K8 runs a warp per component for small G and a thread per component for large G
    (NDG_EPILOGUE_WARP_MAX); both evaluate the same operations in the same order, so a step's gradients
    are byte-identical whichever form ran (checked in two processes, one per form)."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = (
        "import sys, numpy as np, torch; sys.path.insert(0, %r)\n"
        "import paper_2405_20067_b200 as ndg\n"
        "from oracle import ndg_oracle as O\n"
        "om, _ = O.synthetic_mixture(7, 300, seed=5, children=True)\n"
        "mix = ndg.Mixture.from_arrays(7, om.amp_mode, om.params, om.child, om.has_child, om.frozen)\n"
        "q = torch.from_numpy(O.synthetic_queries(7, 1024, seed=6)).cuda()\n"
        "t = torch.from_numpy(O.synthetic_targets(1024, seed=7)).cuda()\n"
        "r = ndg.HotPath(7, projection_seed=2).fwd_bwd(mix, q, t)\n"
        "np.save(sys.argv[1], r.grads.flat.cpu().numpy())\n" % root)
    outs = []
    for tag, env in (("warp", {}), ("thread", {"NDG_EPILOGUE_WARP_MAX": "0"})):
        path = tmp_path / f"{tag}.npy"
        subprocess.check_call([sys.executable, "-c", code, str(path)], env=dict(os.environ, **env))
        outs.append(np.load(path))
    assert outs[0].tobytes() == outs[1].tobytes()
