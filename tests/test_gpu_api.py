"""The reference-named module-level operations (paper_2405_20067_b200.api, exported by `ndgauss`) on the
GPU, against the SPEC's worked examples (tests/golden/spec_kats.json) and the oracle."""
import json
import math
import os

import numpy as np
import pytest
import torch

from oracle import ndg_oracle as O

pytestmark = pytest.mark.gpu
KATS = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_kats.json")))


def _raw_chol(L):
    """Inverse activation of a dense lower factor (diag log, off-diag logit((l + 1) / 2))."""
    n = len(L)
    raw = []
    for i in range(n):
        for j in range(i + 1):
            v = L[i][j]
            raw.append(math.log(v) if i == j else math.log((v + 1) / 2) - math.log1p(-(v + 1) / 2))
    return raw


def _row(mean, L, color=(0.0, 0.0, 0.0), amp=0.0):
    return np.array(list(mean) + _raw_chol(L) + list(color) + [amp], np.float32)


def test_activate_cholesky_kats(cuda):
    import ndgauss
    for k in KATS["activate_cholesky"]:
        L = ndgauss.activate_cholesky(np.array(k["raw"]), k["n"]).cpu().numpy()
        assert np.allclose(L, k["L"], rtol=1e-6, atol=k.get("atol", 0.0) + 1e-7), k["cite"]
    with pytest.raises(ndgauss.InvalidParameterError) as ei:
        ndgauss.activate_cholesky(np.array([[0.0, 0.0, 0.0], [0.0, float("nan"), 0.0]]), 2)
    assert ei.value.component == 1 and ei.value.entry == 1


def test_eval_gaussian_kats(cuda):
    import ndgauss
    for k in KATS["eval_gaussian"]:
        g = ndgauss.eval_gaussian(_row(k["mean"], k["L"]), np.array([k["x"]])).cpu().numpy()[0]
        if "value" in k:
            want = k["value"]
        else:                                   # explicit inverse of the covariance
            L = np.array(k["L"])
            d = np.array(k["x"]) - np.array(k["mean"])
            want = math.exp(-0.5 * d @ np.linalg.inv(L @ L.T) @ d)
        assert abs(g - want) <= 2e-6 * want, k["cite"]


def test_eval_mixture_and_compose_kats(cuda):
    import ndgauss
    one = ndgauss.Mixture.from_arrays(1, 0, [_row([0.4], [[0.3]])])
    assert np.allclose(ndgauss.eval_mixture(one, [[0.4]], "all").cpu().numpy(), 0.5, rtol=1e-6)
    two = ndgauss.Mixture.from_arrays(1, 0, [_row([0.4], [[0.3]])] * 2)
    assert np.allclose(ndgauss.eval_mixture(two, [[0.4]], "all").cpu().numpy(), 1.0, rtol=1e-6)
    # random 5-component N = 4 mixture at 10 points vs the oracle's dense evaluator
    om, _ = O.synthetic_mixture(4, 5, seed=3, sigma0=0.4)
    mix = ndgauss.Mixture.from_arrays(4, 0, om.params)
    x = np.random.default_rng(4).random((10, 4)).astype(np.float32)
    got = ndgauss.eval_mixture(mix, x, "all").cpu().numpy()
    ev = O.build_eval_set(om)
    want = np.zeros((10, 3))
    for e in range(5):
        Li = np.linalg.inv(ev.L[e])
        for b in range(10):
            z = Li @ (x[b] - ev.mean[e])
            want[b] += math.exp(-0.5 * z @ z) * ev.a[e]
    assert np.allclose(got, want, rtol=2e-6, atol=1e-7)
    # compose_child
    L2 = [[2.0, 0.0], [0.0, 2.0]]
    m_c, LU = ndgauss.compose_child(_row([0.0, 0.0], L2), _row([1.0, 0.0], [[1.0, 0.0], [0.0, 1.0]]))
    assert np.allclose(m_c.cpu().numpy(), [2.0, 0.0]) and np.allclose(LU.cpu().numpy(), L2)


def test_projection_and_cull_kats(cuda):
    import ndgauss
    ps = ndgauss.ProjectionSet(np.array([[1.0, 0.0]]), 0)
    mix = ndgauss.Mixture.from_arrays(2, 0, [_row([0.0, 0.0], [[2.0, 0.0], [0.0, 1.0]])])
    pb = ndgauss.project_components(mix, ps)
    # SPEC.md:195 (raw parameters are float32 on the device: exp(float32(ln 2)) = 2 (1 + ~2e-9))
    assert abs(float(pb.sigma_r[0, 0]) - 2.0) < 1e-7
    unit = ndgauss.Mixture.from_arrays(2, 0, [_row([0.0, 0.0], [[1.0, 0.0], [0.0, 1.0]])])
    pb1 = ndgauss.project_components(unit, ps)
    for k in KATS["cull_tile"][:2]:
        q = np.repeat(np.array([k["q"]], np.float32), 256, 0)
        tb = ndgauss.tile_bounds(q, ps)
        cl = ndgauss.cull_tile(tb, pb1, k["multiplier"])
        assert (cl.n_pairs_tiles == 0) == k["culled"], k["cite"]
    # conservativeness: cull(mult 3) contains brute_force_active(exp(-4.5))
    om, _ = O.synthetic_mixture(6, 400, seed=9)
    mix = ndgauss.Mixture.from_arrays(6, 0, om.params)
    q = O.synthetic_queries(6, 1024, seed=10, regime="C")
    ps6 = ndgauss.make_projection_set(6, 16, 2)
    cl = ndgauss.cull_tile(ndgauss.tile_bounds(q, ps6), ndgauss.project_components(mix, ps6), 3.0)
    bf = ndgauss.brute_force_active(q, mix, math.exp(-4.5))
    for kept, act in zip(ndgauss.candidate_lists(cl), bf):
        assert np.isin(act.cpu().numpy(), kept.cpu().numpy()).all()
    # epsilon = 0 -> every nondegenerate component
    assert all(int(a.numel()) == 400 for a in ndgauss.brute_force_active(q, mix, 0.0))


def test_loss_rel_l2_kats(cuda):
    import ndgauss
    for k in KATS["loss_rel_l2"][:2]:
        assert abs(ndgauss.loss_rel_l2(np.array(k["pred"]), np.array(k["target"]), k["eps"]) - k["loss"]) <= 1e-9
    rng = np.random.default_rng(1)
    p, t = rng.random((1000, 3)).astype(np.float32), rng.random((1000, 3)).astype(np.float32)
    want = sum(float((float(p[i, c]) - float(t[i, c])) ** 2 / (float(p[i, c]) ** 2 + 0.01))
               for i in range(1000) for c in range(3)) / 3000.0
    got, dp = ndgauss.loss_rel_l2(p, t, 0.01, return_grad=True)
    assert abs(got - want) <= 1e-12 * want
    p64, t64 = p.astype(np.float64), t.astype(np.float64)
    assert np.allclose(dp.cpu().numpy(), 2 * (p64 - t64) / (p64 ** 2 + 0.01) / 3000.0, rtol=1e-6)


def test_backward_and_finite_diff(cuda):
    import ndgauss
    om, _ = O.synthetic_mixture(4, 8, seed=5, children=True, sigma0=0.3)
    mix = ndgauss.Mixture.from_arrays(4, 0, om.params, om.child, om.has_child, om.frozen)
    q = O.synthetic_queries(4, 512, seed=6)
    # target = prediction -> zero gradients
    pred = ndgauss.eval_mixture(mix, q, "all")
    loss, g = ndgauss.backward(mix, (q, pred), "all")
    assert loss == 0.0 and float(g.params.abs().max()) == 0.0 and float(g.child.abs().max()) == 0.0
    t = O.synthetic_targets(512, seed=7)
    loss, g = ndgauss.backward(mix, (q, t), "all")
    ref = O.fwd_bwd(om, q, t, O.make_projection_set(4, 16, 0), cull=False)
    assert abs(loss - ref["loss"]) <= 1e-5 * ref["loss"]
    gp = g.params.cpu().numpy()
    assert np.linalg.norm(gp - ref["grad_parent"]) <= 1e-4 * np.linalg.norm(ref["grad_parent"])
    # finite_diff_grad on a few coordinates with |grad| > 1e-6: 1e-4 relative
    for which, comp, entry in (("parent", 1, 0), ("parent", 3, 6), ("child", 2, 5), ("parent", 0, 14)):
        fd = ndgauss.finite_diff_grad(mix, (q, t), (which, comp, entry))
        a = (g.params if which == "parent" else g.child)[comp, entry].item()
        if abs(fd) > 1e-6:
            assert abs(a - fd) <= 1e-4 * abs(fd) + 1e-7, (which, comp, entry, a, fd)
    # culled active sets from the public cull path
    ps = ndgauss.make_projection_set(4, 16, 0)
    cl = ndgauss.cull_tile(ndgauss.tile_bounds(q, ps), ndgauss.project_components(mix, ps))
    loss_c, gc = ndgauss.backward(mix, (q, t), cl)
    ref_c = O.fwd_bwd(om, q, t, ps.vectors)
    assert np.linalg.norm(gc.params.cpu().numpy() - ref_c["grad_parent"]) <= 1e-4 * np.linalg.norm(ref_c["grad_parent"])
