"""Pins the CPU oracle to every known-answer value SPEC.md gives for the hot path
(tests/golden/spec_kats.json) and to the SPEC's derived oracles. CPU only."""
import json
import math
import os

import numpy as np
import pytest

from oracle import ndg_oracle as O

KATS = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_kats.json")))


def _mix(n, rows, child=None, has_child=None, amp_mode=O.BRIGHTNESS):
    return O.OMixture(n, amp_mode, np.asarray(rows, np.float64), child, has_child)


@pytest.mark.parametrize("kat", KATS["activate_cholesky"])
def test_activate_cholesky(kat):
    L = O.activate_cholesky(np.asarray(kat["raw"]), kat["n"])
    assert np.allclose(L, kat["L"], rtol=0, atol=kat.get("atol", 0.0))


def test_eval_gaussian_kats():
    k0, k1, k2 = KATS["eval_gaussian"]
    assert O.eval_gaussian(k0["mean"], k0["L"], k0["x"]) == 1.0
    v = O.eval_gaussian(k1["mean"], k1["L"], k1["x"])
    assert v == pytest.approx(k1["value"], rel=1e-15) and round(float(v), 6) == k1["value_printed"]
    L = np.asarray(k2["L"])
    d = np.asarray(k2["x"]) - np.asarray(k2["mean"])
    dense = math.exp(-0.5 * d @ np.linalg.inv(L @ L.T) @ d)
    assert O.eval_gaussian(k2["mean"], L, k2["x"]) == pytest.approx(dense, rel=1e-14)


def test_eval_gaussian_vs_dense_inverse_random():
    """z-solve == dense-inverse evaluation within 1e-10 relative for N <= 12."""
    rng = np.random.default_rng(0)
    for n in range(1, 13):
        raw = rng.normal(0, 0.5, O.n_chol(n))
        L = O.activate_cholesky(raw, n)
        m = rng.random(n)
        x = m + rng.normal(0, 0.5, n)
        d = x - m
        dense = math.exp(-0.5 * d @ np.linalg.inv(L @ L.T) @ d)
        assert O.eval_gaussian(m, L, x) == pytest.approx(dense, rel=1e-10)


def test_eval_gaussian_ray_monotone():
    """maximised at x = m, strictly decreasing along rays."""
    rng = np.random.default_rng(1)
    L = O.activate_cholesky(rng.normal(0, 0.3, O.n_chol(5)), 5)
    m = rng.random(5)
    for _ in range(20):
        dirv = rng.normal(size=5)
        vals = [O.eval_gaussian(m, L, m + t * dirv) for t in np.linspace(0, 3, 30)]
        assert vals[0] == 1.0 and np.all(np.diff(vals) < 0)


def _neutral_row(n, mean):
    row = np.zeros(O.raw_width(n))
    row[:n] = mean
    return row


def test_eval_mixture_kats():
    n = 1
    row = _neutral_row(n, [0.4])
    for kat, rows in ((KATS["eval_mixture"][0], [row]), (KATS["eval_mixture"][1], [row, row])):
        ev = O.build_eval_set(_mix(n, rows))
        off, idx = O.all_active_csr(1, ev)
        pred = O.forward(np.full((256, 1), 0.4, np.float32), ev, off, idx)
        assert np.allclose(pred[0], kat["color"], rtol=0, atol=1e-7)   # x rounded to float32


def test_eval_mixture_dense_random():
    """random 5-component N=4 mixture vs an independent dense evaluator, 1e-12."""
    rng = np.random.default_rng(2)
    n, G = 4, 5
    rows = np.zeros((G, O.raw_width(n)))
    ms, cs, cols, amp = O.raw_slices(n)
    rows[:, ms] = rng.random((G, n))
    rows[:, cs] = rng.normal(-1, 0.3, (G, O.n_chol(n)))
    rows[:, cols] = rng.normal(size=(G, 3))
    rows[:, amp] = rng.normal(size=G)
    ev = O.build_eval_set(_mix(n, rows))
    q = rng.random((256, n)).astype(np.float32)
    pred = O.forward(q, ev, *O.all_active_csr(1, ev))
    for b in range(10):
        x = q[b].astype(np.float64)
        dense = np.zeros(3)
        for i in range(G):
            L = O.activate_cholesky(rows[i, cs], n)
            d = x - rows[i, ms]
            g = math.exp(-0.5 * d @ np.linalg.inv(L @ L.T) @ d)
            c = 1 / (1 + np.exp(-rows[i, cols]))
            dense += g * math.exp(rows[i, amp]) * c
        assert np.allclose(pred[b], dense, rtol=1e-12, atol=0)


def test_eval_mixture_linearity():
    """union of disjoint active sets == sum of separate evaluations (1e-12)."""
    om, _ = O.synthetic_mixture(3, 40, seed=3)
    ev = O.build_eval_set(om)
    q = O.synthetic_queries(3, 256, seed=4)
    all_ = O.forward(q, ev, np.array([0, 40]), np.arange(40, dtype=np.int32))
    a = O.forward(q, ev, np.array([0, 17]), np.arange(17, dtype=np.int32))
    b = O.forward(q, ev, np.array([0, 23]), np.arange(17, 40, dtype=np.int32))
    assert np.allclose(all_, a + b, rtol=1e-12, atol=1e-300)


def test_compose_child_kats():
    k1 = KATS["compose_child"][1]
    mc, LU = O.compose_child(k1["m_p"], k1["L"], k1["m_u"], np.eye(2))
    assert np.array_equal(mc, k1["m_c"])
    rng = np.random.default_rng(5)
    for n in (3, 6, 10):
        L = O.activate_cholesky(rng.normal(0, 0.5, O.n_chol(n)), n)
        mp = rng.random(n)
        mc, LU = O.compose_child(mp, L, np.zeros(n), np.eye(n))
        assert np.array_equal(mc, mp) and np.allclose(LU, L, rtol=0, atol=1e-15)
    L = O.activate_cholesky(rng.normal(0, 0.5, 6), 3)
    U = O.activate_cholesky(rng.normal(0, 0.5, 6), 3)
    _, LU = O.compose_child(np.zeros(3), L, np.zeros(3), U)
    assert np.allclose(np.triu(LU, 1), 0) and np.all(np.diag(LU) > 0)
    assert np.all(np.linalg.eigvalsh(LU @ LU.T) > 0)


def test_projection_set_kats():
    a = O.make_projection_set(3, 4, 7)
    b = O.make_projection_set(3, 4, 7)
    assert np.array_equal(a, b)
    R = O.make_projection_set(10, 32, 0)
    assert np.allclose(np.linalg.norm(R, axis=1), 1.0, atol=1e-12)
    rng = np.random.default_rng(0)
    dots = [float(O.make_projection_set(10, 32, s) [rng.integers(32)] @ O.make_projection_set(10, 32, s + 1000)[rng.integers(32)])
            for s in range(10000)]
    assert abs(np.mean(dots)) < 0.02


def _evset(mean, L):
    mean = np.asarray(mean, np.float64)[None]
    L = np.asarray(L, np.float64)[None]
    return O.EvalSet(G=1, Gev=1, mean=mean, L=L, a=np.ones((1, 3)), live=np.ones(1, bool),
                     degenerate=np.zeros(1, bool))


def test_project_components_kats():
    k0, k1, _ = KATS["project_components"]
    R = O.make_projection_set(3, 8, 0)
    _, sr, _ = O.project_components(_evset([0, 0, 0], k0["L"]), R)
    assert np.allclose(sr, 1.0, rtol=1e-15)
    _, sr, _ = O.project_components(_evset([0, 0], k1["L"]), np.asarray([k1["r"]]))
    assert sr[0, 0] == 2.0
    rng = np.random.default_rng(6)
    L = O.activate_cholesky(rng.normal(0, 0.5, O.n_chol(6)), 6)
    R = O.make_projection_set(6, 16, 1)
    _, sr, _ = O.project_components(_evset(np.zeros(6), L), R)
    dense = np.sqrt(np.einsum("ki,ij,kj->k", R, L @ L.T, R))
    assert np.allclose(sr[:, 0], dense, rtol=1e-12)


def test_cull_tile_axis_kats():
    for kat in KATS["cull_tile"][:2]:
        ev = _evset(kat["mean"], kat["L"])
        R = np.asarray([kat["r"]])
        mr, sr, thr = O.project_components(ev, R, kat["multiplier"])
        q = np.tile(np.asarray(kat["q"], np.float32), (1, 1))
        lo, hi = O.tile_bounds(q, R, 1)
        kept = O.cull_mask(lo, hi, mr, thr)
        assert bool(kept[0, 0]) == (not kat["culled"])


def test_cull_conservative_randomized():
    """zero culled components with density >= exp(-4.5) at a tile query."""
    rng = np.random.default_rng(7)
    viol = 0
    for trial in range(1000):                         # 1000 randomized instances
        n = int(rng.integers(2, 11))
        om, _ = O.synthetic_mixture(n, 60, seed=trial, sigma0=float(rng.uniform(0.03, 0.2)))
        ev = O.build_eval_set(om)
        R = O.make_projection_set(n, int(rng.integers(1, 33)), trial)
        centre = rng.random(n)
        q = np.clip(centre + rng.normal(0, rng.uniform(0.005, 0.2), (16, n)), 0, 1).astype(np.float32)
        mr, sr, thr = O.project_components(ev, R, 3.0)
        lo, hi = O.tile_bounds(q, R, 16)
        kept = O.cull_mask(lo, hi, mr, thr)[0]
        active = O.brute_force_active(q, ev, math.exp(-4.5))
        viol += int(np.count_nonzero(~kept[active]))
    assert viol == 0


def test_cull_monotone_in_k_and_multiplier():
    """SPEC.md:220-221."""
    om, _ = O.synthetic_mixture(6, 300, seed=8)
    ev = O.build_eval_set(om)
    q = O.synthetic_queries(6, 1024, seed=9, regime="C")
    R = O.make_projection_set(6, 32, 3)
    prev = None
    for k in (4, 8, 16, 32):
        mr, sr, thr = O.project_components(ev, R[:k], 3.0)
        kept = O.cull_mask(*O.tile_bounds(q, R[:k], 256), mr, thr)
        if prev is not None:
            assert np.all(kept <= prev)
        prev = kept
    prev = None
    for mult in (1.0, 2.0, 3.0, 4.0):
        mr, sr, thr = O.project_components(ev, R[:16], mult)
        kept = O.cull_mask(*O.tile_bounds(q, R[:16], 256), mr, thr)
        if prev is not None:
            assert np.all(kept >= prev)
        prev = kept


def test_loss_kats():
    for kat in KATS["loss_rel_l2"][:2]:
        loss, _, _ = O.loss_rel_l2(np.asarray(kat["pred"]), np.asarray(kat["target"]), kat["eps"])
        assert loss == pytest.approx(kat["loss"], abs=1e-12)
    rng = np.random.default_rng(10)
    p, t = rng.random((50, 3)), rng.random((50, 3))
    naive = 0.0
    for b in range(50):
        for c in range(3):
            naive += (p[b, c] - t[b, c]) ** 2 / (p[b, c] ** 2 + 0.01)
    assert O.loss_rel_l2(p, t, 0.01)[0] == pytest.approx(naive / 150, rel=1e-12)


@pytest.mark.parametrize("n", [1, 2, 4, 8, 10])
@pytest.mark.parametrize("amp_mode", [O.BRIGHTNESS, O.OPACITY])
def test_backward_finite_differences(n, amp_mode):
    """analytic vs central FD (h=1e-4, culling off, children live),
    1e-4 relative with a 1e-6 absolute floor."""
    om, _ = O.synthetic_mixture(n, 3, seed=11 + n, children=True, amp_mode=amp_mode, sigma0=0.35)
    q = O.synthetic_queries(n, 256, seed=12)
    t = O.synthetic_targets(256, seed=13)
    r = O.fwd_bwd(om, q, t, O.make_projection_set(n, 16, 0), cull=False)
    rng = np.random.default_rng(n)
    R = O.raw_width(n)
    worst = 0.0
    for which, g in (("parent", r["grad_parent"]), ("child", r["grad_child"])):
        for comp in range(om.G):
            entries = rng.choice(R, size=min(R, 12), replace=False)
            for e in entries:
                fd = O.finite_diff_grad(om, q, t, which, comp, int(e))
                an = g[comp, e]
                if max(abs(fd), abs(an)) < 1e-6:
                    continue
                worst = max(worst, abs(fd - an) / max(abs(an), 1e-6))
    assert worst < 1e-4


def test_backward_closed_form_1d():
    """one 1-D Gaussian, one query: d loss / d mean_raw by hand."""
    m, lraw, craw, araw, x, tg = 0.3, math.log(0.2), 0.4, -0.5, 0.45, 0.7
    rows = np.array([[m, lraw, craw, craw, craw, araw]])
    om = _mix(1, rows)
    q = np.full((256, 1), x, np.float32)
    t = np.full((256, 3), tg, np.float32)
    r = O.fwd_bwd(om, q, t, O.make_projection_set(1, 1, 0), cull=False)
    ell = 0.2
    xq = float(np.float32(x))
    g = math.exp(-0.5 * ((xq - m) / ell) ** 2)
    a = math.exp(araw) / (1 + math.exp(-craw))
    p = g * a
    tg32 = float(np.float32(tg))
    dldp = 2 * (p - tg32) / (p * p + 0.01) / 3.0        # per channel, per query (mean over 3 entries)
    dpdm = g * a * (xq - m) / ell ** 2
    assert r["grad_parent"][0, 0] == pytest.approx(3 * dldp * dpdm, rel=1e-10)


def test_backward_zero_at_optimum_and_culled_zero():
    """SPEC.md:269 (target == prediction -> zero gradients) and SPEC.md:285."""
    om, _ = O.synthetic_mixture(4, 200, seed=14)
    q = O.synthetic_queries(4, 512, seed=15, regime="C")
    R = O.make_projection_set(4, 16, 0)
    r = O.fwd_bwd(om, q, np.zeros((512, 3), np.float32), R)
    r0 = O.fwd_bwd(om, q, r["pred"].astype(np.float32), R)
    assert np.max(np.abs(r0["grad_parent"])) < 1e-4 * np.max(np.abs(r["grad_parent"]))
    used = np.zeros(om.G, bool)
    used[np.unique(r["idx"])] = True
    assert (~used).any() and np.all(r["grad_parent"][~used] == 0.0)


def test_spawn_check_materialize():
    rng = np.random.default_rng(16)
    for mode in (O.BRIGHTNESS, O.OPACITY):
        t = O.default_threshold(mode)
        rows = O.spawn_child_rows(4, 10, mode, t, rng)
        assert np.all(O.amp_activate(rows[:, -1], mode) < t / 5)
        om, _ = O.synthetic_mixture(4, 10, seed=17, amp_mode=mode)
        om.child[:] = rows
        om.has_child[:] = True
        assert O.check_materialize(om, t).size == 0
    om, _ = O.synthetic_mixture(4, 10, seed=18, amp_mode=O.OPACITY)
    om.child[:] = O.spawn_child_rows(4, 10, O.OPACITY, 0.1, rng)
    om.has_child[:] = True
    om.child[3, -1] = O.amp_inverse(0.2, O.OPACITY)
    assert list(O.check_materialize(om, 0.1)) == [3]
    om.child[5, -1] = O.amp_inverse(0.15, O.OPACITY)
    assert set(O.check_materialize(om, 0.18)) <= set(O.check_materialize(om, 0.1))


def test_materialize_preserves_output():
    """before/after eval_mixture difference < 1e-6 at 100 random queries."""
    n = 4
    om, _ = O.synthetic_mixture(n, 6, seed=19, children=True, sigma0=0.2)
    q = np.random.default_rng(20).random((256, n)).astype(np.float32)
    ev = O.build_eval_set(om)
    before = O.forward(q, ev, *O.all_active_csr(1, ev))
    idx = np.array([1, 4])
    rows, clamped = O.materialize_rows(om, idx)
    assert clamped == 0
    params = np.concatenate([om.params, rows])
    child = np.concatenate([om.child, np.zeros_like(rows)])
    hc = np.concatenate([om.has_child, np.zeros(2, bool)])
    hc[idx] = False                                   # the materialised children now live as components
    om2 = O.OMixture(n, om.amp_mode, params, child, hc)
    assert om2.G == om.G + idx.size
    ev2 = O.build_eval_set(om2)
    after = O.forward(q, ev2, *O.all_active_csr(1, ev2))
    assert np.max(np.abs(after[:100] - before[:100])) < 1e-6


def test_adam_kats():
    p = np.ones(4, np.float32)
    p2, m1, m2 = O.adam_step(p, np.zeros(4), np.zeros(4), np.zeros(4), 1, 1e-2)
    assert np.array_equal(p2, p)
    m1 = m2 = np.zeros(1)
    x = np.zeros(1, np.float64)
    steps = []
    for s in range(1, 200):
        x_prev = x.copy()
        x, m1, m2 = O.adam_step(x, np.full(1, 0.5), m1, m2, s, 1e-2)
        steps.append(float(x[0] - x_prev[0]))
    # under a constant gradient the bias-corrected step tends to -lr * sign(g)
    assert abs(steps[-1] + 0.01) < 1e-6 and abs(steps[0] + 0.01) < 1e-6
    assert abs(float(x[0]) + 0.01 * 199) < 1e-4
    x = np.array([3.0], np.float32)
    m1 = m2 = np.zeros(1)
    for s in range(1, 501):
        x, m1, m2 = O.adam_step(x, 2 * (x - 1.0), m1, m2, s, 1e-2)
    assert abs(x[0] - 1.0) < 0.05


@pytest.mark.parametrize("ctr,key,want", [
    ((0, 0, 0, 0), (0, 0), "6627e8d5 e169c58d bc57ac4c 9b00dbd8"),
    ((0xFFFFFFFF,) * 4, (0xFFFFFFFF, 0xFFFFFFFF), "408f276d 41c83b0e a20bc7c6 6d5451fd"),
    ((0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344), (0xA4093822, 0x299F31D0),
     "d16cfe09 94fdcceb 5001e420 24126ea1"),
])
def test_philox_random123_kats(ctr, key, want):
    """The sampler's Philox4x32-10 against the published Random123 known-answer vectors
    (kat_vectors: philox4x32 10 ...), which pins the oracle the GPU sampler is checked against."""
    r = O.philox4x32_10(*[[c] for c in ctr], *key)
    assert " ".join(f"{int(x[0]):08x}" for x in r) == want


def test_sampler_oracle_distribution():
    """sample_batch's order-statistics construction: dimension 0 is non-decreasing and, as a set,
    uniform on [0, 1) (Kolmogorov-Smirnov); the other dimensions are iid uniform; rank slices
    partition the global batch."""
    B, n = 1 << 15, 7
    q = O.sample_batch(n, B, 256, seed=11, draw=5)
    assert np.all(np.diff(q[:, 0]) >= 0) and q.min() >= 0 and q.max() < 1
    grid = (np.arange(B) + 0.5) / B
    for d in range(n):
        ks = np.max(np.abs(np.sort(q[:, d]) - grid))
        assert ks < 1.63 / math.sqrt(B), (d, ks)                    # 1% KS critical value
    parts = [O.sample_batch(n, B, 256, 11, 5, r, 3) for r in range(3)]
    T = B // 256
    back = np.empty_like(q).reshape(T, 256, n)
    for r in range(3):
        back[r::3] = parts[r].reshape(-1, 256, n)
    assert np.array_equal(back.reshape(B, n), q)
    assert not np.array_equal(O.sample_batch(n, 4096, 256, 11, 6), O.sample_batch(n, 4096, 256, 11, 5))
