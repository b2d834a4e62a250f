"""condition_gaussian / covariance_from_factor: the SPEC's examples and
the conditioning oracle (weight x conditional = joint on the slice, 1e-9 relative)."""
import numpy as np
import pytest

from paper_2405_20067_b200.conditioning import condition_factor, condition_gaussian, covariance_from_factor
from paper_2405_20067_b200.errors import DegenerateSliceError
from paper_2405_20067_b200.gmm import raw_slices, n_chol
from paper_2405_20067_b200.trainer import _activate


def _eval(mean, L, x):
    """eval_gaussian: exp(-1/2 |z|^2), L z = x - m."""
    z = np.linalg.solve(L, x - mean)
    return np.exp(-0.5 * z @ z)


def test_covariance_from_factor_examples():
    assert np.array_equal(covariance_from_factor(np.eye(3)), np.eye(3))
    assert np.array_equal(covariance_from_factor([[2.0, 0.0], [1.0, 1.0]]), [[4.0, 2.0], [2.0, 2.0]])
    rng = np.random.default_rng(0)
    L = np.tril(rng.normal(size=(8, 8))) + 3 * np.eye(8)
    V = covariance_from_factor(L)
    assert np.array_equal(V, V.T) and np.all(np.linalg.eigvalsh(V) > 0)


def test_condition_examples():
    # diagonal V: conditional = marginal of the free dims, weight = product of 1-D Gaussians
    L = np.diag([0.5, 2.0, 1.5])
    m = np.array([0.1, -0.3, 0.7])
    ma, Va, w = condition_factor(m, L, [1], [0.7])
    assert np.allclose(ma, m[[0, 2]]) and np.allclose(Va, np.diag([0.25, 2.25]))
    assert np.isclose(w, np.exp(-0.5 * ((0.7 + 0.3) / 2.0) ** 2))
    # V = [[2,1],[1,1]], fix dim 2 at m2 + 1 -> mean m1 + 1, variance 1, weight exp(-0.5)
    L = np.linalg.cholesky(np.array([[2.0, 1.0], [1.0, 1.0]]))
    m = np.array([0.25, -0.5])
    ma, Va, w = condition_factor(m, L, [1], [m[1] + 1.0])
    assert np.isclose(ma[0], m[0] + 1.0, rtol=0, atol=1e-15)
    assert np.isclose(Va[0, 0], 1.0, rtol=0, atol=1e-15) and np.isclose(w, np.exp(-0.5), rtol=1e-15)


def test_condition_oracle_n6():
    """100 random N=6 instances, 3 fixed dims: weight * conditional(x_a) == joint(x_a, x_b) to 1e-9
    on a grid along the slice."""
    rng = np.random.default_rng(7)
    n = 6
    ms, cs, cols, amp = raw_slices(n)
    worst = 0.0
    for _ in range(100):
        raw = np.zeros(n + n_chol(n) + 4)
        raw[ms] = rng.uniform(0, 1, n)
        raw[cs] = rng.normal(0, 0.5, n_chol(n))
        fixed = sorted(rng.choice(n, 3, replace=False))
        xb = rng.uniform(0, 1, 3)
        ma, Va, w = condition_gaussian(raw, n, fixed, xb)
        L, m = _activate(raw[cs], n), raw[ms]
        free = [d for d in range(n) if d not in fixed]
        Ca = np.linalg.cholesky(Va)
        for _ in range(20):
            xa = ma + Ca @ rng.normal(0, 1.5, 3)
            x = np.empty(n)
            x[free], x[fixed] = xa, xb
            joint = _eval(m, L, x)
            za = np.linalg.solve(Ca, xa - ma)
            cond = w * np.exp(-0.5 * za @ za)
            if joint > 1e-300:
                worst = max(worst, abs(cond - joint) / joint)
    assert worst < 1e-9, worst


def test_condition_errors():
    L = np.diag([1.0, 0.0, 1.0])              # V_bb singular when fixing dim 1
    with pytest.raises(DegenerateSliceError):
        condition_factor(np.zeros(3), L, [1], [0.0])
    with pytest.raises(ValueError):
        condition_factor(np.zeros(3), np.eye(3), [0, 1, 2], [0, 0, 0])
    with pytest.raises(ValueError):
        condition_factor(np.zeros(3), np.eye(3), [], [])


def test_condition_batched_matches_single():
    rng = np.random.default_rng(3)
    n, G = 5, 7
    means = rng.uniform(0, 1, (G, n))
    Ls = np.tril(rng.normal(0, 0.3, (G, n, n)))
    Ls[:, np.arange(n), np.arange(n)] = rng.uniform(0.2, 0.5, (G, n))
    ma, Va, w = condition_factor(means, Ls, [0, 3], [0.4, 0.6])
    for g in range(G):
        a, V, ww = condition_factor(means[g], Ls[g], [0, 3], [0.4, 0.6])
        assert np.allclose(ma[g], a, rtol=1e-14) and np.allclose(Va[g], V, rtol=1e-13) and np.isclose(w[g], ww)
