"""The device-side batch sampler and shading-toy target (csrc/ndg_sample.cu) against
the oracle: the Philox streams bit-exact, the order-statistics first coordinate within one float32 ulp
(the kernel's float64 log may differ from NumPy's in the last place), rank slices, determinism and the
shading function within float32 tolerance."""
import numpy as np
import pytest
import torch

from oracle import ndg_oracle as O

pytestmark = pytest.mark.gpu


def _D():
    from paper_2405_20067_b200 import datasets as D
    return D


@pytest.mark.parametrize("n,B,tile,seed,draw", [(4, 4096, 256, 1, 0), (10, 1 << 16, 256, 7, 3),
                                                (16, 3 * 1000, 250, 2 ** 40 + 5, 2 ** 33 + 1),
                                                (6, 256 * 4103, 256, 123, 9)])
def test_sampler_matches_oracle(cuda, n, B, tile, seed, draw):
    """B = 256 * 4103 > 2^20 spans more than one pass of the block-sum scan; the 64-bit seed / draw case
    exercises the key's high words."""
    D = _D()
    q = D.QuerySampler(seed, draw).queries(n, B, tile, "cuda").cpu().numpy()
    ref = O.sample_batch(n, B, tile, seed, draw)
    assert q.shape == ref.shape
    assert np.array_equal(q[:, 1:], ref[:, 1:])                               # integer streams: exact
    ulp = np.spacing(np.maximum(np.abs(ref[:, 0]), np.float32(1e-30)))
    assert np.all(np.abs(q[:, 0] - ref[:, 0]) <= ulp)
    assert np.all(np.diff(q[:, 0]) >= 0) and q.min() >= 0 and q.max() < 1    # sorted tiles in [0, 1)


def test_sampler_rank_slices_and_determinism(cuda):
    D = _D()
    B, tile, n = 1 << 14, 256, 8
    full = D.QuerySampler(5, 2).queries(n, B, tile, "cuda")
    again = D.QuerySampler(5, 2).queries(n, B, tile, "cuda")
    assert torch.equal(full, again)
    T = B // tile
    for world in (2, 3, 8):
        for r in range(world):
            part = D.QuerySampler(5, 2).queries(n, B, tile, "cuda", r, world)
            assert torch.equal(part, full.view(T, tile, n)[r::world].reshape(-1, n))
    s = D.QuerySampler(5)
    a, b = s.queries(n, B, tile, "cuda"), s.queries(n, B, tile, "cuda")
    assert s.state() == {"seed": 5, "draw": 2} and not torch.equal(a, b)
    assert torch.equal(b, D.QuerySampler(5, 1).queries(n, B, tile, "cuda"))


def test_sample_batch_targets_and_errors(cuda):
    D = _D()
    tgt = D.ShadingToyTarget(0, 6)
    q, t = D.sample_batch(tgt, 6, 2048, 256, D.QuerySampler(4), "cuda", rank=1, world=2)
    assert q.shape == (1024, 6) and t.shape == (1024, 3)
    with pytest.raises(ValueError):
        D.sample_batch(tgt, 6, 2000, 256, 4, "cuda")
    with pytest.raises(ValueError):
        D.sample_batch(tgt, 6, 512, 256, 4, "cuda", rank=0, world=4)


@pytest.mark.parametrize("n", [4, 5, 6, 8, 9, 10])
def test_shading_target_matches_oracle(cuda, n):
    D = _D()
    tgt = D.ShadingToyTarget(3, n)
    q = D.QuerySampler(8).queries(n, 1 << 15, 256, "cuda")
    got = tgt(q).cpu().numpy()
    ref = O.shading_toy(q.cpu().numpy(), tgt.freq, tgt.phase)
    assert got.shape == (1 << 15, 3) and got.dtype == np.float32
    assert np.max(np.abs(got - ref)) < 2e-5, np.max(np.abs(got - ref))


def test_sorted_tiling_culls_at_least_random_tiling(cuda):
    """on a 10k-component mixture, tiles of queries sorted by the first position dimension
    cull a larger or equal fraction than random tiles of the same queries, on average over 100 batches."""
    import paper_2405_20067_b200 as ndg
    D = _D()
    om, _ = O.synthetic_mixture(6, 10000, seed=1, sigma0=0.05)
    mix = ndg.Mixture.from_arrays(6, om.amp_mode, om.params)
    hp = ndg.HotPath(6, projection_seed=2)
    recs = hp.activate(mix)
    pb = hp.project(recs)
    s = D.QuerySampler(21)
    kept_sorted, kept_random = [], []
    for b in range(100):
        q = s.queries(6, 4096, 256, "cuda")
        perm = torch.randperm(4096, generator=torch.Generator(device="cuda").manual_seed(b), device="cuda")
        for qq, acc in ((q, kept_sorted), (q[perm].contiguous(), kept_random)):
            acc.append(hp.cull(hp.tile_bounds(qq), pb).kept_fraction(recs.Gev))
    assert np.mean(kept_sorted) <= np.mean(kept_random), (np.mean(kept_sorted), np.mean(kept_random))


def test_gmm_target_spec_examples(cuda):
    """one component queried at its mean gives alpha * c exactly (to float32); the same
    seed twice gives identical targets; sample_batch with batch_size = tile_size is one tile."""
    D = _D()
    tgt = D.GmmOracleTarget(3, 5, 1)
    row = tgt.mixture.params[0].double().cpu().numpy()
    mean = torch.tensor(row[:5], dtype=torch.float32, device="cuda")
    q = mean.repeat(256, 1).contiguous()
    got = tgt(q)[0].double().cpu().numpy()
    n, P = 5, 15
    color = 1.0 / (1.0 + np.exp(-row[n + P:n + P + 3]))
    alpha = np.exp(row[n + P + 3])
    assert np.allclose(got, alpha * color, rtol=1e-6, atol=0)
    a = D.GmmOracleTarget(11, 6, 4)(D.QuerySampler(1).queries(6, 1024, 256, "cuda"))
    b = D.GmmOracleTarget(11, 6, 4)(D.QuerySampler(1).queries(6, 1024, 256, "cuda"))
    assert torch.equal(a, b)
    q1, t1 = D.sample_batch(tgt, 5, 256, 256, D.QuerySampler(2), "cuda")
    assert q1.shape == (256, 5) and t1.shape == (256, 3) and torch.all(q1[1:, 0] >= q1[:-1, 0])


def test_shading_toy_spec_examples(cuda):
    """the glossy lobe's exponent is at its minimum at roughness 1 (the broadest lobe: for
    the same view / reflection alignment the glossy term is largest), and a grid slice equals the
    generator evaluated pointwise (the kernel against the float64 restatement, per query)."""
    D = _D()
    tgt = D.ShadingToyTarget(5, 10)
    q = D.QuerySampler(3).queries(10, 4096, 256, "cuda")
    lo, hi = q.clone(), q.clone()
    lo[:, 9], hi[:, 9] = 0.0, 1.0
    lo[:, 6:9] = hi[:, 6:9] = 0.0                          # albedo 0: only the glossy term 0.4 * lobe remains
    glossy0, glossy1 = tgt(lo).double().cpu().numpy(), tgt(hi).double().cpu().numpy()
    assert np.all(glossy1 >= glossy0 - 1e-7) and glossy1.mean() > glossy0.mean()
    u = torch.linspace(0, 1, 64, device="cuda")
    grid = torch.full((64 * 64, 10), 0.5, device="cuda")
    grid[:, 0] = u.repeat_interleave(64)
    grid[:, 1] = u.repeat(64)
    img = tgt(grid).double().cpu().numpy()
    ref = O.shading_toy(grid.cpu().numpy(), tgt.freq, tgt.phase)
    assert np.max(np.abs(img - ref)) < 2e-5
