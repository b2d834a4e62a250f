"""File-source training data: datasets.FileDataset draws random slices
without replacement per epoch (reshuffled at the wrap), sorts each slice by the first dimension into
tiles, splits them over ranks like the procedural sampler, perturbs only direction-tagged dimensions
(clamped to [0, 1]); `ndgauss fit` trains from an NDGT file and resumes bit-identically."""
import os

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _data(M=3000, N=6, seed=0):
    rng = np.random.default_rng(seed)
    q = rng.random((M, N), dtype=np.float32)
    q[:, 5] = np.arange(M, dtype=np.float32) / M          # an exact per-point id (unique, in [0, 1))
    t = rng.random((M, 3), dtype=np.float32)
    return q, t


def test_epochs_without_replacement_and_sorted_tiles(cuda):
    from paper_2405_20067_b200 import datasets as D
    q, t = _data()
    ds = D.FileDataset(q, t, seed=3)
    seen = []
    for _ in range(5):                                     # 5 x 1024 = 5120 > 3000: one wrap
        qb, tb = D.sample_batch(ds, 6, 1024, 256, None, "cuda")
        qn = qb.cpu().numpy()
        assert np.all(np.diff(qn[:, 0]) >= 0)              # whole batch sorted by dim 0 -> tiles sorted
        ids = np.rint(qn[:, 5] * 3000).astype(int)
        assert np.array_equal(tb.cpu().numpy(), t[ids])    # targets follow their queries
        seen.append(ids)
    allids = np.concatenate(seen)                          # batches are sorted, so epochs mix in batch 3
    assert len(np.unique(np.concatenate(seen[:2]))) == 2048  # within an epoch: no repeats
    counts = np.bincount(allids, minlength=3000)
    assert counts.min() == 1 and counts.max() == 2           # epoch 1 covers every point once ...
    assert int((counts == 2).sum()) == 5120 - 3000           # ... epoch 2 (partial) adds no repeats
    assert ds.state()["epoch"] == 1 and ds.state()["pos"] == 5120 - 3000


def test_rank_slices_and_state_replay(cuda):
    from paper_2405_20067_b200 import datasets as D
    q, t = _data()
    full = D.FileDataset(q, t, seed=5)
    st0 = full.state()
    qa, ta = D.sample_batch(full, 6, 1024, 256, None, "cuda")
    parts = []
    for r in range(2):
        ds = D.FileDataset(q, t, seed=5)
        ds.set_state(st0)
        parts.append(D.sample_batch(ds, 6, 1024, 256, None, "cuda", rank=r, world=2)[0])
    back = torch.empty_like(qa).view(4, 256, 6)
    back[0::2], back[1::2] = parts[0].view(2, 256, 6), parts[1].view(2, 256, 6)
    assert torch.equal(back.view(-1, 6), qa)
    again = D.FileDataset(q, t, seed=5)
    again.set_state(st0)
    assert torch.equal(D.sample_batch(again, 6, 1024, 256, None, "cuda")[0], qa)


def test_perturb_directions_only_direction_dims(cuda):
    from paper_2405_20067_b200 import datasets as D
    q, t = _data()
    roles = [0, 0, 0, 1, 1, 3]                             # position x3, direction x2, variable
    plain = D.FileDataset(q, t, roles, seed=1)
    pert = D.FileDataset(q, t, roles, seed=1, perturb_sigma=0.05)
    a, ta = D.sample_batch(plain, 6, 1024, 256, None, "cuda")
    b, tb = D.sample_batch(pert, 6, 1024, 256, None, "cuda")
    a, b = a.cpu().numpy(), b.cpu().numpy()
    # the same points (dim 5 is the id; the sort key dim 0 is not perturbed, so the order matches)
    assert np.array_equal(a[:, [0, 1, 2, 5]], b[:, [0, 1, 2, 5]]) and torch.equal(ta, tb)
    assert np.any(a[:, 3:5] != b[:, 3:5]) and b[:, 3:5].min() >= 0 and b[:, 3:5].max() <= 1
    zero = D.FileDataset(q, t, roles, seed=1, perturb_sigma=0.0)
    assert np.array_equal(D.sample_batch(zero, 6, 1024, 256, None, "cuda")[0].cpu().numpy(), a)


def test_fit_from_ndgt_file_and_resume(cuda, tmp_path):
    """`ndgauss fit` with data.target = file: the loss falls, and fit-20 -> resume -> 40 equals an
    uninterrupted 40-iteration run byte for byte (the file source's epoch / position state is in the
    checkpoint)."""
    from paper_2405_20067_b200 import cli
    from paper_2405_20067_b200 import datasets as D
    from paper_2405_20067_b200 import formats as F
    tgt = D.GmmOracleTarget(4, 6, 6)
    qd, td = D.sample_batch(tgt, 6, 4096, 256, D.QuerySampler(9), "cuda")
    path = tmp_path / "train.ndgt"
    F.write_ndgt(path, qd.cpu().numpy(), td.cpu().numpy(), roles=[0, 0, 0, 1, 1, 1])

    def cfg(iters):
        p = tmp_path / f"c{iters}.cfg"
        p.write_text(f"[trainer]\niterations = {iters}\nphase_length = 20\nn_components = 48\nbatch_size = 1024\n"
                     f"seed = 2\n[data]\ntarget = file\npath = {path}\nn_dims = 6\nperturb_sigma = 0.01\n")
        return str(p)

    assert cli.main(["fit", "--config", cfg(40), "--out", str(tmp_path / "full")]) == 0
    rows = (tmp_path / "full" / "metrics.csv").read_text().splitlines()[1:]
    losses = [float(r.split(",")[1]) for r in rows]
    assert len(losses) == 40 and np.mean(losses[-5:]) < np.mean(losses[:5])
    assert cli.main(["fit", "--config", cfg(20), "--out", str(tmp_path / "half")]) == 0
    assert cli.main(["fit", "--config", cfg(40), "--out", str(tmp_path / "half"),
                     "--resume", str(tmp_path / "half" / "checkpoint.ndgc")]) == 0
    a = (tmp_path / "full" / "checkpoint.ndgc").read_bytes()
    b = (tmp_path / "half" / "checkpoint.ndgc").read_bytes()
    assert a == b
