"""Bit-reproducibility (SPEC.md:294 fixed-order reduction, :380 deterministic training, :552 resume
is bit-identical, :581 byte-identical checkpoints) and the data-parallel step on the product path.

The backward's cross-tile sums are exact int64 fixed point (ndg_common.cuh), so repeated steps give
byte-identical gradients whatever order the work items finish in; the fit loop's only other state is
the sampling generator and the spawn RNG, both carried by the checkpoint."""
import os
import socket

import numpy as np
import pytest
import torch

from oracle import ndg_oracle as O

pytestmark = pytest.mark.gpu


def _mk(N, G, B, *, children=False, regime="R", seed=0, amp_mode=0):
    import paper_2405_20067_b200 as ndg
    om, _ = O.synthetic_mixture(N, G, seed=seed, children=children, amp_mode=amp_mode)
    q = O.synthetic_queries(N, B, seed=seed + 1, regime=regime)
    t = O.synthetic_targets(B, seed=seed + 3)
    mix = ndg.Mixture.from_arrays(N, amp_mode, om.params, om.child, om.has_child, om.frozen)
    return om, mix, q, t


@pytest.mark.parametrize("N,G,B,children,regime,bwd", [
    (10, 3000, 8192, True, "R", "fp32"),
    (10, 3000, 8192, False, "C", "fp32"),
    (16, 2000, 4096, True, "R", "mma"),
    (6, 4096, 16384, False, "R", "fp32"),
])
def test_backward_bitwise_repeatable(cuda, N, G, B, children, regime, bwd):
    """Two identical steps -> byte-identical gradients, statistics and loss (many work items per
    Gaussian, so a float atomic reduction would differ in the last bits)."""
    import paper_2405_20067_b200 as ndg
    om, mix, q, t = _mk(N, G, B, children=children, regime=regime)
    hp = ndg.HotPath(N, projection_seed=2, backward=bwd)
    qd, td = torch.from_numpy(q).cuda(), torch.from_numpy(t).cuda()
    outs = []
    for _ in range(3):
        res = hp.fwd_bwd(mix, qd, td)
        outs.append((res.loss, res.grads.flat.cpu().numpy().tobytes()))
    assert hp.last_backward_impl == bwd
    assert outs[0] == outs[1] == outs[2]
    ref = O.fwd_bwd(om, q, t, hp.ps.vectors)
    g = res.grads.params.cpu().numpy()
    assert np.linalg.norm(g - ref["grad_parent"]) <= 1e-4 * np.linalg.norm(ref["grad_parent"])


def _fit_cfg(tmp_path, iterations, name="fit.cfg"):
    p = tmp_path / name
    p.write_text(f"[trainer]\niterations = {iterations}\nphase_length = 100\nbatch_size = 4096\n"
                 "n_components = 96\nseed = 5\n[data]\ntarget = gmm\nn_dims = 6\ntarget_components = 6\n")
    return p


def test_fit_bitwise_repeatable_and_resume(cuda, tmp_path):
    """Two 300-step fits (three refinement events) write byte-identical checkpoints; fit 150 ->
    resume -> 300 equals the uninterrupted 300-step run byte for byte, and the
    resumed metrics.csv continues the first run's rows."""
    from paper_2405_20067_b200 import cli
    c300 = _fit_cfg(tmp_path, 300)
    a, b = tmp_path / "a", tmp_path / "b"
    assert cli.main(["fit", "--config", str(c300), "--out", str(a)]) == 0
    assert cli.main(["fit", "--config", str(c300), "--out", str(b)]) == 0
    ca, cb = (a / "checkpoint.ndgc").read_bytes(), (b / "checkpoint.ndgc").read_bytes()
    assert ca == cb
    c200 = _fit_cfg(tmp_path, 200, "fit200.cfg")
    r = tmp_path / "r"
    assert cli.main(["fit", "--config", str(c200), "--out", str(r)]) == 0
    assert cli.main(["fit", "--config", str(c300), "--out", str(r), "--resume", str(r / "checkpoint.ndgc")]) == 0
    assert (r / "checkpoint.ndgc").read_bytes() == ca
    rows = (r / "metrics.csv").read_text().strip().splitlines()
    assert len(rows) == 301 and rows[1].startswith("1,") and rows[-1].startswith("300,")
    ref_rows = (a / "metrics.csv").read_text().strip().splitlines()
    assert [x.split(",")[:4] for x in rows] == [x.split(",")[:4] for x in ref_rows]


def _rank_worker(rank, world, port, q):
    """One rank of a world-2 data-parallel step on the same GPU (gloo carries the allreduce)."""
    import torch.distributed as dist

    import paper_2405_20067_b200 as ndg
    from paper_2405_20067_b200 import parallel as P
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    om, mix, qq, tt = _mk(10, 1500, 8192, children=True, regime="C", seed=4)
    ql, tl, _ = P.shard_queries(qq, tt, 256, rank, world)
    hp = ndg.HotPath(10, projection_seed=2)
    res = hp.fwd_bwd(mix, torch.from_numpy(np.ascontiguousarray(ql)).cuda(),
                     torch.from_numpy(np.ascontiguousarray(tl)).cuda(), n_total=qq.shape[0],
                     allreduce=P.make_allreduce())
    q.put((rank, res.loss, res.grads.flat.cpu().numpy(), res.grads.reduced().numel()))
    dist.barrier()
    dist.destroy_process_group()


def test_data_parallel_two_ranks_product_path(cuda):
    """world_size 2 on one GPU through the product step (gloo allreduce of the flat buffer): both ranks
    end with identical buffers equal to the 1-rank product step and to the oracle; the child block is
    reduced only because children are live."""
    import torch.multiprocessing as mp

    import paper_2405_20067_b200 as ndg
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    qres = ctx.Queue()
    procs = [ctx.Process(target=_rank_worker, args=(r, 2, port, qres)) for r in range(2)]
    for p in procs:
        p.start()
    outs = {}
    for _ in procs:
        r, loss, flat, nred = qres.get(timeout=600)
        outs[r] = (loss, flat, nred)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert np.array_equal(outs[0][1], outs[1][1])
    om, mix, q, t = _mk(10, 1500, 8192, children=True, regime="C", seed=4)
    hp = ndg.HotPath(10, projection_seed=2)
    one = hp.fwd_bwd(mix, torch.from_numpy(q).cuda(), torch.from_numpy(t).cuda())
    assert outs[0][2] == one.grads.flat.numel()                 # children live: the whole buffer is reduced
    f1 = one.grads.flat.cpu().numpy()
    G, R = mix.G, O.raw_width(10)
    for name, sl in (("params", slice(0, G * R)), ("child", slice(f1.size - G * R, f1.size))):
        a, b = outs[0][1][sl], f1[sl]
        assert np.linalg.norm(a - b) <= 1e-5 * np.linalg.norm(b), name
    assert abs(outs[0][0] - one.loss) <= 1e-6 * abs(one.loss)
    ref = O.fwd_bwd(om, q, t, hp.ps.vectors)
    gp = outs[0][1][:G * R].reshape(G, R)
    assert np.linalg.norm(gp - ref["grad_parent"]) <= 1e-4 * np.linalg.norm(ref["grad_parent"])


def test_allreduce_skips_dead_child_block(cuda):
    import paper_2405_20067_b200 as ndg
    om, mix, q, t = _mk(6, 500, 2048)
    hp = ndg.HotPath(6, projection_seed=2)
    seen = []
    res = hp.fwd_bwd(mix, torch.from_numpy(q).cuda(), torch.from_numpy(t).cuda(), allreduce=lambda x: seen.append(x.numel()))
    G, R = mix.G, O.raw_width(6)
    assert seen == [G * R + 3 * G + 2] and res.grads.flat.numel() == 2 * G * R + 3 * G + 2
