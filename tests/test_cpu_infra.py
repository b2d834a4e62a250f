"""CPU-only checks: C oracle == NumPy oracle, libndg.so exports the header's ABI, product dataset
generators == oracle generators, data-parallel sharding + one allreduce == the unsharded step
(world_size 2, gloo), status-word decoding."""
import os
import re

import numpy as np
import pytest

from oracle import c_oracle as CO
from oracle import ndg_oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("N,G,B,children,mode,regime", [
    (2, 120, 512, True, 1, "R"), (6, 300, 1024, False, 0, "C"), (10, 150, 512, True, 0, "R"),
    (16, 60, 256, True, 1, "C")])
def test_c_oracle_matches_numpy_oracle(N, G, B, children, mode, regime):
    om, _ = O.synthetic_mixture(N, G, seed=1, children=children, amp_mode=mode)
    q = O.synthetic_queries(N, B, seed=2, regime=regime)
    t = O.synthetic_targets(B, seed=3)
    R = O.make_projection_set(N, 16, 4)
    a = O.fwd_bwd(om, q, t, R)
    b = CO.step(om, q, t, R)
    assert np.array_equal(a["offsets"], b["offsets"]) and np.array_equal(a["idx"], b["idx"])
    for k in ("pred", "grad_parent", "grad_child", "stats"):
        scale = max(np.max(np.abs(a[k])), 1e-300)
        assert np.max(np.abs(a[k] - b[k])) <= 1e-12 * scale, k
    assert b["loss"] == pytest.approx(a["loss"], rel=1e-13)


def _header_functions():
    src = open(os.path.join(ROOT, "include", "ndg.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(ndg_[a-z0-9_]+)\s*\(", src)))


def test_abi_library_exports_every_header_symbol():
    """libndg.so loads without a GPU and exports exactly what include/ndg.h declares."""
    from paper_2405_20067_b200 import kernels
    lib = kernels.load()
    declared = _header_functions()
    assert declared, "no declarations parsed"
    for name in declared:
        assert hasattr(lib, name), f"libndg.so does not export {name}"
    assert sorted(kernels.SIGNATURES) == declared
    out = os.popen(f"nm -D --defined-only {kernels.LIB_PATH}").read()
    exported = set(re.findall(r"\bT (ndg_[a-z0-9_]+)", out))
    assert set(declared) <= exported


def test_abi_layout_queries():
    from paper_2405_20067_b200 import kernels
    lib = kernels.load()
    assert lib.ndg_abi_version() == 1
    for n in range(1, 17):
        assert lib.ndg_supported_dims(n)
        assert lib.ndg_raw_floats(n) == O.raw_width(n)
        rs = lib.ndg_record_floats(n)
        assert rs % 4 == 0 and rs >= 2 * n + n * (n - 1) // 2 + 3
        assert lib.ndg_query_floats(n) % 4 == 0 and lib.ndg_query_floats(n) >= n + 4
        # S'[P] | t'[N] | non-finite flag | gA[3] | stats[3]
        assert lib.ndg_accum_doubles(n) == O.n_chol(n) + n + 7
        # warp-MMA backward: one m16 block of dims, only where the FP32 K7's registers run short
        assert lib.ndg_backward_mma_supported(n) == (1 if 9 <= n <= 16 else 0)
    assert not lib.ndg_supported_dims(0) and not lib.ndg_supported_dims(17)
    assert lib.ndg_num_stats() == O.N_STATS


def test_no_oracle_import_in_product():
    """The product package never imports the checker (oracle/)."""
    pkg = os.path.join(ROOT, "paper_2405_20067_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith(".py"):
                src = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"^\s*(from|import)\s+oracle\b", src, flags=re.M), f


def test_product_generators_match_oracle():
    from paper_2405_20067_b200 import datasets as D
    for n, G, ch, mode in ((4, 50, True, 0), (10, 200, False, 1)):
        om, s0 = O.synthetic_mixture(n, G, seed=5, children=ch, amp_mode=mode)
        pm, s1 = D.synthetic_mixture(n, G, seed=5, children=ch, amp_mode=mode)
        assert s0 == s1
        assert np.array_equal(om.params, pm["params"].astype(np.float64))
        assert np.array_equal(om.child, pm["child"].astype(np.float64))
        assert np.array_equal(om.has_child, pm["has_child"])
    for reg in ("R", "C"):
        assert np.array_equal(O.synthetic_queries(6, 1024, seed=3, regime=reg),
                              D.synthetic_queries(6, 1024, seed=3, regime=reg))
    assert np.array_equal(O.synthetic_targets(512, 9), D.synthetic_targets(512, 9))


def test_projection_set_product_matches_oracle():
    from paper_2405_20067_b200.engine import make_projection_set
    for n, k, s in ((3, 4, 7), (10, 16, 2), (16, 32, 0)):
        assert np.array_equal(make_projection_set(n, k, s).vectors, O.make_projection_set(n, k, s))


def test_sharding_covers_every_tile_once():
    from paper_2405_20067_b200 import parallel as P
    for T, w in ((17, 2), (64, 8), (5, 4), (4096, 8)):
        got = np.sort(np.concatenate([P.shard_tiles(T, r, w) for r in range(w)]))
        assert np.array_equal(got, np.arange(T))
        counts = [P.shard_tiles(T, r, w).size for r in range(w)]
        assert max(counts) - min(counts) <= 1


def _dist_worker(rank, world, port, result_q):
    import torch
    import torch.distributed as dist

    from paper_2405_20067_b200 import parallel as P
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    N, G, B = 4, 80, 2048
    om, _ = O.synthetic_mixture(N, G, seed=21, children=True)
    q = O.synthetic_queries(N, B, seed=22, regime="C")
    t = O.synthetic_targets(B, seed=23)
    R = O.make_projection_set(N, 16, 0)
    ql, tl, tiles = P.shard_queries(q, t, 256, rank, world)
    r = O.fwd_bwd(om, ql, tl, R, n_total=B)                   # per-rank partial, GLOBAL normalisation
    flat = torch.from_numpy(np.concatenate([r["grad_parent"].ravel(), r["grad_child"].ravel(),
                                            r["stats"].ravel(), [r["loss"]]]))
    P.make_allreduce()(flat)                                  # the step's one collective
    result_q.put((rank, flat.numpy()))
    dist.barrier()
    dist.destroy_process_group()


def test_data_parallel_two_ranks_gloo():
    """world_size 2 over gloo: strided tile sharding + one SUM allreduce of the flat buffer equals
    the unsharded single-process step (loss, gradients and density statistics)."""
    import socket

    import torch.multiprocessing as mp
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    qres = ctx.Queue()
    procs = [ctx.Process(target=_dist_worker, args=(r, 2, port, qres)) for r in range(2)]
    for p in procs:
        p.start()
    outs = dict(qres.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    N, G, B = 4, 80, 2048
    om, _ = O.synthetic_mixture(N, G, seed=21, children=True)
    q = O.synthetic_queries(N, B, seed=22, regime="C")
    t = O.synthetic_targets(B, seed=23)
    ref = O.fwd_bwd(om, q, t, O.make_projection_set(N, 16, 0))
    want = np.concatenate([ref["grad_parent"].ravel(), ref["grad_child"].ravel(), ref["stats"].ravel(), [ref["loss"]]])
    assert np.array_equal(outs[0], outs[1])                    # replicas agree bitwise after the allreduce
    assert np.allclose(outs[0], want, rtol=1e-11, atol=1e-13 * np.max(np.abs(want)))


def test_status_decoding():
    from paper_2405_20067_b200 import engine
    n, G = 3, 10
    R = O.raw_width(n)
    st = [engine._INT64_MAX - (4 * R + 5), 0, 2, 0]
    with pytest.raises(engine.InvalidParameterError) as ei:
        engine.decode_status(st, G, n)
    assert ei.value.component == 4 and ei.value.entry == 5 and ei.value.block == "chol"
    st = [0, engine._INT64_MAX - (G * R + 7 * R + R - 1), 0, 0]
    with pytest.raises(engine.NonFiniteGradientError) as ei:
        engine.decode_status(st, G, n)
    assert ei.value.component == 7 and ei.value.block == "amp"
    assert engine.decode_status([0, 0, 3, 0], G, n) == 3
