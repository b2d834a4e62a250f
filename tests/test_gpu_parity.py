"""GPU parity: every stage of the CUDA hot path (through the C ABI) against the CPU oracle.

Bars:
  * candidate lists (CSR offsets + indices), tile bounds and projected means: bit-exact;
  * sigma_r given the same activated factors: bit-exact; activated factors vs oracle: 1e-15 rel;
  * pred, loss, gradients: block-relative ||gpu - ref|| <= RTOL * ||ref|| with RTOL = 1e-4
    (north_star's FP32 tolerance), per block (mean / chol / color / amp, parent / child).
"""
import numpy as np
import pytest
import torch

from oracle import ndg_oracle as O

pytestmark = pytest.mark.gpu
RTOL = 1e-4


def _ndg():
    import paper_2405_20067_b200 as ndg
    return ndg


def _mk(N, G, B, *, children=False, amp_mode=0, seed=0, regime="R", sigma0=None):
    ndg = _ndg()
    om, _ = O.synthetic_mixture(N, G, seed=seed, children=children, amp_mode=amp_mode, sigma0=sigma0)
    q = O.synthetic_queries(N, B, seed=seed + 1, regime=regime)
    t = O.synthetic_targets(B, seed=seed + 3)
    mix = ndg.Mixture.from_arrays(N, amp_mode, om.params, om.child, om.has_child, om.frozen)
    return om, mix, q, t


def _rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def _check_grads(N, got, ref, tag):
    ms, cs, cols, amp = O.raw_slices(N)
    for name, sl in (("mean", ms), ("chol", cs), ("color", cols), ("amp", slice(amp, amp + 1))):
        r = ref[:, sl]
        if np.linalg.norm(r) == 0:
            assert np.linalg.norm(got[:, sl]) <= 1e-12, (tag, name)
            continue
        e = _rel(got[:, sl], r)
        assert e < RTOL, f"{tag}.{name}: block-relative error {e:.3e} >= {RTOL}"


@pytest.mark.parametrize("N", [1, 2, 3, 6, 10, 16])
@pytest.mark.parametrize("amp_mode", [0, 1])
def test_prologue_activation(cuda, N, amp_mode):
    ndg = _ndg()
    om, mix, q, t = _mk(N, 300, 256, children=True, amp_mode=amp_mode)
    hp = ndg.HotPath(N)
    recs = hp.activate(mix)
    ev = O.build_eval_set(om)
    P = O.n_chol(N)
    Lref = np.stack([ev.L[:, i, j] for i in range(N) for j in range(i + 1)], axis=1)
    assert np.allclose(recs.mean64.cpu().numpy(), ev.mean, rtol=1e-14, atol=1e-15)
    assert np.allclose(recs.chol64.cpu().numpy(), Lref, rtol=1e-14, atol=1e-15)
    ef = recs.eflags.cpu().numpy()
    assert np.array_equal(ef & 1, ev.live.astype(np.uint8))
    assert P == recs.chol64.shape[1]


@pytest.mark.parametrize("N", [2, 6, 10, 16])
def test_projection_tilebounds_cull_bitexact(cuda, N):
    ndg = _ndg()
    om, mix, q, t = _mk(N, 700, 2048, children=True, regime="C" if N > 6 else "R")
    hp = ndg.HotPath(N, projection_seed=5)
    recs = hp.activate(mix)
    pb = hp.project(recs)
    qd = torch.from_numpy(q).cuda()
    tb = hp.tile_bounds(qd)
    cl = hp.cull(tb, pb)
    torch.cuda.synchronize()
    # oracle on the GPU's own activated factors -> every float64 quantity must match bit for bit
    ev = O.build_eval_set(om)
    Lg = np.zeros_like(ev.L)
    c64 = recs.chol64.cpu().numpy()
    for i in range(N):
        for j in range(i + 1):
            Lg[:, i, j] = c64[:, O.tri(i, j)]
    ev.L = Lg
    ev.mean = recs.mean64.cpu().numpy()
    mr, sr, thr = O.project_components(ev, hp.ps.vectors, 3.0)
    assert np.array_equal(pb.m_r.cpu().numpy(), mr)
    assert np.array_equal(pb.sigma_r.cpu().numpy(), sr)
    assert np.array_equal(pb.thr.cpu().numpy(), thr)
    lo, hi = O.tile_bounds(q, hp.ps.vectors, 256)
    assert np.array_equal(tb.lo.cpu().numpy(), lo) and np.array_equal(tb.hi.cpu().numpy(), hi)
    off, idx = O.cull_csr(lo, hi, mr, thr)
    assert np.array_equal(cl.offsets.cpu().numpy(), off)
    assert np.array_equal(cl.idx.cpu().numpy(), idx)
    # and end to end against the fully independent oracle (activations computed on the CPU)
    ev2 = O.build_eval_set(om)
    mr2, sr2, thr2 = O.project_components(ev2, hp.ps.vectors, 3.0)
    off2, idx2 = O.cull_csr(lo, hi, mr2, thr2)
    assert np.array_equal(cl.offsets.cpu().numpy(), off2) and np.array_equal(cl.idx.cpu().numpy(), idx2)


@pytest.mark.parametrize("fwd", ["fp32", "tc"])
@pytest.mark.parametrize("N,G,B,children,amp_mode,regime", [
    (1, 50, 512, False, 0, "R"),
    (2, 200, 1024, True, 1, "R"),
    (4, 300, 1024, True, 0, "C"),
    (6, 512, 2048, True, 0, "R"),
    (8, 300, 1024, False, 1, "R"),
    (10, 400, 1024, True, 0, "R"),
    (10, 600, 2048, False, 1, "C"),
    (16, 200, 512, True, 0, "R"),
])
def test_fwd_bwd_parity(cuda, N, G, B, children, amp_mode, regime, fwd):
    ndg = _ndg()
    om, mix, q, t = _mk(N, G, B, children=children, amp_mode=amp_mode, regime=regime)
    hp = ndg.HotPath(N, projection_seed=2, forward=fwd)
    res = hp.fwd_bwd(mix, torch.from_numpy(q).cuda(), torch.from_numpy(t).cuda())
    ref = O.fwd_bwd(om, q, t, hp.ps.vectors)
    assert np.array_equal(res.candidates.offsets.cpu().numpy(), ref["offsets"])
    assert np.array_equal(res.candidates.idx.cpu().numpy(), ref["idx"])
    assert _rel(res.pred.cpu().numpy(), ref["pred"]) < RTOL
    assert abs(res.loss - ref["loss"]) <= RTOL * abs(ref["loss"])
    _check_grads(N, res.grads.params.cpu().numpy(), ref["grad_parent"], "parent")
    if children:
        _check_grads(N, res.grads.child.cpu().numpy(), ref["grad_child"], "child")
    st = res.grads.stats.cpu().numpy()
    for j in range(3):
        assert _rel(st[:, j], ref["stats"][:, j]) < RTOL, f"stat {j}"


@pytest.mark.parametrize("N,G,B,children,regime", [
    (9, 300, 1024, True, "R"),
    (11, 300, 1024, False, "C"),
    (13, 300, 1024, True, "R"),
    (14, 200, 512, False, "R"),
    (15, 200, 1024, True, "C"),
    (16, 300, 1024, True, "R"),
    (16, 400, 2048, False, "C"),
])
def test_mma_backward_parity(cuda, N, G, B, children, regime):
    """Warp-MMA K7 (ndg_backward_mma, the default at N >= 14; forced here down to N = 9) against the float64 oracle, at the
    default sigma0 (sharper than the tcgen05-moments cases above: z~ is formed in z-space)."""
    ndg = _ndg()
    om, mix, q, t = _mk(N, G, B, children=children, regime=regime)
    hp = ndg.HotPath(N, projection_seed=2, backward="mma")
    assert hp.backward_impl == "mma"
    res = hp.fwd_bwd(mix, torch.from_numpy(q).cuda(), torch.from_numpy(t).cuda())
    assert hp.last_backward_impl == "mma"
    ref = O.fwd_bwd(om, q, t, hp.ps.vectors)
    assert np.array_equal(res.candidates.idx.cpu().numpy(), ref["idx"])
    _check_grads(N, res.grads.params.cpu().numpy(), ref["grad_parent"], "parent")
    if children:
        _check_grads(N, res.grads.child.cpu().numpy(), ref["grad_child"], "child")
    st = res.grads.stats.cpu().numpy()
    for j in range(3):
        assert _rel(st[:, j], ref["stats"][:, j]) < RTOL, f"stat {j}"


@pytest.mark.parametrize("tile,amp_mode", [(8, 0), (64, 1), (512, 0), (1024, 1)])
def test_mma_backward_tile_sizes(cuda, tile, amp_mode):
    """K7-MMA's per-work-item x-hat fragments scale with the tile (tile * 144 B of shared memory):
    the smallest (8 = one MMA column block) to the largest (1024) tile, both amplitude modes."""
    ndg = _ndg()
    om, mix, q, t = _mk(16, 200, 2048, children=True, amp_mode=amp_mode)
    hp = ndg.HotPath(16, projection_seed=2, tile_size=tile, forward="fp32")
    assert hp.backward_impl == "mma"
    res = hp.fwd_bwd(mix, torch.from_numpy(q).cuda(), torch.from_numpy(t).cuda())
    assert hp.last_backward_impl == "mma"
    ref = O.fwd_bwd(om, q, t, hp.ps.vectors, tile_size=tile)
    assert np.array_equal(res.candidates.idx.cpu().numpy(), ref["idx"])
    _check_grads(16, res.grads.params.cpu().numpy(), ref["grad_parent"], "parent")
    _check_grads(16, res.grads.child.cpu().numpy(), ref["grad_child"], "child")


def test_mma_backward_selection(cuda):
    """auto: FP32 K7 below MMA_MIN_N, warp-MMA K7 from it on; tiles not a multiple of 8 and
    ill-conditioned steps (the z-GEMM bound) run the FP32 K7; the entry point refuses N < 9."""
    ndg = _ndg()
    from paper_2405_20067_b200 import kernels as K
    M = ndg.HotPath.MMA_MIN_N
    assert ndg.HotPath(M - 1).backward_impl == "fp32"
    assert ndg.HotPath(M).backward_impl == "mma"
    assert ndg.HotPath(16, tile_size=100).backward_impl == "fp32"
    assert ndg.HotPath(16, backward="fp32").backward_impl == "fp32"
    with pytest.raises(RuntimeError):
        K.call("ndg_backward_mma", 8, 256, 256, 0, 0, 0, 0, 0, 1, 1, 0, 0, 0)
    # a sharp mixture: conditioning past TC_FORWARD_MAX_BOUND -> this step's K7 is the FP32 one
    om, mix, q, t = _mk(16, 64, 512, sigma0=0.002)
    hp = ndg.HotPath(16, projection_seed=2)
    assert hp.backward_impl == "mma"
    res = hp.fwd_bwd(mix, torch.from_numpy(q).cuda(), torch.from_numpy(t).cuda())
    assert hp.activate(mix).tc_conditioning() > hp.TC_FORWARD_MAX_BOUND
    assert hp.last_backward_impl == "fp32"
    ref = O.fwd_bwd(om, q, t, hp.ps.vectors)
    _check_grads(16, res.grads.params.cpu().numpy(), ref["grad_parent"], "parent")


@pytest.mark.parametrize("N,regime", [(2, "R"), (6, "C"), (10, "C")])
def test_brute_force_active_mask_vs_oracle(cuda, N, regime):
    """ndg_active_mask == oracle brute_force_active per tile, and the cull keeps a
    superset of it at multiplier 3 (conservativeness)."""
    ndg = _ndg()
    om, mix, q, t = _mk(N, 300, 1024, children=True, regime=regime)
    hp = ndg.HotPath(N, projection_seed=2)
    recs = hp.activate(mix)
    qd = torch.from_numpy(q).cuda()
    eps = float(np.exp(-4.5))
    mask, counts = hp.brute_force_active(qd, recs, eps)
    m = mask.cpu().numpy().view(np.uint32)
    ev = O.build_eval_set(om)
    for tt in range(1024 // 256):
        want = O.brute_force_active(q[tt * 256:(tt + 1) * 256], ev, eps)
        got = np.flatnonzero((m[tt][np.arange(ev.Gev) // 32] >> (np.arange(ev.Gev) % 32)) & 1)
        assert np.array_equal(got, want), tt
        assert int(counts[tt]) == want.size
    cl = hp.cull(hp.tile_bounds(qd), hp.project(recs))
    kept = cl.mask.cpu().numpy().view(np.uint32)
    assert not np.any(m & ~kept)


@pytest.mark.parametrize("N,G,fwd,sigma0", [(1, 400, "tc", None), (1, 400, "fp32", None), (2, 400, "tc", 0.002),
                                              (4, 300, "fp32", 0.002), (10, 300, "tc", 0.004)])
def test_very_sharp_mixture_centred_fp32(cuda, N, G, fwd, sigma0):
    """sigma ~ 1e-3 of the domain: rho x + nb2 would cancel in float32, so the step runs the FP32 K5 /
    K7 on centred records (HotPath.FP32_CENTRE_BOUND) and still meets the 1e-4 bar."""
    ndg = _ndg()
    om, mix, q, t = _mk(N, G, 1024, children=True, regime="C", sigma0=sigma0)
    hp = ndg.HotPath(N, projection_seed=2, forward=fwd)
    res = hp.fwd_bwd(mix, torch.from_numpy(q).cuda(), torch.from_numpy(t).cuda())
    assert hp.last_forward_impl == "fp32" and hp.last_centred
    ref = O.fwd_bwd(om, q, t, hp.ps.vectors)
    assert _rel(res.pred.cpu().numpy(), ref["pred"]) < RTOL
    _check_grads(N, res.grads.params.cpu().numpy(), ref["grad_parent"], "parent")
    _check_grads(N, res.grads.child.cpu().numpy(), ref["grad_child"], "child")


@pytest.mark.parametrize("N", list(range(1, 17)))
def test_tc_forward_every_dimension(cuda, N):
    """The tcgen05 K5 launches and matches the oracle at every supported N (its shared-memory /
    TMEM configuration is derived per N: chunk size, staging depth, B-ring stages)."""
    ndg = _ndg()
    om, mix, q, t = _mk(N, 300, 512, sigma0=0.3)
    hp = ndg.HotPath(N, projection_seed=2, forward="tc")
    res = hp.fwd_bwd(mix, torch.from_numpy(q).cuda(), torch.from_numpy(t).cuda())
    assert hp.last_forward_impl == "tc"
    ref = O.fwd_bwd(om, q, t, hp.ps.vectors)
    assert _rel(res.pred.cpu().numpy(), ref["pred"]) < RTOL
    assert abs(res.loss - ref["loss"]) <= RTOL * abs(ref["loss"])


@pytest.mark.parametrize("fwd", ["fp32", "tc"])
def test_cfg1_full_size_vs_c_oracle(cuda, fwd):
    """BASELINE.json configs[0] at full size: 6-D, 4096 Gaussians, 16384 queries (64 tiles)."""
    from oracle import c_oracle as CO
    ndg = _ndg()
    om, mix, q, t = _mk(6, 4096, 16384, seed=0)
    hp = ndg.HotPath(6, projection_seed=2, forward=fwd)
    res = hp.fwd_bwd(mix, torch.from_numpy(q).cuda(), torch.from_numpy(t).cuda())
    ref = CO.step(om, q, t, hp.ps.vectors)
    assert np.array_equal(res.candidates.offsets.cpu().numpy(), ref["offsets"])
    assert np.array_equal(res.candidates.idx.cpu().numpy(), ref["idx"])
    assert _rel(res.pred.cpu().numpy(), ref["pred"]) < RTOL
    assert abs(res.loss - ref["loss"]) <= RTOL * abs(ref["loss"])
    _check_grads(6, res.grads.params.cpu().numpy(), ref["grad_parent"], "parent")


def test_culled_get_zero_gradient_and_cull_on_off(cuda):
    """SPEC.md:285 (culled -> exactly zero gradient) and SPEC.md:528 (cull on vs off < 1e-6)."""
    ndg = _ndg()
    om, mix, q, t = _mk(6, 2000, 2048, regime="C")
    hp = ndg.HotPath(6, projection_seed=2)
    qd, td = torch.from_numpy(q).cuda(), torch.from_numpy(t).cuda()
    res = hp.fwd_bwd(mix, qd, td)
    used = np.zeros(mix.G, bool)
    used[np.unique(res.candidates.idx.cpu().numpy())] = True
    assert (~used).sum() > 0
    assert np.all(res.grads.params.cpu().numpy()[~used] == 0.0)
    on = hp.evaluate(mix, qd, cull=True).cpu().numpy()
    off = hp.evaluate(mix, qd, cull=False).cpu().numpy()
    # conservativeness consequence: every culled pair has g <= exp(-mult^2/2), so per query
    # |on - off| <= exp(-4.5) * sum over that tile's culled Gaussians of a
    ev = O.build_eval_set(om)
    off_r = O.forward(q, ev, *O.all_active_csr(q.shape[0] // 256, ev))
    assert _rel(off, off_r) < RTOL
    counts = np.diff(res.candidates.offsets.cpu().numpy())
    idx = res.candidates.idx.cpu().numpy()
    for tt in range(q.shape[0] // 256):
        culled = np.setdiff1d(np.arange(mix.G), idx[res.candidates.offsets[tt].item():][:counts[tt]])
        bound = np.exp(-4.5) * ev.a[culled].sum(axis=0) + 1e-6
        assert np.all(np.abs(on - off)[tt * 256:(tt + 1) * 256] <= bound)
    # at a 6-sigma multiplier the culled tail is below 1e-6 per channel (SPEC.md:528's property)
    hp6 = ndg.HotPath(6, projection_seed=2, multiplier=6.0)
    on6 = hp6.evaluate(mix, qd, cull=True).cpu().numpy()
    assert np.max(np.abs(on6 - off)) < 1e-6


def test_invalid_parameter_reported(cuda):
    ndg = _ndg()
    om, mix, q, t = _mk(4, 64, 256)
    p = mix.params.clone()
    p[17, 5] = float("nan")
    p[40, 2] = float("inf")
    mix.params = p
    hp = ndg.HotPath(4)
    with pytest.raises(ndg.InvalidParameterError) as ei:
        hp.fwd_bwd(mix, torch.from_numpy(q).cuda(), torch.from_numpy(t).cuda())
    assert ei.value.component == 17 and ei.value.entry == 5 and ei.value.block == "chol"


def test_adam_matches_oracle(cuda):
    ndg = _ndg()
    om, mix, q, t = _mk(5, 100, 256)
    rng = np.random.default_rng(0)
    g = rng.normal(size=mix.params.shape).astype(np.float32)
    grads = ndg.alloc_gradients(mix.G, mix.G, 5, mix.device)
    grads.params.copy_(torch.from_numpy(g))
    state = ndg.new_adam_state(mix)
    p0 = mix.params.cpu().numpy()
    ndg.adam_step(mix, grads, state, step=1)
    ndg.adam_step(mix, grads, state, step=2)
    lr = O.block_lr(5)
    p, m1, m2 = O.adam_step(p0, g, np.zeros_like(p0), np.zeros_like(p0), 1, lr)
    p, m1, m2 = O.adam_step(p, g, m1, m2, 2, lr)
    assert np.array_equal(mix.params.cpu().numpy(), p)


def test_adam_rows_from_flags_frozen_and_children(cuda):
    """adam_step selects rows on the device from the flag bytes (ndg_adam_flags): frozen parents and
    children, and absent children, stay bit-for-bit untouched; the rest equal the oracle's Adam."""
    ndg = _ndg()
    om, mix, q, t = _mk(5, 100, 256, children=True)
    rng = np.random.default_rng(1)
    has_child = rng.random(100) < 0.5
    frozen = rng.random(100) < 0.3
    mix = ndg.Mixture.from_arrays(5, om.amp_mode, om.params, om.child, has_child, frozen)
    assert mix.children_live
    gp = rng.normal(size=mix.params.shape).astype(np.float32)
    gc = rng.normal(size=mix.child.shape).astype(np.float32)
    grads = ndg.alloc_gradients(mix.G, 2 * mix.G, 5, mix.device)
    grads.params.copy_(torch.from_numpy(gp))
    grads.child.copy_(torch.from_numpy(gc))
    state = ndg.new_adam_state(mix)
    p0, c0 = mix.params.cpu().numpy(), mix.child.cpu().numpy()
    ndg.adam_step(mix, grads, state, step=1)
    lr = O.block_lr(5)
    z = np.zeros_like(p0)
    p1 = O.adam_step(p0, gp, z, z, 1, lr)[0]
    c1 = O.adam_step(c0, gc, z, z, 1, lr)[0]
    upd_p = ~frozen
    upd_c = has_child & ~frozen
    got_p, got_c = mix.params.cpu().numpy(), mix.child.cpu().numpy()
    assert np.array_equal(got_p[upd_p], p1[upd_p]) and np.array_equal(got_p[~upd_p], p0[~upd_p])
    assert np.array_equal(got_c[upd_c], c1[upd_c]) and np.array_equal(got_c[~upd_c], c0[~upd_c])


@pytest.mark.parametrize("sigma0,regime,want_tc", [(0.15, "R", True), (0.05, "C", True), (0.02, "C", False),
                                                    (0.005, "R", False)])
def test_tc_forward_sharp_gaussians(cuda, sigma0, regime, want_tc):
    """Tensor-core forward (3xTF32 z-GEMM) vs the float64 oracle on sharp Gaussians (the regime where
    the fp32 cancellation of the centred features is largest, tools/tc_precision_study.py). Past the
    conditioning bound (HotPath.TC_FORWARD_MAX_BOUND) the step runs the FP32-pipe K5 instead; both
    sides of the bound must meet the 1e-4 bar."""
    ndg = _ndg()
    om, mix, q, t = _mk(10, 800, 2048, regime=regime, sigma0=sigma0)
    hp = ndg.HotPath(10, projection_seed=2, forward="tc")
    res = hp.fwd_bwd(mix, torch.from_numpy(q).cuda(), torch.from_numpy(t).cuda())
    assert hp.last_forward_impl == ("tc" if want_tc else "fp32")
    ref = O.fwd_bwd(om, q, t, hp.ps.vectors)
    assert np.array_equal(res.candidates.idx.cpu().numpy(), ref["idx"])
    assert _rel(res.pred.cpu().numpy(), ref["pred"]) < RTOL
    _check_grads(10, res.grads.params.cpu().numpy(), ref["grad_parent"], "parent")


@pytest.mark.parametrize("N,amp_mode", [(1, 0), (4, 1), (10, 0)])
def test_loss_f64_evaluator_vs_oracle(cuda, N, amp_mode):
    """ndg_loss_f64 (gradcheck's finite-difference evaluator) is the float64 model itself: its base
    prediction and its loss with the base denominator match the oracle (culling off) to ~1e-12."""
    from paper_2405_20067_b200 import kernels as K
    om, mix, q, t = _mk(N, 6, 256, children=True, amp_mode=amp_mode, sigma0=0.2)
    ref = O.fwd_bwd(om, q, t, O.make_projection_set(N, 16, 0), tile_size=256, cull=False)
    dev = torch.device("cuda", 0)
    base = torch.from_numpy(np.concatenate([om.params, om.child]).astype(np.float64)).to(dev)
    par, chi = base[:6].contiguous(), base[6:].contiguous()
    qd, td = torch.from_numpy(q).to(dev), torch.from_numpy(t).to(dev)
    pred = torch.empty(256, 3, dtype=torch.float64, device=dev)
    loss = torch.empty(1, dtype=torch.float64, device=dev)
    s = torch.cuda.current_stream().cuda_stream
    K.call("ndg_loss_f64", N, 6, amp_mode, 1, par.data_ptr(), chi.data_ptr(), mix.flags.data_ptr(), 256,
           qd.data_ptr(), td.data_ptr(), None, pred.data_ptr(), loss.data_ptr(), s)
    p = pred.cpu().numpy()
    assert np.abs(p - ref["pred"]).max() <= 1e-12 * max(1.0, np.abs(ref["pred"]).max())
    inv = (1.0 / (pred * pred + 0.01)).contiguous()
    K.call("ndg_loss_f64", N, 6, amp_mode, 1, par.data_ptr(), chi.data_ptr(), mix.flags.data_ptr(), 256,
           qd.data_ptr(), td.data_ptr(), inv.data_ptr(), None, loss.data_ptr(), s)
    assert abs(float(loss.cpu()[0]) - ref["loss"]) <= 1e-12 * abs(ref["loss"])


@pytest.mark.parametrize("shrink", [1.5, 10.0, 400.0])
def test_sharp_outliers_among_broad(cuda, shrink):
    """A few Gaussians `shrink` x sharper than the rest: the conditioning guard looks at the worst
    single Gaussian (HotPath.TC_FORWARD_PEAK_BOUND), not only the RMS, so the outliers' OWN gradient
    rows stay within 1e-4 (row-relative) as well as every block."""
    ndg = _ndg()
    om, _ = O.synthetic_mixture(10, 3000, seed=3, sigma0=0.15)
    sharp = np.arange(0, 3000, 375)                    # 8 outliers among 3000
    ms, cs, cols, amp = O.raw_slices(10)
    for i in range(10):
        om.params[sharp, cs.start + O.tri(i, i)] -= np.log(shrink)
        for j in range(i):        # off-diagonal activations are not scale-relative: keep them 0
            om.params[sharp, cs.start + O.tri(i, j)] = 0.0
    q = O.synthetic_queries(10, 2048, seed=4, regime="C")
    q[:256 * len(sharp)] = np.clip(om.params[np.repeat(sharp, 256), :10] +
                                   np.random.default_rng(5).normal(0, 0.15 / shrink, (256 * len(sharp), 10)), 0, 1)
    t = O.synthetic_targets(2048, seed=6)
    mix = ndg.Mixture.from_arrays(10, 0, om.params, om.child, om.has_child, om.frozen)
    hp = ndg.HotPath(10, projection_seed=2)
    res = hp.fwd_bwd(mix, torch.from_numpy(q).cuda(), torch.from_numpy(t).cuda())
    recs = hp.activate(mix)
    assert recs.tc_conditioning() <= hp.TC_FORWARD_MAX_BOUND          # the RMS alone would allow TC
    assert (hp.last_forward_impl == "tc") == (recs.tc_peak() <= hp.TC_FORWARD_PEAK_BOUND)
    if shrink > 100:
        assert hp.last_forward_impl == "fp32" and hp.last_centred
    ref = O.fwd_bwd(om, q, t, hp.ps.vectors)
    got = res.grads.params.cpu().numpy()
    _check_grads(10, got, ref["grad_parent"], "parent")
    for r in sharp:
        nr = np.linalg.norm(ref["grad_parent"][r])
        if nr > 1e-6 * np.linalg.norm(ref["grad_parent"]):
            e = np.linalg.norm(got[r] - ref["grad_parent"][r]) / nr
            assert e < RTOL, f"outlier row {r}: {e:.3e}"


@pytest.mark.parametrize("k", [37, 64, 200])
def test_cull_many_projection_vectors(cuda, k):
    """k past the register path (k > 16) up to 256: the cull reads (m_r, thr) through L1 and keeps its
    shared memory bounded; candidate lists stay bit-exact."""
    ndg = _ndg()
    om, mix, q, t = _mk(6, 700, 2048, regime="C")
    hp = ndg.HotPath(6, k=k, projection_seed=4)
    cl = hp.cull(hp.tile_bounds(torch.from_numpy(q).cuda()), hp.project(hp.activate(mix)))
    ev = O.build_eval_set(om)
    mr, sr, thr = O.project_components(ev, hp.ps.vectors, 3.0)
    lo, hi = O.tile_bounds(q, hp.ps.vectors, 256)
    off, idx = O.cull_csr(lo, hi, mr, thr)
    assert np.array_equal(cl.offsets.cpu().numpy(), off) and np.array_equal(cl.idx.cpu().numpy(), idx)


def test_nonfinite_gradient_names_component_block_and_batch_index(cuda):
    """SPEC.md:267 / errors.py:26-33: a non-finite target at query 300 makes the backward non-finite;
    the error names the lowest offending component, its block, and the batch index 300."""
    ndg = _ndg()
    om, mix, q, t = _mk(4, 64, 1024, regime="R")
    t = t.copy()
    t[300, 1] = np.nan
    hp = ndg.HotPath(4, projection_seed=2)
    with pytest.raises(ndg.NonFiniteGradientError) as ei:
        hp.fwd_bwd(mix, torch.from_numpy(q).cuda(), torch.from_numpy(t).cuda())
    e = ei.value
    assert e.block in ("mean", "chol", "color", "amp") and 0 <= e.component < 64
    assert e.batch_index == 300


@pytest.mark.parametrize("N,G,B,regime,children,k", [
    (10, 3000, 16384, "G", False, 16),
    (10, 2000, 16384, "G", True, 16),
    (6, 1500, 4096, "C", True, 16),
    (10, 1200, 4096, "R", False, 16),
    (4, 800, 4096, "G", False, 2),
    (8, 900, 4096, "C", False, 40),
])
def test_prefilter_candidate_lists_bit_identical(cuda, N, G, B, regime, children, k):
    """The bucket pre-filter (ndg_cull_prefilter) forced on, left to the device plan, and off all give
    the oracle's candidate lists bit for bit; in the G-buffer-like regime the plan takes the
    pre-filter, with uniform queries (R) it keeps the dense pass."""
    ndg = _ndg()
    from paper_2405_20067_b200 import datasets as D
    if regime == "G":
        om = O.gbuffer_mixture(N, G, seed=3)
        if children:
            om2, _ = O.synthetic_mixture(N, G, seed=3, children=True)
            om.child, om.has_child = om2.child, om2.has_child
    else:
        om, _ = O.synthetic_mixture(N, G, seed=3, children=children)
    q = D.synthetic_queries(N, B, seed=4, regime=regime)
    mix = ndg.Mixture.from_arrays(N, 0, om.params, om.child, om.has_child, om.frozen)
    qd = torch.from_numpy(q).cuda()
    ev = O.build_eval_set(om)
    R = O.make_projection_set(N, k, 2)
    mr, sr, thr = O.project_components(ev, R, 3.0)
    lo, hi = O.tile_bounds(q, R, 256)
    off, idx = O.cull_csr(lo, hi, mr, thr)
    plans = {}
    for mode in ("on", "auto", "off"):
        hp = ndg.HotPath(N, k=k, projection_seed=2, prefilter=mode)
        hp.PREFILTER_MIN_TESTS = 0                   # let the device plan decide even at test sizes
        cl = hp.cull(hp.tile_bounds(qd), hp.project(hp.activate(mix)))
        assert np.array_equal(cl.offsets.cpu().numpy(), off), mode
        assert np.array_equal(cl.idx.cpu().numpy(), idx), mode
        plans[mode] = hp.prefilter_plan()
    assert plans["on"][1] == 1 and plans["off"] is None
    if regime == "G" and k == 16:
        assert plans["auto"][1] == 1
    if regime == "R":
        assert plans["auto"][1] == 0
