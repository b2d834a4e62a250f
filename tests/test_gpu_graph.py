"""engine.GraphedStep: the CUDA-graph replay of fwd_bwd (worst-case-sized candidate list, no mid-step
read-back) gives byte-identical results to the eager step, across replays with new inputs and Adam
updates in between, and falls back eagerly when the mixture's conditioning changes the kernel choice."""
import numpy as np
import pytest
import torch

from oracle import ndg_oracle as O

pytestmark = pytest.mark.gpu


def _setup(N, G, B, children, seed=0, sigma0=None):
    import paper_2405_20067_b200 as ndg
    kw = {} if sigma0 is None else dict(sigma0=sigma0)
    om, _ = O.synthetic_mixture(N, G, seed=seed, children=children, **kw)
    mix = ndg.Mixture.from_arrays(N, om.amp_mode, om.params, om.child, om.has_child, om.frozen)
    q = torch.from_numpy(O.synthetic_queries(N, B, seed=seed + 1)).cuda()
    t = torch.from_numpy(O.synthetic_targets(B, seed=seed + 2)).cuda()
    return ndg, om, mix, q, t


@pytest.mark.parametrize("N,G,B,children", [(6, 4096, 16384, False), (10, 700, 2048, True), (16, 300, 1024, False)])
def test_graph_replay_equals_eager_over_adam_steps(cuda, N, G, B, children):
    ndg, om, mix, q, t = _setup(N, G, B, children)
    mix_e = mix.clone()
    hp_g, hp_e = ndg.HotPath(N, projection_seed=2), ndg.HotPath(N, projection_seed=2)
    qg, tg = q.clone(), t.clone()
    gs = ndg.GraphedStep(hp_g, mix, qg, tg)
    st_g, st_e = ndg.new_adam_state(mix), ndg.new_adam_state(mix_e)
    ge = ndg.alloc_gradients(mix_e.G, mix_e.Gev, N, "cuda")
    for step in range(1, 5):
        qn = torch.from_numpy(O.synthetic_queries(N, B, seed=10 + step)).cuda()
        qg.copy_(qn)
        rg = gs()
        re = hp_e.fwd_bwd(mix_e, qn, t, grads=ge)
        assert torch.equal(rg.grads.flat, re.grads.flat), step
        assert torch.equal(rg.pred, re.pred) and rg.loss == re.loss
        assert rg.candidates.n_pairs_tiles == re.candidates.n_pairs_tiles
        assert torch.equal(rg.candidates.idx, re.candidates.idx)
        assert rg.kept_fraction == re.kept_fraction
        ndg.adam_step(mix, rg.grads, st_g, step)
        ndg.adam_step(mix_e, re.grads, st_e, step)
    assert torch.equal(mix.params, mix_e.params) and gs.matches(mix) and gs.launches >= 10
    assert hp_g.last_backward_impl == hp_e.last_backward_impl


def test_graph_matches_oracle_and_times_kernels(cuda):
    ndg, om, mix, q, t = _setup(6, 512, 2048, True)
    hp = ndg.HotPath(6, projection_seed=2)
    hp.enable_kernel_timing(True)
    gs = ndg.GraphedStep(hp, mix, q, t)
    hp.enable_kernel_timing(True)
    for _ in range(3):
        res = gs()
    assert len(hp.kernel_ms("forward")) == 3 and all(x > 0 for x in hp.kernel_ms("backward"))
    ref = O.fwd_bwd(om, q.cpu().numpy(), t.cpu().numpy(), hp.ps.vectors)
    assert np.array_equal(res.candidates.offsets.cpu().numpy(), ref["offsets"])
    assert np.array_equal(res.candidates.idx.cpu().numpy(), ref["idx"])
    g, r = res.grads.params.cpu().numpy(), ref["grad_parent"]
    assert np.linalg.norm(g - r) <= 1e-4 * np.linalg.norm(r)


def test_graph_falls_back_when_kernel_choice_changes(cuda):
    """Sharpen the mixture in place past the tensor-core conditioning bound: the replay notices from
    its read-back, re-runs the step eagerly on the FP32 kernels and marks itself stale."""
    ndg, om, mix, q, t = _setup(6, 256, 1024, False)
    hp = ndg.HotPath(6, projection_seed=2)
    gs = ndg.GraphedStep(hp, mix, q, t)
    assert gs.choice[0] is True                          # captured with the tcgen05 K5
    for i in range(6):
        mix.params[:, 6 + O.tri(i, i)] -= 7.0            # log-diagonal of L: sigma x e^-7
    res = gs()
    assert gs.stale and hp.last_forward_impl == "fp32" and not gs.matches(mix)
    ref = ndg.HotPath(6, projection_seed=2).fwd_bwd(mix.clone(), q, t)
    assert torch.equal(res.grads.flat, ref.grads.flat)
    with pytest.raises(RuntimeError):
        gs()


def test_graph_reports_invalid_parameters(cuda):
    ndg, om, mix, q, t = _setup(6, 256, 1024, False)
    gs = ndg.GraphedStep(ndg.HotPath(6, projection_seed=2), mix, q, t)
    mix.params[17, 2] = float("nan")
    with pytest.raises(ndg.InvalidParameterError) as ei:
        gs()
    assert ei.value.component == 17


def test_graphed_eval_equals_eager_target(cuda):
    """GmmOracleTarget.evaluate_into replays a captured evaluation (no read-back) into the caller's buffer:
    byte-identical to the eager evaluation, for new queries drawn into the same buffer."""
    from paper_2405_20067_b200 import datasets as D
    tgt = D.GmmOracleTarget(3, 6, 8)
    q = torch.empty(2048, 6, device="cuda")
    out = torch.empty(2048, 3, device="cuda")
    s = D.QuerySampler(4)
    for _ in range(3):
        s.queries(6, 2048, 256, "cuda", out=q)
        tgt.evaluate_into(q, out)
        assert torch.equal(out, tgt(q))
