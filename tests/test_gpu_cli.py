"""CLI fit / eval on the GPU: exit codes, metrics.csv, checkpoints, resume, outputs."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_fit_eval_resume(cuda, tmp_path):
    from paper_2405_20067_b200 import cli
    from paper_2405_20067_b200 import formats as F
    cfgp = tmp_path / "fit.cfg"
    cfgp.write_text("[trainer]\niterations = 40\nphase_length = 20\nbatch_size = 2048\nn_components = 64\n"
                    "[data]\ntarget = gmm\nn_dims = 4\ntarget_components = 4\n")
    out = tmp_path / "run"
    assert cli.main(["fit", "--config", str(cfgp), "--out", str(out)]) == 0
    rows = (out / "metrics.csv").read_text().strip().splitlines()
    assert rows[0] == "iteration,loss,n_components,culled_fraction,ms_per_iter" and len(rows) == 41
    ck = F.load_checkpoint(out / "checkpoint.ndgc")
    assert ck["iteration"] == 40 and ck["params"].shape[0] >= 64
    # refinement events at iterations 20 and 40, each with the phase's density statistics
    import json
    evs = [json.loads(x) for x in (out / "events.jsonl").read_text().splitlines()]
    assert [e["iteration"] for e in evs] == [20, 40] and evs[0]["spawned"] > 0
    assert all(e["density_stats"]["pairs"] > 0 for e in evs)
    # resume for 20 more iterations
    cfgp.write_text(cfgp.read_text().replace("iterations = 40", "iterations = 60"))
    out2 = tmp_path / "run2"
    assert cli.main(["fit", "--config", str(cfgp), "--out", str(out2), "--resume", str(out / "checkpoint.ndgc")]) == 0
    assert F.load_checkpoint(out2 / "checkpoint.ndgc")["iteration"] == 60
    # bad config -> exit 2
    bad = tmp_path / "bad.cfg"
    bad.write_text("[trainer]\nnope = 1\n")
    assert cli.main(["fit", "--config", str(bad), "--out", str(tmp_path / "x")]) == 2
    # eval on a 2-D grid slice and on NDGT queries with a reference
    ev = tmp_path / "ev"
    assert cli.main(["eval", "--ckpt", str(out / "checkpoint.ndgc"), "--grid", "0,1:16,8", "--out", str(ev)]) == 0
    assert os.path.exists(ev / "slice.pfm") and os.path.exists(ev / "slice.ppm")
    q, p, _ = F.read_ndgt(ev / "pred.ndgt")
    assert q.shape == (128, 4) and p.shape == (128, 3) and np.all(np.isfinite(p))
    F.write_ndgt(tmp_path / "q.ndgt", q[:100], p[:100])
    ev2 = tmp_path / "ev2"
    assert cli.main(["eval", "--ckpt", str(out / "checkpoint.ndgc"), "--queries", str(tmp_path / "q.ndgt"),
                     "--ref", str(tmp_path / "q.ndgt"), "--out", str(ev2), "--no-cull"]) == 0
    _, p2, _ = F.read_ndgt(ev2 / "pred.ndgt")
    assert p2.shape == (100, 3) and np.all(np.isfinite(p2))


def test_bench_cull_ablation(cuda, tmp_path):
    """cmd_bench_cull on a small inference-shaped workload: multiplier 3 culls
    nothing active at the 3-sigma level (0 false culls); multiplier 1 culls contributing Gaussians
    (the paper's artifact regime) and moves the output far more; more projection vectors never keep
    more pairs."""
    from paper_2405_20067_b200 import cli
    cfgp = tmp_path / "bc.cfg"
    cfgp.write_text("[data]\nn_dims = 10\n[bench]\ngaussians = 4000\nqueries = 16384\nregime = C\n"
                    "k_list = 4, 16\nmultiplier_list = 1, 3\ntile_list = 64, 256\nreps = 1\n")
    out = tmp_path / "bc.csv"
    assert cli.main(["bench-cull", "--config", str(cfgp), "--out", str(out)]) == 0
    lines = out.read_text().strip().splitlines()
    hdr = lines[0].split(",")
    rows = [dict(zip(hdr, ln.split(","))) for ln in lines[1:]]
    assert len(rows) == 2 * 2 * 2
    for r in rows:
        if float(r["multiplier"]) == 3:
            assert int(r["false_culls"]) == 0
        else:
            assert int(r["false_culls"]) > 0
    err = {m: max(float(r["max_abs_err"]) for r in rows if float(r["multiplier"]) == m) for m in (1.0, 3.0)}
    assert err[3.0] < 0.1 * err[1.0]
    for tile in ("64", "256"):
        for m in ("1", "3"):
            kept = {int(r["k"]): int(r["kept_pairs"]) for r in rows
                    if r["tile_size"] == tile and float(r["multiplier"]) == float(m)}
            assert kept[16] <= kept[4]


def test_gradcheck_command(cuda):
    """cmd_gradcheck: the default run enforces SPEC.md:572's per-coordinate rule
    (1e-4 relative, 1e-6 absolute floor) on the analytic chain rule fed by the float64 pair loop;
    --fp32 checks the float32 product kernels under the relaxed block-relative rule. Reduced mixture
    count here; the negative control (a corrupted analytic coordinate) fails both."""
    from paper_2405_20067_b200 import cli, gradcheck
    assert cli.main(["gradcheck", "--seed", "3", "--per-n", "4"]) == 0
    assert cli.main(["gradcheck", "--seed", "3", "--per-n", "2", "--fp32"]) == 0
    assert not gradcheck.run(seed=3, per_n=1, dims=(4,), corrupt=True, out=lambda *_: None)
    assert not gradcheck.run(seed=3, per_n=1, dims=(4,), corrupt=True, out=lambda *_: None, analytic="fp32")


def test_cli_spec_examples(cuda, tmp_path):
    """a fixed-seed gmm-oracle fit run twice writes the same metrics.csv (every column
    but the wall-clock ms_per_iter); eval of an empty query file writes an empty output and exits 0; a
    query file of the wrong dimension exits 2."""
    from paper_2405_20067_b200 import cli
    from paper_2405_20067_b200 import formats as F
    cfgp = tmp_path / "fit.cfg"
    cfgp.write_text("[trainer]\niterations = 30\nphase_length = 15\nbatch_size = 2048\nn_components = 32\nseed = 4\n"
                    "[data]\ntarget = gmm\nn_dims = 4\ntarget_components = 4\n")
    runs = []
    for k in range(2):
        out = tmp_path / f"r{k}"
        assert cli.main(["fit", "--config", str(cfgp), "--out", str(out)]) == 0
        runs.append([r.rsplit(",", 1)[0] for r in (out / "metrics.csv").read_text().splitlines()])
    assert runs[0] == runs[1] and len(runs[0]) == 31
    ck = tmp_path / "r0" / "checkpoint.ndgc"
    F.write_ndgt(tmp_path / "empty.ndgt", np.zeros((0, 4), np.float32), np.zeros((0, 3), np.float32))
    assert cli.main(["eval", "--ckpt", str(ck), "--queries", str(tmp_path / "empty.ndgt"), "--out",
                     str(tmp_path / "e0")]) == 0
    q, p, _ = F.read_ndgt(tmp_path / "e0" / "pred.ndgt")
    assert q.shape == (0, 4) and p.shape == (0, 3)
    F.write_ndgt(tmp_path / "q5.ndgt", np.zeros((8, 5), np.float32), np.zeros((8, 3), np.float32))
    assert cli.main(["eval", "--ckpt", str(ck), "--queries", str(tmp_path / "q5.ndgt"), "--out",
                     str(tmp_path / "e1")]) == 2
