"""CPU tests of the CLI file formats."""
import numpy as np
import pytest

from paper_2405_20067_b200 import formats as F
from paper_2405_20067_b200.errors import ConfigError, FileFormatError


def test_config_parse_and_errors():
    cfg = F.parse_config("# c\n[trainer]\niterations = 20\nlr_mean = 0.002\namp_mode = opacity\n"
                         "[culling]\nk = 8\ncull = false\n[data]\ntarget = gmm\nn_dims = 4\n")
    assert cfg["trainer"]["iterations"] == 20 and cfg["trainer"]["amp_mode"] == 1
    assert cfg["culling"]["cull"] is False and cfg["data"]["target"] == "gmm"
    tc = F.train_config_from(cfg)
    assert tc.iterations == 20 and tc.k == 8 and tc.cull is False
    with pytest.raises(ConfigError) as e:
        F.parse_config("[trainer]\niterations = 3\nbogus = 1\n")
    assert e.value.line == 3 and e.value.field == "bogus"
    with pytest.raises(ConfigError) as e:
        F.parse_config("[nope]\n")
    assert e.value.line == 1


def test_config_bench_section_lists():
    cfg = F.parse_config("[data]\nn_dims = 10\n[bench]\ngaussians = 20000\nregime = C\n"
                         "k_list = 4, 8, 16, 32\nmultiplier_list = 1, 2.5, 3\ntile_list = 64\n")
    b = cfg["bench"]
    assert b["k_list"] == [4, 8, 16, 32] and b["multiplier_list"] == [1, 2.5, 3]
    assert b["tile_list"] == 64 and b["regime"] == "C" and b["gaussians"] == 20000
    with pytest.raises(ConfigError):
        F.parse_config("[bench]\nk_list = 4, $\n")


def test_ndgt_roundtrip_and_errors(tmp_path):
    rng = np.random.default_rng(0)
    q = rng.random((37, 6)).astype(np.float32)
    t = rng.random((37, 3)).astype(np.float32)
    p = tmp_path / "a.ndgt"
    F.write_ndgt(p, q, t, roles=[0, 0, 0, 1, 1, 1])
    q2, t2, roles = F.read_ndgt(p)
    assert np.array_equal(q, q2) and np.array_equal(t, t2) and roles == [0, 0, 0, 1, 1, 1]
    data = p.read_bytes()
    (tmp_path / "trunc.ndgt").write_bytes(data[:-5])
    with pytest.raises(FileFormatError) as e:
        F.read_ndgt(tmp_path / "trunc.ndgt")
    assert e.value.offset is not None
    (tmp_path / "swap.ndgt").write_bytes(b"TGDN" + data[4:])
    with pytest.raises(FileFormatError):
        F.read_ndgt(tmp_path / "swap.ndgt")


def test_images(tmp_path):
    img = np.random.default_rng(1).random((5, 7, 3)).astype(np.float32)
    F.write_pfm(tmp_path / "x.pfm", img)
    assert np.array_equal(F.read_pfm(tmp_path / "x.pfm"), img)
    F.write_ppm(tmp_path / "b.ppm", np.zeros((1, 1, 3)))
    raw = (tmp_path / "b.ppm").read_bytes()
    assert raw.endswith(b"\x00\x00\x00") and raw.startswith(b"P6\n1 1\n255\n")
    F.write_ppm(tmp_path / "c.ppm", np.full((1, 1, 3), 7.0))
    assert (tmp_path / "c.ppm").read_bytes()[-3:] == b"\xff\xff\xff"


def test_checkpoint_byte_identical(tmp_path):
    rng = np.random.default_rng(2)
    n, G = 4, 9
    R = n + n * (n + 1) // 2 + 4
    st = dict(n_dims=n, amp_mode=0, iteration=17, adam_step=17, config={"trainer": {"iterations": 30}},
              dataset={"target": "gmm"}, rng={"seed": 3}, params=rng.random((G, R)).astype(np.float32),
              child=rng.random((G, R)).astype(np.float32), flags=rng.integers(0, 3, G).astype(np.uint8),
              m1p=rng.random((G, R)).astype(np.float32), m2p=rng.random((G, R)).astype(np.float32),
              m1c=rng.random((G, R)).astype(np.float32), m2c=rng.random((G, R)).astype(np.float32),
              low_count=rng.integers(0, 5, G).astype(np.int32))
    a, b = tmp_path / "a.ndgc", tmp_path / "b.ndgc"
    F.save_checkpoint(a, st)
    F.save_checkpoint(b, F.load_checkpoint(a))
    assert a.read_bytes() == b.read_bytes()
    with pytest.raises(FileFormatError):
        (tmp_path / "t.ndgc").write_bytes(a.read_bytes()[:-3])
        F.load_checkpoint(tmp_path / "t.ndgc")


def test_config_file_dataset_keys():
    """data.target = file with a path (slashes allowed in bare values) and the direction perturbation."""
    cfg = F.parse_config("[data]\ntarget = file\npath = /data/run-1/train_q.ndgt\nn_dims = 6\nperturb_sigma = 0.02\n")
    assert cfg["data"] == dict(target="file", path="/data/run-1/train_q.ndgt", n_dims=6, perturb_sigma=0.02)
