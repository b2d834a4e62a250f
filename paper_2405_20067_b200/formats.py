"""File formats of the reference CLI: flat config, NDGT
tensor files, PFM / PPM images and the versioned little-endian checkpoint.

Host-side plumbing around the hot path; no GPU code here.
"""
from __future__ import annotations

import dataclasses
import io as _io
import json
import struct

import numpy as np

from .errors import ConfigError, FileFormatError

# ------------------------------------------------------------------------------------------------
# flat config: "[section]" headers and "key = value" lines; unknown keys are errors
# ------------------------------------------------------------------------------------------------
SECTIONS = {
    "trainer": ("iterations", "phase_length", "warmup_phases", "materialize_threshold", "lr_mean", "lr_chol",
                "lr_color", "lr_amp", "beta1", "beta2", "adam_eps", "batch_size", "seed", "n_components",
                "amp_mode", "loss_eps"),
    "culling": ("k", "multiplier", "tile_size", "cull"),
    "data": ("target", "n_dims", "target_components", "target_seed", "path", "perturb_sigma"),
    # cmd_bench_cull: synthetic workload + the sweep (comma-separated lists)
    "bench": ("gaussians", "queries", "regime", "sigma0", "seed", "k_list", "multiplier_list", "tile_list", "reps",
              "epsilon"),
}


def _convert(raw: str, line: int, field: str):
    v = raw.strip()
    if "," in v:                                   # list value, e.g. k_list = 4, 8, 16, 32
        return [_convert(x, line, field) for x in v.split(",") if x.strip()]
    if v.lower() in ("true", "false"):
        return v.lower() == "true"
    if v.lower() in ("brightness", "opacity"):
        return 0 if v.lower() == "brightness" else 1
    for cast in (int, float):
        try:
            return cast(v)
        except ValueError:
            pass
    if v and all(c.isalnum() or c in "_-./" for c in v):
        return v
    raise ConfigError(f"line {line}: cannot parse value {raw!r} for {field}", line=line, field=field)


def parse_config(text: str) -> dict:
    """Returns {section: {key: value}}; raises ConfigError(line, field) on any unknown key / section
    or malformed line."""
    out = {k: {} for k in SECTIONS}
    section = None
    for ln, raw in enumerate(text.splitlines(), 1):
        s = raw.split("#", 1)[0].strip()
        if not s:
            continue
        if s.startswith("[") and s.endswith("]"):
            section = s[1:-1].strip()
            if section not in SECTIONS:
                raise ConfigError(f"line {ln}: unknown section [{section}]", line=ln, field=section)
            continue
        if "=" not in s:
            raise ConfigError(f"line {ln}: expected key = value", line=ln, field=None)
        key, val = (p.strip() for p in s.split("=", 1))
        if section is None:
            raise ConfigError(f"line {ln}: key {key!r} outside a section", line=ln, field=key)
        if key not in SECTIONS[section]:
            raise ConfigError(f"line {ln}: unknown key {section}.{key}", line=ln, field=key)
        out[section][key] = _convert(val, ln, key)
    return out


def train_config_from(cfg: dict):
    from .trainer import TrainConfig
    kw = dict(cfg.get("trainer", {}))
    cul = cfg.get("culling", {})
    for k in ("k", "multiplier", "tile_size", "cull"):
        if k in cul:
            kw[k] = cul[k]
    fields = {f.name for f in dataclasses.fields(TrainConfig)}
    return TrainConfig(**{k: v for k, v in kw.items() if k in fields})


# ------------------------------------------------------------------------------------------------
# NDGT tensor file: magic "NDGT", u32 version = 1, u32 N, N role bytes, u64 count,
# count x N float32 queries, count x 3 float32 targets; little-endian.
# ------------------------------------------------------------------------------------------------
ROLES = {"position": 0, "direction": 1, "material": 2, "variable": 3}


def write_ndgt(path, queries, targets, roles=None):
    q = np.ascontiguousarray(queries, dtype="<f4")
    t = np.ascontiguousarray(targets, dtype="<f4")
    if q.ndim != 2 or t.shape != (q.shape[0], 3):
        raise ValueError("queries [count, N] and targets [count, 3] required")
    n = q.shape[1]
    roles = bytes(roles if roles is not None else [3] * n)
    with open(path, "wb") as f:
        f.write(b"NDGT" + struct.pack("<II", 1, n) + roles + struct.pack("<Q", q.shape[0]))
        f.write(q.tobytes())
        f.write(t.tobytes())


def read_ndgt(path):
    data = open(path, "rb").read()
    if len(data) < 12 or data[:4] != b"NDGT":
        raise FileFormatError("bad magic (not an NDGT file or foreign endianness)", offset=0)
    version, n = struct.unpack_from("<II", data, 4)
    if version != 1:
        raise FileFormatError(f"unsupported NDGT version {version}", offset=4)
    off = 12
    if len(data) < off + n + 8:
        raise FileFormatError("truncated header", offset=len(data))
    roles = list(data[off:off + n])
    off += n
    (count,) = struct.unpack_from("<Q", data, off)
    off += 8
    need = off + count * (n + 3) * 4
    if len(data) != need:
        raise FileFormatError(f"size mismatch: expected {need} bytes", offset=min(len(data), need))
    q = np.frombuffer(data, "<f4", count * n, off).reshape(count, n)
    t = np.frombuffer(data, "<f4", count * 3, off + count * n * 4).reshape(count, 3)
    return q.copy(), t.copy(), roles


# ------------------------------------------------------------------------------------------------
# images
# ------------------------------------------------------------------------------------------------
def write_pfm(path, img):
    img = np.ascontiguousarray(img, dtype="<f4")
    h, w = img.shape[:2]
    with open(path, "wb") as f:
        f.write(f"PF\n{w} {h}\n-1.0\n".encode())
        f.write(img[::-1].tobytes())          # PFM rows bottom-to-top


def read_pfm(path):
    data = open(path, "rb").read()
    parts = data.split(b"\n", 3)
    if parts[0] != b"PF":
        raise FileFormatError("bad PFM magic", offset=0)
    w, h = map(int, parts[1].split())
    return np.frombuffer(parts[3], "<f4", w * h * 3).reshape(h, w, 3)[::-1].copy()


def write_ppm(path, img, gamma: float = 2.2):
    img = np.asarray(img, np.float64)
    h, w = img.shape[:2]
    v = np.clip(np.power(np.clip(img, 0.0, None), 1.0 / gamma) * 255.0 + 0.5, 0, 255).astype(np.uint8)
    with open(path, "wb") as f:
        f.write(f"P6\n{w} {h}\n255\n".encode())
        f.write(v.tobytes())


# ------------------------------------------------------------------------------------------------
# checkpoint: single little-endian versioned binary; save -> load -> save is
# byte-identical (all fields fixed-width or length-prefixed; JSON written with sorted keys).
# ------------------------------------------------------------------------------------------------
CKPT_MAGIC = b"NDGC"
CKPT_VERSION = 1


def _blob(b: bytes) -> bytes:
    return struct.pack("<Q", len(b)) + b


def save_checkpoint(path, state: dict):
    """state: n_dims, amp_mode, iteration, adam_step, config (dict), dataset (dict), rng (dict),
    params/child (float32 [G,R]), flags (uint8 [G]), m1p/m2p/m1c/m2c (float32 [G,R]), low_count (int32 [G])."""
    G, R = np.asarray(state["params"]).shape
    buf = _io.BytesIO()
    buf.write(CKPT_MAGIC + struct.pack("<IIIQQQ", CKPT_VERSION, state["n_dims"], state["amp_mode"], G,
                                         state["iteration"], state["adam_step"]))
    for key in ("config", "dataset", "rng"):
        buf.write(_blob(json.dumps(state.get(key, {}), sort_keys=True, separators=(",", ":")).encode()))
    for key, dt in (("params", "<f4"), ("child", "<f4"), ("flags", "u1"), ("m1p", "<f4"), ("m2p", "<f4"),
                    ("m1c", "<f4"), ("m2c", "<f4"), ("low_count", "<i4")):
        arr = np.ascontiguousarray(state[key], dtype=dt)
        buf.write(_blob(arr.tobytes()))
    with open(path, "wb") as f:
        f.write(buf.getvalue())


def load_checkpoint(path) -> dict:
    data = open(path, "rb").read()
    if data[:4] != CKPT_MAGIC:
        raise FileFormatError("bad checkpoint magic", offset=0)
    version, n, amp, G, it, step = struct.unpack_from("<IIIQQQ", data, 4)
    if version != CKPT_VERSION:
        raise FileFormatError(f"unsupported checkpoint version {version}", offset=4)
    off = 4 + struct.calcsize("<IIIQQQ")
    out = dict(n_dims=n, amp_mode=amp, iteration=it, adam_step=step)

    def take():
        nonlocal off
        if off + 8 > len(data):
            raise FileFormatError("truncated checkpoint", offset=off)
        (ln,) = struct.unpack_from("<Q", data, off)
        off += 8
        if off + ln > len(data):
            raise FileFormatError("truncated checkpoint", offset=off)
        b = data[off:off + ln]
        off += ln
        return b

    for key in ("config", "dataset", "rng"):
        out[key] = json.loads(take().decode())
    R = n + n * (n + 1) // 2 + 4
    for key, dt, shape in (("params", "<f4", (G, R)), ("child", "<f4", (G, R)), ("flags", "u1", (G,)),
                           ("m1p", "<f4", (G, R)), ("m2p", "<f4", (G, R)), ("m1c", "<f4", (G, R)),
                           ("m2c", "<f4", (G, R)), ("low_count", "<i4", (G,))):
        out[key] = np.frombuffer(take(), dt).reshape(shape).copy()
    if off != len(data):
        raise FileFormatError("trailing bytes after checkpoint", offset=off)
    return out
