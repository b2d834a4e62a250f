"""gmm-core types on the device (reference module gmm-core).

A ``Mixture`` is stored as structure-of-rows float32 tensors in HBM, exactly the raw layouts of
SPEC.md:28-50 (mean_raw | chol_raw | color_raw | amp_raw, chol_raw in the row-major lower packing
of SPEC.md:31), plus one flag byte per component (bit0 = live child, bit1 = frozen).
Evaluated Gaussians use the fixed index space e = i (parent i) and e = G + i (child of i).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

BRIGHTNESS = 0
OPACITY = 1
FLAG_CHILD = 1
FLAG_FROZEN = 2


def n_chol(n: int) -> int:
    return n * (n + 1) // 2


def tri(i: int, j: int) -> int:
    """Row-major lower packing index."""
    return i * (i + 1) // 2 + j


def raw_width(n: int) -> int:
    return n + n_chol(n) + 4


def raw_slices(n: int):
    """(mean, chol, color, amp) column slices of a raw row."""
    p = n_chol(n)
    return slice(0, n), slice(n, n + p), slice(n + p, n + p + 3), n + p + 3


def default_device() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("ndgauss-b200 needs a CUDA device (no CPU fallback)")
    return torch.device("cuda", torch.cuda.current_device())


@dataclass
class Mixture:
    """Ordered components with parent/child links and frozen flags."""
    n_dims: int
    amp_mode: int
    params: torch.Tensor        # [G, R] float32, device
    child: torch.Tensor         # [G, R] float32, device (rows of components without a child unused)
    flags: torch.Tensor         # [G] uint8, device
    children_live: bool = False  # host mirror of "any component has a live child" (sizes Gev = 2G)

    @classmethod
    def from_arrays(cls, n_dims, amp_mode, params, child=None, has_child=None, frozen=None, device=None):
        device = device or default_device()
        params = np.asarray(params, dtype=np.float32)
        if params.ndim != 2 or params.shape[1] != raw_width(n_dims):
            raise ValueError(f"params must be [G, {raw_width(n_dims)}]")
        G = params.shape[0]
        child = np.zeros_like(params) if child is None else np.asarray(child, dtype=np.float32)
        hc = np.zeros(G, bool) if has_child is None else np.asarray(has_child, bool)
        fr = np.zeros(G, bool) if frozen is None else np.asarray(frozen, bool)
        flags = hc.astype(np.uint8) * FLAG_CHILD | fr.astype(np.uint8) * FLAG_FROZEN
        return cls(n_dims, int(amp_mode), torch.from_numpy(params).to(device), torch.from_numpy(child).to(device),
                   torch.from_numpy(flags).to(device), bool(np.any(hc & ~fr)))

    @property
    def G(self) -> int:
        return int(self.params.shape[0])

    @property
    def Gev(self) -> int:
        return 2 * self.G if self.children_live else self.G

    @property
    def device(self):
        return self.params.device

    def has_child(self) -> np.ndarray:
        return (self.flags.cpu().numpy() & FLAG_CHILD).astype(bool)

    def frozen(self) -> np.ndarray:
        return (self.flags.cpu().numpy() & FLAG_FROZEN).astype(bool)

    def numpy(self):
        return dict(n_dims=self.n_dims, amp_mode=self.amp_mode, params=self.params.cpu().numpy(),
                    child=self.child.cpu().numpy(), has_child=self.has_child(), frozen=self.frozen())

    def clone(self) -> "Mixture":
        return Mixture(self.n_dims, self.amp_mode, self.params.clone(), self.child.clone(), self.flags.clone(),
                       self.children_live)
