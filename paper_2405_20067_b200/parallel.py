"""Query-batch data parallelism across the GPUs of one box.

The reference has no multi-process parallelism (its only concurrency is per-tile work inside one
process). Here one process drives one GPU:
  * the mixture is replicated (every rank runs K1/K2 on it redundantly -- it is cheap);
  * tiles are sharded: global tile i goes to rank i mod world (strided, balances candidate counts
    statistically without a global count pass);
  * each rank runs K3-K8 on its own tiles with the loss normalised by the GLOBAL batch size, so
    gradients, density statistics and the loss are plain sums over ranks;
  * ONE collective per step: all_reduce(SUM) of the flat buffer [grad_params | grad_child | stats |
    loss | pairs] (engine.GradientBuffer.flat) -- NCCL over NVLink on GPUs, gloo in CPU tests;
  * Adam then runs replicated and deterministically, keeping parameters bitwise identical.
"""
from __future__ import annotations

import numpy as np


def tile_owner(T: int, world: int) -> np.ndarray:
    """Rank that owns each global tile (strided assignment)."""
    return np.arange(T) % world


def shard_tiles(T: int, rank: int, world: int) -> np.ndarray:
    """Global tile indices owned by `rank`, ascending."""
    if not 0 <= rank < world:
        raise ValueError("rank out of range")
    return np.arange(rank, T, world)


def shard_queries(queries, targets, tile_size: int, rank: int, world: int):
    """This rank's queries/targets (contiguous tiles of tile_size, in global tile order)."""
    B = queries.shape[0]
    if B % tile_size:
        raise ValueError("batch size must be a multiple of tile_size (SPEC.md:441-442)")
    T = B // tile_size
    tiles = shard_tiles(T, rank, world)
    rows = (tiles[:, None] * tile_size + np.arange(tile_size)[None, :]).reshape(-1)
    return queries[rows], (None if targets is None else targets[rows]), tiles


def make_allreduce(group=None):
    """The step's single collective: in-place SUM of the flat gradient/statistics buffer."""
    import torch.distributed as dist

    def allreduce(flat):
        dist.all_reduce(flat, op=dist.ReduceOp.SUM, group=group)
    return allreduce
