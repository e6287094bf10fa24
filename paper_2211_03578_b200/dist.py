"""Host-side data-parallel layout; no arithmetic of the method.

Scoring shards candidates contiguously across ranks with boundaries at
multiples of 5 (one fused-kernel tile = 5 candidates), which keeps every
candidate in the same tile slot as in a single-GPU run (batch invariance,
R34) so the merged sharded top-k equals the single-GPU top-k bit for bit.
Training assigns whole groups (subgraphs) to ranks so LambdaRank pairs never
cross ranks; the per-task strict-pair counts and the gradients are summed by
the library's NCCL allreduces.
"""
from __future__ import annotations

from typing import List, Sequence, Tuple

import numpy as np

TILE = 5  # candidates per fused-kernel tile


def shard_range(n: int, world: int, rank: int, align: int = TILE) -> Tuple[int, int]:
    """[lo, hi) of rank's contiguous shard of n candidates; lo is a multiple of
    `align`, shards differ in size by at most `align`, and they tile [0, n)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    units = -(-n // align)
    base, extra = divmod(units, world)
    lo_u = rank * base + min(rank, extra)
    hi_u = lo_u + base + (1 if rank < extra else 0)
    return min(n, lo_u * align), min(n, hi_u * align)


def shard_subgraphs(n_subgraphs: int, world: int, rank: int) -> Tuple[int, int]:
    """[lo, hi) of rank's contiguous block of subgraphs for the sharded tuning
    round (NEXT-1): a rank sets its block with id_base = lo, so every random
    draw (counter = global subgraph id, R44) and hence every survivor equals
    the unsharded run's; no collective on the data path."""
    return shard_range(n_subgraphs, world, rank, align=1)


def local_task_off(task_off: Sequence[int], lo: int, hi: int) -> np.ndarray:
    """Task segment offsets restricted to the shard [lo, hi), rebased to 0."""
    t = np.asarray(task_off, np.int64)
    return np.clip(t, lo, hi) - lo


def assign_groups(group_off: Sequence[int], world: int, seed: int = 0) -> List[np.ndarray]:
    """Whole groups dealt to ranks from a seeded permutation, balancing items:
    each group goes to the rank with the fewest items so far (ties -> lower
    rank).  Returns the sorted group ids of every rank."""
    off = np.asarray(group_off, np.int64)
    sizes = np.diff(off)
    order = np.random.default_rng(seed).permutation(len(sizes))
    load = np.zeros(world, np.int64)
    out: List[list] = [[] for _ in range(world)]
    for g in order:
        r = int(np.argmin(load))
        out[r].append(int(g))
        load[r] += sizes[g]
    return [np.sort(np.asarray(o, np.int64)) for o in out]


def gather_groups(group_off: Sequence[int], groups: Sequence[int]) -> Tuple[np.ndarray, np.ndarray]:
    """Row indices of the selected groups (in order) and their new offsets."""
    off = np.asarray(group_off, np.int64)
    rows = [np.arange(off[g], off[g + 1]) for g in groups]
    sizes = [off[g + 1] - off[g] for g in groups]
    new_off = np.zeros(len(groups) + 1, np.int64)
    if sizes:
        new_off[1:] = np.cumsum(sizes)
    return (np.concatenate(rows) if rows else np.zeros(0, np.int64)), new_off
