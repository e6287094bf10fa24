"""O8: data-parallel emulation of one training step over R ranks, in-process.
TEST INFRASTRUCTURE.

SURVEY §8(c) O8 / §8(e): whole groups are assigned to ranks (a seeded
permutation dealt round-robin) so LambdaRank pairs never cross ranks.  Each rank
counts its per-task strict pairs; the counts are summed (the C-0 allreduce);
each rank scales its dL/ds by 1/P_t (global) BEFORE backward; the parameter
gradients are summed (the C-1 allreduce); one Adam step follows.  The result
must equal the unsharded step.
"""
from __future__ import annotations

from typing import List, Tuple

import numpy as np

from .rank_loss import mtl_lambdarank, strict_pair_counts
from .model import Config, backward, flatten, forward, unflatten


def assign_groups(n_groups: int, R: int, seed: int) -> List[np.ndarray]:
    perm = np.random.default_rng(seed).permutation(n_groups)
    return [np.sort(perm[r::R]) for r in range(R)]


def _gather(X, labels, group_off, groups):
    xs, ys, off = [], [], [0]
    for g in groups:
        lo, hi = int(group_off[g]), int(group_off[g + 1])
        xs.append(X[lo:hi]); ys.append(labels[lo:hi]); off.append(off[-1] + hi - lo)
    return np.concatenate(xs), np.concatenate(ys), np.asarray(off, np.int64)


def full_grad(cfg: Config, flat: np.ndarray, X, labels, group_off, pair_counts=None):
    p = unflatten(cfg, flat)
    s, acts = forward(cfg, p, X, save=True)
    loss, g = mtl_lambdarank(s, labels, group_off, pair_counts)
    return loss, flatten(cfg, backward(cfg, p, acts, g))


def dp_emulate(cfg: Config, flat: np.ndarray, X, labels, group_off, R: int,
               seed: int = 0) -> Tuple[float, np.ndarray]:
    """Sum over ranks of (loss, grad) with the global pair count; equals
    full_grad(...) on the unsharded batch."""
    labels = np.asarray(labels, np.float64)
    if labels.ndim == 1:
        labels = labels[:, None]
    parts = assign_groups(len(group_off) - 1, R, seed)
    shards = [_gather(X, labels, group_off, gs) for gs in parts]
    P = sum(strict_pair_counts(y, off) for _, y, off in shards)   # C-0 allreduce
    loss, grad = 0.0, np.zeros_like(flat, dtype=np.float64)
    for x, y, off in shards:
        l, g = full_grad(cfg, flat, x, y, off, P)
        loss += l
        grad += g                                                    # C-1 allreduce
    return loss, grad
