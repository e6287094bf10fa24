"""O4 + MTL: LambdaRank loss and its gradient per group, float64.
TEST INFRASTRUCTURE.

Paper: "We use the Mean Square Error (MSE) loss function or the rank
loss [cao2007learning, wang2018lambdaloss]"; "lambda rank loss designed
for ranking tasks"; P:409 attention + rank is the chosen combination.  The
formula is not printed; reading R16:

  rank pi by (s desc, index asc)                                   (R17)
  D(r)   = log2(1 + r)
  maxDCG = max(sum_r (2^{y_(r)} - 1) / D(r), 1e-10)   (y sorted descending)
  G_i    = (2^{y_i} - 1) / maxDCG
  for each pair with y_i > y_j (same group):
      w_ij = |G_i - G_j| * |1/D(pi_i) - 1/D(pi_j)|     (|dNDCG|, held constant)
      l_ij = w_ij * log2(1 + exp(-sigma (s_i - s_j)))   sigma = 1
  L_task = sum l_ij / P_task  (P_task = strict pairs in the whole batch; 0 -> 0)
  dl_ij/ds_i = -(sigma / ln 2) w_ij sigmoid(-sigma (s_i - s_j)) = -dl_ij/ds_j

MTL: loss = sum over tasks with a present label; absent labels
(NaN) are ignored and, R19, ranks / maxDCG / pairs of task t use only the items
with a present label for t.
"""
from __future__ import annotations

import math
from typing import Optional, Tuple

import numpy as np

SIGMA = 1.0
LN2 = math.log(2.0)


def _log2_1p_exp_neg(z):
    """log2(1 + exp(-z)), sign-stable (R30)."""
    return (np.maximum(-z, 0.0) + np.log1p(np.exp(-np.abs(z)))) / LN2


def _sigmoid_neg(z):
    """sigmoid(-z) = 1 / (1 + exp(z)), sign-stable (R30)."""
    ez = np.exp(-np.abs(z))
    return np.where(z >= 0, ez / (1.0 + ez), 1.0 / (1.0 + ez))


def ranks(s: np.ndarray) -> np.ndarray:
    """1-based ranks by (score desc, index asc) (R17)."""
    order = sorted(range(len(s)), key=lambda i: (-s[i], i))
    r = np.empty(len(s), np.int64)
    for pos, i in enumerate(order):
        r[i] = pos + 1
    return r


def max_dcg(y: np.ndarray) -> float:
    """maxDCG = max(sum_r (2^{y_(r)} - 1) / log2(1 + r), 1e-10), y sorted desc."""
    ys = sorted(np.asarray(y, np.float64), reverse=True)
    return max(sum((2.0 ** ys[r] - 1.0) / math.log2(2.0 + r) for r in range(len(ys))), 1e-10)


def pair_weights(s: np.ndarray, y: np.ndarray) -> np.ndarray:
    """W[i, j] = |G_i - G_j| * |1/D(pi_i) - 1/D(pi_j)| where y_i > y_j, else 0."""
    s = np.asarray(s, np.float64)
    y = np.asarray(y, np.float64)
    pi = ranks(s)
    G = (np.exp2(y) - 1.0) / max_dcg(y)
    invD = 1.0 / np.log2(1.0 + pi)
    strict = y[:, None] > y[None, :]
    W = np.abs(G[:, None] - G[None, :]) * np.abs(invD[:, None] - invD[None, :])
    return np.where(strict, W, 0.0)


def group_terms(s: np.ndarray, y: np.ndarray) -> Tuple[float, np.ndarray, int]:
    """Sum of l_ij over the strict pairs of one group, d/ds of that sum, and the
    number of strict pairs.  All (i, j) pairs at once: entry [i, j] is the pair
    term for y_i > y_j."""
    s = np.asarray(s, np.float64)
    y = np.asarray(y, np.float64)
    n = len(s)
    if n == 0:
        return 0.0, np.zeros(0), 0
    W = pair_weights(s, y)
    strict = y[:, None] > y[None, :]
    Z = SIGMA * (s[:, None] - s[None, :])
    loss = float((W * _log2_1p_exp_neg(Z)).sum())
    dl_dsi = -(SIGMA / LN2) * W * _sigmoid_neg(Z)       # d l_ij / d s_i ; d/ds_j = -that
    grad = dl_dsi.sum(axis=1) - dl_dsi.sum(axis=0)
    return loss, grad, int(strict.sum())


def strict_pair_counts(labels: np.ndarray, group_off: np.ndarray) -> np.ndarray:
    """P_t: strict pairs (y_i > y_j, same group, both labels present) per task."""
    labels = np.asarray(labels, np.float64)
    if labels.ndim == 1:
        labels = labels[:, None]
    out = np.zeros(labels.shape[1], np.int64)
    for t in range(labels.shape[1]):
        for g in range(len(group_off) - 1):
            y = labels[group_off[g]:group_off[g + 1], t]
            y = y[~np.isnan(y)]
            out[t] += int((y[:, None] > y[None, :]).sum())
    return out


def lambdarank(scores: np.ndarray, labels: np.ndarray, group_off: np.ndarray,
               pair_count: Optional[float] = None, reduction: str = "mean"):
    """Single-task O4.  Returns (loss, dloss/dscores).  ``pair_count`` overrides
    P_task (used by the DP emulation, O8, where P_task is global)."""
    loss, grad = mtl_lambdarank(np.asarray(scores, np.float64)[:, None],
                                np.asarray(labels, np.float64)[:, None], group_off,
                                None if pair_count is None else np.array([pair_count]),
                                reduction)
    return loss, grad[:, 0]


def mtl_lambdarank(scores: np.ndarray, labels: np.ndarray, group_off: np.ndarray,
                   pair_counts: Optional[np.ndarray] = None, reduction: str = "mean"):
    """MTL masked loss: L = sum_t L_t over present labels (R19, R20).
    scores/labels [B, n_tasks]; NaN label = absent.  Returns (loss, grad [B, n_tasks])."""
    scores = np.asarray(scores, np.float64)
    labels = np.asarray(labels, np.float64)
    B, nt = scores.shape
    grad = np.zeros((B, nt))
    total = 0.0
    if pair_counts is None:
        pair_counts = strict_pair_counts(labels, group_off)
    for t in range(nt):
        lt = 0.0
        gt = np.zeros(B)
        for g in range(len(group_off) - 1):
            lo, hi = int(group_off[g]), int(group_off[g + 1])
            idx = np.arange(lo, hi)
            present = ~np.isnan(labels[lo:hi, t])
            idx = idx[present]
            l, gr, _ = group_terms(scores[idx, t], labels[idx, t])
            lt += l
            gt[idx] += gr
        if reduction == "mean":
            P = float(pair_counts[t])
            if P > 0:
                lt, gt = lt / P, gt / P
            else:
                lt, gt = 0.0, np.zeros(B)
        total += lt
        grad[:, t] = gt
    return total, grad


# ---------------------------------------------------------------- NEXT-3: MSE
# P:296 "We use the Mean Square Error (MSE) loss function or the rank loss";
# P:393 "the label of TLP is a normalization value in the range of (0,1], so MSE
# loss is an option"; mean of squared residuals, gradient
# 2 (score - label) / B.  MTL: sum over tasks of the
# per-task mean over its present labels; absent labels give zero loss and zero
# gradient.  R41: a task with no present label contributes 0 (as R16's P = 0).
def mse_counts(labels: np.ndarray) -> np.ndarray:
    """Present labels per task (the MSE denominator; global under DP)."""
    labels = np.asarray(labels, np.float64)
    if labels.ndim == 1:
        labels = labels[:, None]
    return (~np.isnan(labels)).sum(axis=0).astype(np.int64)


def mtl_mse(scores: np.ndarray, labels: np.ndarray, counts: Optional[np.ndarray] = None):
    """Returns (loss, grad [B, n_tasks]) of sum_t mean_{i present} (s_it - y_it)^2."""
    scores = np.asarray(scores, np.float64)
    labels = np.asarray(labels, np.float64)
    if scores.ndim == 1:
        scores, labels = scores[:, None], labels[:, None]
    B, nt = scores.shape
    if counts is None:
        counts = mse_counts(labels)
    grad = np.zeros((B, nt))
    total = 0.0
    for t in range(nt):
        n = float(counts[t])
        if n == 0:
            continue
        for i in range(B):
            if np.isnan(labels[i, t]):
                continue
            r = scores[i, t] - labels[i, t]
            total += r * r / n
            grad[i, t] = 2.0 * r / n
    return total, grad
