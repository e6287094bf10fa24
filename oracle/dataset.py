"""O9 duplicate analysis / dedup and O10 the top-k score metric (SURVEY §8(f)
NEXT-2: the dataset-side steps before training and the evaluation after it).
TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

O9 (§4.3): "there are 8.56 million different schedule primitive
sequences in a total of 8.65 million tensor programs.  The repetition rate is
only 1.0430%.  Even if the features are limited to 25x22, there are 8.53
million differences ..." -- the repetition (duplicate) rate is
1 - distinct / total over the extracted feature matrices.  The
labels of the tensor programs that share a sequence collapse to their optimal
(maximum) value ("the optimal value of the labels ... can be used
as the label").

O10 (§6.1):
    top-k = sum_{m,s} min_latency_{m,s} w_{m,s}
            / sum_{m,s} min_{1<=i<=k} latency_{m,s,i} w_{m,s}
where latency_{m,s,i} is the latency of the program with the i-th largest
predicted score in group (m, s) and w_{m,s} the number of occurrences of
subgraph s in model m.

Readings (R39, R40):
  R39  two feature matrices are equal iff their fp32 bit patterns are equal
       (the encoder produces neither -0 nor NaN); duplicate classes never span
       groups (a group = one (hardware, subgraph) store); the class
       representative is its lowest index; the global duplicate rate is the
       single-group case.
  R40  "i-th largest" ranks by (score desc, index asc) exactly as the top-k
       selection (R21); k larger than a group uses the whole group.
"""
from __future__ import annotations

from typing import Tuple

import numpy as np


def feature_classes(X: np.ndarray, group_off: np.ndarray) -> np.ndarray:
    """rep[i] = lowest index j in i's group whose feature matrix has the same
    bytes as i's (R39).  X is [N, ...] float32."""
    X = np.ascontiguousarray(X, np.float32)
    N = X.shape[0]
    rows = X.reshape(N, -1)
    rep = np.empty(N, np.int64)
    for g in range(len(group_off) - 1):
        first = {}
        for i in range(int(group_off[g]), int(group_off[g + 1])):
            key = rows[i].tobytes()
            rep[i] = first.setdefault(key, i)
    return rep


def duplicate_rate(X: np.ndarray) -> Tuple[float, int]:
    """(1 - distinct / total, distinct) over all records."""
    N = X.shape[0]
    rep = feature_classes(X, np.array([0, N], np.int64))
    distinct = int((rep == np.arange(N)).sum())
    return ((N - distinct) / N if N else 0.0), distinct  # = 1 - distinct/total, exact numerator


def dedup_labels(X: np.ndarray, group_off: np.ndarray,
                 labels: np.ndarray) -> Tuple[np.ndarray, np.ndarray, int]:
    """keep[i] = i is its class representative; label_out[i] = the
    maximum label of i's class (the kept sample carries it); distinct count."""
    labels = np.asarray(labels, np.float32)
    rep = feature_classes(X, group_off)
    best = {}
    for i, r in enumerate(rep):
        best[r] = max(best.get(r, labels[i]), labels[i])
    label_out = np.array([best[r] for r in rep], np.float32)
    keep = rep == np.arange(len(rep))
    return keep, label_out, int(keep.sum())


def topk_score(scores: np.ndarray, latency: np.ndarray, group_off: np.ndarray,
               weight: np.ndarray, k: int) -> float:
    """P:384-390 top-k score in fp64 (R40 ranking and clamping)."""
    scores = np.asarray(scores, np.float32)
    latency = np.asarray(latency, np.float64)
    num = 0.0
    den = 0.0
    for g in range(len(group_off) - 1):
        lo, hi = int(group_off[g]), int(group_off[g + 1])
        if hi <= lo:
            continue
        order = sorted(range(lo, hi), key=lambda i: (-float(scores[i]) + 0.0, i))
        best_true = min(latency[lo:hi])
        best_pred = min(latency[i] for i in order[:k])
        num += best_true * float(weight[g])
        den += best_pred * float(weight[g])
    return num / den
