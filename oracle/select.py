"""O5 top-k and O6 label normalisation.  TEST INFRASTRUCTURE.

O5: "the auto-tuner obtains the prediction score through the cost model
and screens out the top-k potential candidates ... according to the prediction
score"; "the i-th largest value of the output score" (R15: higher score
= better).  R21: order by (score desc, global index asc); -0 == +0; NaN is an
error; k > segment size -> clamp and pad with (-1, -inf).

O6: "label = min_latency / latency, where min_latency refers to the
minimum value among all tensor programs of a subgraph ... The value range of
the label is (0, 1]."  R22: min over the whole group.  Computed in fp64, then
rounded to fp32.
"""
from __future__ import annotations

from typing import Tuple

import numpy as np


def topk(scores: np.ndarray, task_off: np.ndarray, k: int,
         base: int = 0) -> Tuple[np.ndarray, np.ndarray]:
    """Per task segment [task_off[t], task_off[t+1]): indices (global = base +
    local position) and values of the k best by a full stable sort."""
    scores = np.asarray(scores, np.float32)
    if np.isnan(scores).any():
        raise ValueError("NONFINITE: NaN score")
    T = len(task_off) - 1
    idx = np.full((T, k), -1, np.int64)
    val = np.full((T, k), -np.inf, np.float32)
    for t in range(T):
        lo, hi = int(task_off[t]), int(task_off[t + 1])
        items = [(-float(scores[i]) + 0.0, base + i) for i in range(lo, hi)]  # +0.0: -0 -> +0
        items.sort()
        for r, (_, i) in enumerate(items[:k]):
            idx[t, r] = i
            val[t, r] = scores[i - base]  # the score itself, bits unchanged
    return idx, val


def normalize_labels(latency: np.ndarray, group_off: np.ndarray) -> np.ndarray:
    """label_i = min_{j in g} lat_j / lat_i in fp64, rounded to fp32."""
    lat = np.asarray(latency, np.float64)
    out = np.zeros(lat.shape, np.float32)
    for g in range(len(group_off) - 1):
        lo, hi = int(group_off[g]), int(group_off[g + 1])
        if hi > lo:
            m = lat[lo:hi].min()
            out[lo:hi] = (m / lat[lo:hi]).astype(np.float32)
    return out
