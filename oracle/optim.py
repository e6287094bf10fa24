"""O7: Adam with bias correction (torch.optim.Adam semantics; the paper names no
optimizer, R23 / S:356: lr 1e-3, betas (0.9, 0.999), eps 1e-8).
TEST INFRASTRUCTURE.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass
class AdamState:
    m: np.ndarray
    v: np.ndarray
    t: int = 0

    @staticmethod
    def zeros(n: int) -> "AdamState":
        return AdamState(np.zeros(n), np.zeros(n), 0)


def adam_step(param: np.ndarray, grad: np.ndarray, st: AdamState, lr: float = 1e-3,
              beta1: float = 0.9, beta2: float = 0.999, eps: float = 1e-8) -> np.ndarray:
    """One step:  m = b1 m + (1-b1) g;  v = b2 v + (1-b2) g^2;
    p -= lr * (m / (1-b1^t)) / (sqrt(v / (1-b2^t)) + eps)."""
    st.t += 1
    st.m = beta1 * st.m + (1.0 - beta1) * grad
    st.v = beta2 * st.v + (1.0 - beta2) * grad * grad
    mhat = st.m / (1.0 - beta1 ** st.t)
    vhat = st.v / (1.0 - beta2 ** st.t)
    return param - lr * mhat / (np.sqrt(vhat) + eps)
