"""O1: the TLP tokenizer (feature extraction + post-processing).  TEST INFRASTRUCTURE.

Paper: P:215-225 (fig 3_1_feature_extraction_abstract (b)):
    f = F(p) ::= F1(tau) (F2(id) | F3(num))*
    F1: PrimitiveType -> OnehotVector, F2: NameParam -> Token, F3: Number -> Number
P:239: "For primitive types, convert it to a one-hot vector ... For numeric
parameters, leave their value unchanged.  For character parameters, convert
them into tokens ... all the features are concatenated according to the
element's original position.  After that, the extracted features are
post-processed by methods such as cropping, padding, and normalization."
P:273 / P:428: 11-wide one-hot, feature size cropped to L x E = 25 x 22.

Readings: R1 tokens 0 pad / 1 unknown / >=2 first-seen; R2 raw
scalar token; R3 per-column max-abs scale, fp32 IEEE division; R4 keep the head
when cropping; R5 numbers rounded to fp32, non-finite is an error; R6 T = 11;
R7 all-zero pad rows.  Validation covers kept data only.
"""
from __future__ import annotations

from typing import Dict, Iterable, List, Sequence, Tuple, Union

import numpy as np

PAD, UNKNOWN, FIRST = 0, 1, 2
MAX_TOKENS = 1 << 24  # R1: tokens stay exact in fp32


class TokenizeError(ValueError):
    def __init__(self, code: str, msg: str):
        super().__init__("%s: %s" % (code, msg))
        self.code = code


def build_token_table(names_in_order: Iterable[str]) -> Dict[str, int]:
    """F2's table ("We map different character parameters to different
    tokens"); R1: first-occurrence order over the training stream from 2."""
    table: Dict[str, int] = {}
    for s in names_in_order:
        if s not in table:
            if len(table) + FIRST >= MAX_TOKENS:
                raise TokenizeError("ARG", "token table exceeds 2^24 entries")
            table[s] = len(table) + FIRST
    return table


def extract_rows(seq: Sequence[Tuple[int, Sequence[Union[float, str]]]],
                 tokens: Dict[str, int], L: int, E: int, T: int) -> np.ndarray:
    """F applied to one primitive sequence, then crop + pad (un-normalised).

    Row r < min(len, L): X[r, tau] = 1 (F1), then args in original order at
    columns T.. (F2 token / F3 value), cropped to E - T slots (R4).  Rows >= len
    are zero (R7).  Only kept data is validated."""
    if len(seq) == 0:
        raise TokenizeError("EMPTY_SEQ", "empty primitive sequence")
    X = np.zeros((L, E), dtype=np.float32)
    for r in range(min(len(seq), L)):
        tau, args = seq[r]
        if not (0 <= tau < T):
            raise TokenizeError("UNKNOWN_TYPE", "type id %d >= T=%d" % (tau, T))
        X[r, tau] = 1.0
        for c in range(min(len(args), E - T)):
            a = args[c]
            if isinstance(a, str):
                v = np.float32(tokens.get(a, UNKNOWN))
            else:
                v = np.float32(a)  # R5: RN to fp32
                if not np.isfinite(np.float64(a)) or not np.isfinite(v):
                    raise TokenizeError("NONFINITE", "non-finite number argument")
            X[r, T + c] = v
    return X


def fit_scales(Xs: np.ndarray) -> np.ndarray:
    """R3: scale[c] = max over the training matrices of |X[:, :, c]|, 1.0 if 0."""
    m = np.abs(np.asarray(Xs, np.float32)).reshape(-1, Xs.shape[-1]).max(axis=0)
    return np.where(m > 0, m, np.float32(1.0)).astype(np.float32)


def encode(seqs: Sequence, tokens: Dict[str, int], scale: np.ndarray,
           L: int = 25, E: int = 22, T: int = 11) -> np.ndarray:
    """O1: fp32 [N, L, E] = extract_rows(...) / scale (element-wise IEEE fp32
    division, R3)."""
    scale = np.asarray(scale, np.float32)
    if scale.shape != (E,):
        raise TokenizeError("SHAPE", "scale must have E entries")
    out = np.zeros((len(seqs), L, E), dtype=np.float32)
    for n, seq in enumerate(seqs):
        out[n] = extract_rows(seq, tokens, L, E, T) / scale
    return out
