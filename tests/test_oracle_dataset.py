"""Pins of oracle/dataset.py (O9 duplicate analysis / dedup, O10 top-k score):
the SPEC worked examples, brute-force pairwise
comparison, and invariants."""
import numpy as np
import pytest

from oracle import dataset as D


def _store(rng, n, planted):
    """n random feature matrices [n, 25, 22]; `planted` = list of (dst, src)
    copies that create duplicates."""
    X = rng.random((n, 25, 22)).astype(np.float32)
    for dst, src in planted:
        X[dst] = X[src]
    return X


# ---------------------------------------------------------------- SPEC examples
def test_spec_duplicate_rate_examples():
    rng = np.random.default_rng(0)
    # S:228 "10 records, 2 identical pairs (8 distinct) -> 0.2"
    X = _store(rng, 10, [(3, 1), (9, 6)])
    rate, distinct = D.duplicate_rate(X)
    assert distinct == 8 and rate == pytest.approx(0.2, abs=0)
    # S:229 "all distinct -> 0.0"
    assert D.duplicate_rate(_store(rng, 10, []))[0] == 0.0


def test_spec_dedup_examples():
    rng = np.random.default_rng(1)
    X = _store(rng, 4, [(2, 0)])
    # S:237 duplicates with labels {0.5, 0.9} -> one sample with label 0.9
    keep, lab, n = D.dedup_labels(X, np.array([0, 4]), np.array([0.5, 0.3, 0.9, 1.0], np.float32))
    assert n == 3 and keep.tolist() == [True, True, False, True]
    assert lab[0] == np.float32(0.9) and lab[2] == np.float32(0.9)
    # S:238 no duplicates -> unchanged
    Y = _store(rng, 5, [])
    y = np.linspace(0.2, 1.0, 5).astype(np.float32)
    keep, lab, n = D.dedup_labels(Y, np.array([0, 5]), y)
    assert n == 5 and keep.all() and np.array_equal(lab, y)
    # S:239 duplicates with equal labels -> one sample, same label
    keep, lab, n = D.dedup_labels(X, np.array([0, 4]), np.array([0.7, 0.3, 0.7, 1.0], np.float32))
    assert n == 3 and lab[0] == np.float32(0.7)


def test_dedup_never_crosses_groups():
    rng = np.random.default_rng(2)
    X = _store(rng, 6, [(4, 1)])  # identical matrices in different groups
    keep, _, n = D.dedup_labels(X, np.array([0, 3, 6]), np.ones(6, np.float32))
    assert n == 6 and keep.all()
    keep, _, n = D.dedup_labels(X, np.array([0, 6]), np.ones(6, np.float32))
    assert n == 5 and not keep[4]


def test_spec_topk_score_examples():
    lat = np.array([2.0, 4.0, 8.0])
    off = np.array([0, 3])
    w = np.array([2.0])
    # S:450 the model ranks the latency-4 program first -> top-1 = (2*2)/(4*2) = 0.5
    s = np.array([0.1, 0.9, 0.5], np.float32)
    assert D.topk_score(s, lat, off, w, 1) == 0.5
    # S:451 perfect model -> 1.0
    assert D.topk_score(-lat.astype(np.float32), lat, off, w, 1) == 1.0
    # S:452 k = 2 with top-2 = {4, 2} -> 1.0
    s2 = np.array([0.8, 0.9, 0.1], np.float32)
    assert D.topk_score(s2, lat, off, w, 2) == 1.0


# ---------------------------------------------------------------- brute force / invariants
def test_classes_equal_bruteforce_pairwise():
    rng = np.random.default_rng(3)
    X = _store(rng, 40, [(5, 2), (9, 2), (17, 11), (30, 29), (39, 0)])
    X[20] = X[21]
    X[20, 24, 21] = np.nextafter(X[20, 24, 21], 2)  # one ulp apart in the last element: distinct
    off = np.array([0, 13, 27, 40])
    rep = D.feature_classes(X, off)
    g = np.searchsorted(off, np.arange(40), side="right") - 1
    for i in range(40):
        same = [j for j in range(40) if g[j] == g[i] and np.array_equal(X[j].view(np.uint32), X[i].view(np.uint32))]
        assert rep[i] == min(same)
    assert rep[20] == 20 and rep[21] == 21


def test_duplicate_rate_permutation_invariant():
    rng = np.random.default_rng(4)
    X = _store(rng, 50, [(i + 25, i) for i in range(0, 25, 3)])
    r0 = D.duplicate_rate(X)
    perm = rng.permutation(50)
    assert D.duplicate_rate(X[perm]) == r0


def test_topk_score_properties():
    rng = np.random.default_rng(5)
    off = np.array([0, 7, 7, 20, 21, 60])  # includes an empty and a 1-element group
    lat = rng.uniform(1, 10, 60)
    w = rng.integers(1, 5, 5).astype(np.float64)
    s = rng.normal(size=60).astype(np.float32)
    prev = 0.0
    for k in (1, 2, 5, 40, 100):  # k beyond every group clamps to the group
        v = D.topk_score(s, lat, off, w, k)
        assert 0.0 < v <= 1.0 and v >= prev
        prev = v
    assert prev == 1.0
