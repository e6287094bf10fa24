"""Pins for oracle O4 (LambdaRank), MTL masking, O5 top-k, O6 labels, O7 Adam, O8 DP."""
import itertools
import json
import math
import os

import numpy as np
import pytest
import torch

import synth
from oracle import rank_loss as LR
from oracle import model as M
from oracle import select as SEL
from oracle.dp import dp_emulate, full_grad
from oracle.optim import AdamState, adam_step

HERE = os.path.dirname(__file__)
GOLD = json.load(open(os.path.join(HERE, "golden", "lambdarank_derived.json")))


def ndcg_of_order(y, order):
    """Brute force: NDCG of the list ``order`` (position 0 = rank 1)."""
    dcg = sum((2.0 ** y[i] - 1.0) / math.log2(2.0 + r) for r, i in enumerate(order))
    ideal = sorted(y, reverse=True)
    idcg = sum((2.0 ** v - 1.0) / math.log2(2.0 + r) for r, v in enumerate(ideal))
    return dcg / max(idcg, 1e-10)


def test_pair_weight_equals_bruteforce_delta_ndcg():
    """w_ij == |NDCG(pi) - NDCG(pi with i, j swapped)| for all pairs, all n <= 6."""
    rng = np.random.default_rng(0)
    for n in range(2, 7):
        for _ in range(6):
            y = rng.choice([0.1, 0.25, 0.5, 0.8, 1.0], size=n)
            s = rng.normal(size=n)
            W = LR.pair_weights(s, y)
            order = sorted(range(n), key=lambda i: (-s[i], i))
            base = ndcg_of_order(y, order)
            for i, j in itertools.permutations(range(n), 2):
                if y[i] > y[j]:
                    sw = list(order)
                    a, b = sw.index(i), sw.index(j)
                    sw[a], sw[b] = sw[b], sw[a]
                    assert abs(W[i, j] - abs(base - ndcg_of_order(y, sw))) < 1e-13
                else:
                    assert W[i, j] == 0.0


@pytest.mark.parametrize("case", GOLD["cases"])
def test_derived_values(case):
    y, s = np.array(case["y"]), np.array(case["s"])
    assert LR.ranks(s).tolist() == case["ranks"]
    assert abs(LR.max_dcg(y) - case["max_dcg"]) < 1e-10
    W = LR.pair_weights(s, y)
    for k, v in case["w"].items():
        i, j = map(int, k.split(","))
        assert abs(W[i, j] - v) < 1e-11
    loss, grad = LR.lambdarank(s, y, np.array([0, len(y)]), reduction="sum")
    assert abs(loss - case["sum_loss"]) < 1e-11
    assert np.abs(grad - case["grad"]).max() < 1e-11
    P = LR.strict_pair_counts(y, np.array([0, len(y)]))[0]
    lm, gm = LR.lambdarank(s, y, np.array([0, len(y)]))
    assert abs(lm - case["sum_loss"] / P) < 1e-11 and np.abs(gm - np.array(case["grad"]) / P).max() < 1e-11


def test_mtl_r19_discriminating_example():
    c = GOLD["mtl_r19"]
    lab = np.array([np.nan if v is None else v for v in c["labels"]])
    loss, grad = LR.mtl_lambdarank(np.array(c["s"])[:, None], lab[:, None], np.array([0, 3]),
                                   reduction="sum")
    assert abs(loss - c["sum_loss"]) < 1e-11
    assert np.abs(grad[:, 0] - c["grad"]).max() < 1e-11
    assert abs(loss - c["all_items_reading_sum_loss"]) > 0.1


def test_ties_and_single_pair():
    loss, grad = LR.lambdarank(np.array([0.3, 0.1]), np.array([0.7, 0.7]), np.array([0, 2]))
    assert loss == 0.0 and not grad.any()
    y = np.array([1.0, 0.5])
    W = LR.pair_weights(np.zeros(2), y)
    loss, _ = LR.lambdarank(np.zeros(2), y, np.array([0, 2]), reduction="sum")
    assert abs(loss - W[0, 1]) < 1e-15  # log2(2) == 1


def test_loss_ordering():
    y = np.array([1.0, 0.4, 0.2])
    s = np.array([0.1, 0.5, -0.2])
    l0, _ = LR.lambdarank(s, y, np.array([0, 3]))
    s2 = s.copy(); s2[1] -= 0.05  # lower the lower-labelled item, no rank change
    l1, _ = LR.lambdarank(s2, y, np.array([0, 3]))
    assert l1 < l0


def test_lambdarank_finite_differences():
    """gradient vs central differences, min score gap > 10h, rel < 1e-5."""
    rng = np.random.default_rng(1)
    h = 1e-6
    off = np.array([0, 8, 13, 20])
    for _ in range(5):
        s = np.sort(rng.permutation(20) * 0.01 + rng.uniform(0, 0.001, 20))
        s = rng.permutation(s)
        y = rng.uniform(0.05, 1.0, 20)
        _, g = LR.lambdarank(s, y, off)
        for i in range(20):
            e = np.zeros(20); e[i] = h
            fd = (LR.lambdarank(s + e, y, off)[0] - LR.lambdarank(s - e, y, off)[0]) / (2 * h)
            assert abs(fd - g[i]) <= 1e-5 * max(abs(fd), 1e-4)


def test_mtl_masking_and_additivity():
    cfg = M.Config(L=6, E=8, T=3, hidden=16, up_dims=(16,), attn_heads=4, head_dim=8, n_tasks=3)
    shapes = M.param_shapes(cfg)
    p = {n: v for (n, _), v in zip(shapes, synth.init_params(2, shapes, bf16=False))}
    X = np.random.default_rng(3).normal(size=(12, cfg.L, cfg.E))
    off = np.array([0, 5, 12])
    lab = np.random.default_rng(4).uniform(0.1, 1, (12, 3))
    lab[:, 0] = np.nan  # task 0 absent everywhere -> its head gets exactly 0
    s, acts = M.forward(cfg, p, X, save=True)
    loss, g = LR.mtl_lambdarank(s, lab, off)
    assert not g[:, 0].any()
    grads = M.backward(cfg, p, acts, g)
    for k in ("W1", "c1", "w2", "c2"):
        assert not grads["head0." + k].any()
    # Shared-gradient additivity: grad(L1 + L2) == grad(L1) + grad(L2).
    g1 = g.copy(); g1[:, 2] = 0
    g2 = g.copy(); g2[:, 1] = 0
    a = M.flatten(cfg, grads)
    b = M.flatten(cfg, M.backward(cfg, p, acts, g1)) + M.flatten(cfg, M.backward(cfg, p, acts, g2))
    assert np.abs(a - b).max() < 1e-12 * np.abs(a).max()
    # One task reduces to single-task.
    l1, gg1 = LR.mtl_lambdarank(s[:, 1:2], lab[:, 1:2], off)
    l1s, gg1s = LR.lambdarank(s[:, 1], lab[:, 1], off)
    assert l1 == l1s and np.array_equal(gg1[:, 0], gg1s)


def test_head_separation():
    cfg = M.Config(L=6, E=8, T=3, hidden=16, up_dims=(16,), attn_heads=4, head_dim=8, n_tasks=3)
    shapes = M.param_shapes(cfg)
    p = {n: v for (n, _), v in zip(shapes, synth.init_params(5, shapes, bf16=False))}
    X = np.random.default_rng(6).normal(size=(4, cfg.L, cfg.E))
    s0 = M.forward(cfg, p, X)
    p["head1.W1"] += 0.5
    s1 = M.forward(cfg, p, X)
    assert np.array_equal(s0[:, [0, 2]], s1[:, [0, 2]]) and not np.array_equal(s0[:, 1], s1[:, 1])


def test_topk_equals_full_sort_and_merge():
    rng = np.random.default_rng(7)
    scores = rng.choice(np.float32([-1, -0.0, 0.0, 0.5, 2, 3]), size=300).astype(np.float32)
    off = np.array([0, 10, 10, 150, 300])
    idx, val = SEL.topk(scores, off, 16)
    for t in range(4):
        lo, hi = off[t], off[t + 1]
        order = sorted(range(lo, hi), key=lambda i: (-(scores[i] + 0.0), i))[:16]
        assert idx[t, :len(order)].tolist() == order
        assert np.all(idx[t, len(order):] == -1) and np.all(np.isneginf(val[t, len(order):]))
    # shard merge: per-shard top-k with global indices, merged, == unsharded
    for R in (2, 4, 8):
        cuts = np.linspace(0, 300, R + 1).astype(int)
        cand = [[] for _ in range(4)]
        for r in range(R):
            lo, hi = cuts[r], cuts[r + 1]
            loc = np.clip(off, lo, hi) - lo
            i2, v2 = SEL.topk(scores[lo:hi], loc, 16, base=lo)
            for t in range(4):
                cand[t] += [(float(v), int(i)) for v, i in zip(v2[t], i2[t]) if i >= 0]
        for t in range(4):
            m = sorted(cand[t], key=lambda c: (-(c[0] + 0.0), c[1]))[:16]
            assert [i for _, i in m] == [i for i in idx[t] if i >= 0]
    with pytest.raises(ValueError):
        SEL.topk(np.array([0.0, np.nan], np.float32), np.array([0, 2]), 1)


def test_normalize_labels():
    lab = SEL.normalize_labels(np.array([2e-3, 4e-3, 8e-3]), np.array([0, 3]))
    assert lab.tolist() == [1.0, 0.5, 0.25]
    b = synth.generate(1, 500)
    off = np.array([0, 100, 101, 350, 500])
    lat = synth.latencies(b, off, 3)
    lab = SEL.normalize_labels(lat, off)
    assert np.all(lab > 0) and np.all(lab <= 1)
    for g in range(4):
        assert lab[off[g]:off[g + 1]].max() == 1.0


def test_adam_matches_torch():
    rng = np.random.default_rng(8)
    p0 = rng.normal(size=50)
    grads = [rng.normal(size=50) for _ in range(5)]
    tp = torch.tensor(p0.copy(), requires_grad=True)
    opt = torch.optim.Adam([tp], lr=1e-3, betas=(0.9, 0.999), eps=1e-8)
    st = AdamState.zeros(50)
    p = p0.copy()
    for g in grads:
        tp.grad = torch.tensor(g)
        opt.step()
        p = adam_step(p, g, st)
    assert np.abs(p - tp.detach().numpy()).max() < 1e-15


@pytest.mark.parametrize("R", [2, 4])
def test_dp_emulation_equals_unsharded(R):
    cfg = M.Config(L=6, E=8, T=3, hidden=16, up_dims=(16,), attn_heads=4, head_dim=8, n_tasks=2)
    shapes = M.param_shapes(cfg)
    flat = np.concatenate([v.ravel() for v in synth.init_params(9, shapes, bf16=False)])
    rng = np.random.default_rng(10)
    off = np.array([0, 6, 9, 17, 20, 28, 33])
    X = rng.normal(size=(33, cfg.L, cfg.E))
    lab = rng.uniform(0.05, 1, (33, 2))
    lab[rng.random(33) < 0.6, 0] = np.nan  # MTL: target labels sparse
    l_full, g_full = full_grad(cfg, flat, X, lab, off)
    l_dp, g_dp = dp_emulate(cfg, flat, X, lab, off, R, seed=R)
    assert abs(l_full - l_dp) < 1e-12 * abs(l_full)
    assert np.abs(g_full - g_dp).max() < 1e-12 * np.abs(g_full).max()


# ---------------------------------------------------------------- NEXT-3: MSE
def test_mse_spec_examples():
    from oracle.rank_loss import mtl_mse
    # S:305 scores [0.5], labels [1.0] -> 0.25
    assert mtl_mse(np.array([0.5]), np.array([1.0]))[0] == 0.25
    # S:306 scores == labels -> 0.0
    y = np.array([0.3, 0.7, 1.0])
    assert mtl_mse(y, y)[0] == 0.0
    # S:392 labels [None, 0.5], preds [0.3, 0.5], MSE both tasks -> 0.0 (one sample, two tasks)
    loss, g = mtl_mse(np.array([[0.3, 0.5]]), np.array([[np.nan, 0.5]]))
    assert loss == 0.0 and g[0, 0] == 0.0
    # S:393 labels [1.0, None], preds [0.5, 0.9] -> 0.25
    assert mtl_mse(np.array([[0.5, 0.9]]), np.array([[1.0, np.nan]]))[0] == 0.25


def test_mse_gradient_finite_differences():
    from oracle.rank_loss import mtl_mse
    rng = np.random.default_rng(0)
    s = rng.normal(size=(13, 3))
    y = rng.uniform(0.1, 1.0, (13, 3))
    y[rng.random((13, 3)) < 0.3] = np.nan
    _, g = mtl_mse(s, y)
    h = 1e-6
    for i in range(13):
        for t in range(3):
            sp, sm = s.copy(), s.copy()
            sp[i, t] += h
            sm[i, t] -= h
            fd = (mtl_mse(sp, y)[0] - mtl_mse(sm, y)[0]) / (2 * h)
            assert abs(fd - g[i, t]) <= 1e-7 * max(1.0, abs(fd))
            if np.isnan(y[i, t]):
                assert g[i, t] == 0.0  # S:394 masked task: exactly zero gradient
