"""GPU parity: the CUDA path (through the C-ABI) against the CPU oracle on the same
seeded inputs.  Tokenizer, top-k and labels bit-exact; fp32 path within 1e-5
(R25 norm-wise); bf16 path within 1e-2."""
import json
import os
import re

import numpy as np
import pytest
import torch

import synth
import oracle
from oracle import model as OM
from oracle import rank_loss as OLR
from oracle.optim import AdamState, adam_step

from helpers import (encoded_batch, fit_scales, flat_params, grad_mismatches, oracle_cfg, product_cfg,
                     rel_err, token_table)

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(__file__)
# Gradients that are identically zero in exact arithmetic, so both sides are
# rounding noise: attn*.bk (q . bk shifts a whole softmax row) and head*.c2
# (adds L c2 to every score of a group; LambdaRank is shift invariant, so
# sum_i dL/ds_i = 0 per group).
ZERO_GRAD = re.compile(r"(attn\d+\.bk|head\d+\.c2)$")
# head*.c1: dc1[k] = sum_{n,l} g_n w2[k] [u>0] cancels almost completely for the
# same reason (rows active in every candidate contribute g_n * const), so it is
# compared against the magnitude of the summed terms (summation error bound).
CANCEL_GRAD = re.compile(r"head(\d+)\.c1$")


@pytest.fixture(scope="module")
def tp():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_2211_03578_b200 as tp
    tp._lib.load()
    return tp


@pytest.fixture(scope="module")
def tokscale():
    tokens = token_table()
    return tokens, fit_scales(tokens)


def make_encoder(tp, tokens, scale, **kw):
    cfg = tp.TLPConfig(precision="fp32", **kw)
    m = tp.TLP(cfg)
    m.set_token_table(sorted(tokens, key=tokens.get))
    m.set_norm_scales(scale)
    return m


# ---------------------------------------------------------------- tokenizer
def test_encode_bit_exact(tp, tokscale):
    tokens, scale = tokscale
    m = make_encoder(tp, tokens, scale)
    b = synth.generate(5, 3001, unseen_rate=0.05)
    X_ref = oracle.encode(b.to_lists(), tokens, scale)
    X = m.encode(tp.DeviceBatch.from_packed(b))
    m.sync()
    assert np.array_equal(X.cpu().numpy().view(np.uint32), X_ref.view(np.uint32))


def test_encode_worked_example_bits(tp):
    g = json.load(open(os.path.join(HERE, "golden", "tokenizer_worked_example.json")))
    reg = {n: i for i, n in enumerate(g["registry"])}
    seq = [(reg[t], [a if isinstance(a, str) else float(a) for a in args]) for t, args in g["sequence"]]
    tokens = g["tokens"]
    scale = np.ones(22, np.float32)
    for c, v in g["scales_nonunit"].items():
        scale[int(c)] = v
    m = make_encoder(tp, tokens, scale)
    X = m.encode(tp.DeviceBatch.from_packed(synth.pack([seq]))).cpu().numpy()[0]
    m.sync()
    for rc, bits in g["normalized_bits_nonunit"].items():
        r, c = map(int, rc.split(","))
        assert "0x%08X" % X[r, c].view(np.uint32) == bits


@pytest.mark.parametrize("bad,code", [
    ([[(0, [1.0])], []], "ERR_EMPTY_SEQ"),
    ([[(11, [1.0])]], "ERR_UNKNOWN_TYPE"),
    ([[(2, [float("nan")])]], "ERR_NONFINITE"),
    ([[(2, [1e300])]], "ERR_NONFINITE"),
])
def test_encode_device_errors(tp, tokscale, bad, code):
    tokens, scale = tokscale
    m = make_encoder(tp, tokens, scale)
    m.encode(tp.DeviceBatch.from_packed(synth.pack(bad)))
    with pytest.raises(tp.TLPError) as e:
        m.sync()
    assert e.value.code == code
    # kept-data-only validation: junk beyond the crop raises nothing
    ok = [[(0, [1.0] * 11 + [float("nan")])] + [(0, [])] * 24 + [(99, [float("inf")])]]
    m.encode(tp.DeviceBatch.from_packed(synth.pack(ok)))
    m.sync()


# ---------------------------------------------------------------- top-k / labels
def test_topk_bit_exact(tp):
    m = tp.TLP(tp.TLPConfig(precision="fp32"))
    rng = np.random.default_rng(3)
    sizes = [0, 1, 5, 16, 17, 2047, 2048, 2049, 4096, 9000, 300]
    off = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    N = int(off[-1])
    # many ties, signed zeros
    s = rng.choice(np.float32([-2.0, -0.0, 0.0, 0.25, 1.0, 3.5]), size=N).astype(np.float32)
    mask = rng.random(N) < 0.5
    s[mask] = rng.normal(size=int(mask.sum())).astype(np.float32)
    cols = np.stack([rng.normal(size=N).astype(np.float32), s], axis=1)  # stride 2, head 1
    for k in (1, 16, 100, 1024):
        idx_ref, val_ref = oracle.topk(cols[:, 1], off, k, base=7)
        idx, val = m.topk(torch.from_numpy(cols).cuda(), off, k, head=1, shard_base=7)
        m.sync()
        assert np.array_equal(idx.cpu().numpy(), idx_ref), k
        assert np.array_equal(val.cpu().numpy().view(np.uint32), val_ref.view(np.uint32)), k


def test_topk_nan_is_an_error(tp):
    m = tp.TLP(tp.TLPConfig(precision="fp32"))
    s = torch.tensor([[0.0], [float("nan")]], device="cuda")
    m.topk(s, np.array([0, 2]), 1)
    with pytest.raises(tp.TLPError) as e:
        m.sync()
    assert e.value.code == "ERR_NONFINITE"


def test_normalize_labels_bit_exact(tp):
    m = tp.TLP(tp.TLPConfig(precision="fp32"))
    sizes = list(synth.group_sizes(4, 3, lo=24, hi=4000, mean=1600)) + [1, 0, 2]
    off = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    b = synth.generate(2, int(off[-1]))
    lat = synth.latencies(b, off, 7).astype(np.float32)
    ref = oracle.normalize_labels(lat, off)
    out = m.normalize_labels(torch.from_numpy(lat).cuda(), off)
    m.sync()
    assert np.array_equal(out.cpu().numpy().view(np.uint32), ref.view(np.uint32))


# ---------------------------------------------------------------- fp32 forward
FWD_CASES = {
    "tiny_C1": dict(hidden=64, up=(32, 64), head_dim=32),
    "paper_1layer": dict(),
    "paper_2layer": dict(n_attn=2),
    "mtl4": dict(n_tasks=4),
}


@pytest.mark.parametrize("name", list(FWD_CASES))
def test_forward_fp32_parity(tp, tokscale, name):
    tokens, scale = tokscale
    ocfg = oracle_cfg(**FWD_CASES[name])
    flat = flat_params(ocfg, seed=11)
    _, X = encoded_batch(21, 37, tokens, scale)  # 925 rows: 7 full 128-row tiles + tail
    ref = OM.forward(ocfg, OM.unflatten(ocfg, flat), X)
    m = tp.TLP(product_cfg(ocfg, "fp32"))
    m.set_params(flat.astype(np.float32))
    s = m.score(torch.from_numpy(X).cuda())
    m.sync()
    assert rel_err(s.cpu().numpy(), ref) <= 1e-5


def test_score_batch_invariance(tp, tokscale):
    tokens, scale = tokscale
    ocfg = oracle_cfg()
    flat = flat_params(ocfg, seed=12)
    _, X = encoded_batch(22, 300, tokens, scale)
    m = tp.TLP(product_cfg(ocfg, "fp32"))
    m.set_params(flat.astype(np.float32))
    Xd = torch.from_numpy(X).cuda()
    full = m.score(Xd).cpu().numpy()
    part = m.score(Xd[113:250].contiguous()).cpu().numpy()
    m.sync()
    assert np.array_equal(full[113:250].view(np.uint32), part.view(np.uint32))


# ---------------------------------------------------------------- LambdaRank unit (R26)
def test_lambdarank_unit_parity(tp):
    m = tp.TLP(tp.TLPConfig(precision="fp32", n_tasks=2))
    rng = np.random.default_rng(5)
    sizes = [1, 2, 7, 64, 300, 512]
    off = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    B = int(off[-1])
    s = rng.normal(size=(B, 2)).astype(np.float32)
    y = rng.uniform(0.05, 1.0, (B, 2)).astype(np.float32)
    y[rng.random(B) < 0.3, 0] = np.nan  # MTL: absent labels
    y[:5, 1] = y[5, 1]                    # label ties -> no pairs
    loss_ref, g_ref = OLR.mtl_lambdarank(s.astype(np.float64), y.astype(np.float64), off)
    loss, g = m.lambdarank(torch.from_numpy(s).cuda(), torch.from_numpy(y).cuda(), off)
    m.sync()
    assert abs(float(loss.cpu()) - loss_ref) <= 1e-5 * abs(loss_ref)
    assert rel_err(g.cpu().numpy(), g_ref) <= 1e-5
    assert not g.cpu().numpy()[np.isnan(y)].any()


def test_lambdarank_large_groups_parity(tp):
    """Groups larger than a block (1,100 and 2,600 items: the present-label
    compaction and the pair counts take several block-wide passes; the rank
    kernels split each group over 8 CTAs) with absent labels, vs the oracle."""
    m = tp.TLP(tp.TLPConfig(precision="fp32", n_tasks=2))
    rng = np.random.default_rng(7)
    sizes = [1100, 2600, 33]
    off = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    B = int(off[-1])
    s = rng.normal(size=(B, 2)).astype(np.float32)
    y = rng.uniform(0.05, 1.0, (B, 2)).astype(np.float32)
    y[rng.random(B) < 0.3, 0] = np.nan
    loss_ref, g_ref = OLR.mtl_lambdarank(s.astype(np.float64), y.astype(np.float64), off)
    loss, g = m.lambdarank(torch.from_numpy(s).cuda(), torch.from_numpy(y).cuda(), off)
    m.sync()
    assert abs(float(loss.cpu()) - loss_ref) <= 1e-5 * abs(loss_ref)
    assert rel_err(g.cpu().numpy(), g_ref) <= 1e-5
    assert not g.cpu().numpy()[np.isnan(y)].any()


# ---------------------------------------------------------------- training (fp32)
def train_inputs(tokens, scale, n_tasks=1, seed=31, sizes=(9, 16, 12, 16, 11, 7)):
    off = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    b, X = encoded_batch(seed, int(off[-1]), tokens, scale)
    labs = []
    for t in range(n_tasks):
        lat = synth.latencies(b, off, seed + 100 * t, task_noise=0.3 * t)
        labs.append(oracle.normalize_labels(lat, off))
    y = np.stack(labs, axis=1).astype(np.float32)
    if n_tasks > 1:
        y[np.random.default_rng(seed).random(len(y)) < 0.5, 0] = np.nan
    return X, y, off


def min_rel_gap(scores, off):
    g = np.inf
    for t in range(scores.shape[1]):
        for i in range(len(off) - 1):
            s = np.sort(scores[off[i]:off[i + 1], t])
            if len(s) > 1:
                g = min(g, np.min(np.diff(s)) / max(np.abs(s).max(), 1e-30))
    return g


# (n_tasks, n_attn, weight seed, group sizes): seeds chosen so that every
# within-group score gap exceeds 2e-4 relative -- ranks are then decided far
# above fp32 noise (R26) and the oracle and the GPU rank identically.
GRAD_CASES = [(1, 1, 17, (9, 16, 12, 16, 11, 7)), (4, 1, 20, (8, 6, 9, 7, 10, 8)),
              (1, 2, 14, (9, 16, 12, 16, 11, 7))]


@pytest.mark.parametrize("precision,tol", [("fp32", 1e-5), ("bf16", 1e-2)])
@pytest.mark.parametrize("n_tasks,n_attn,seed,sizes", GRAD_CASES)
def test_grads_parity(tp, tokscale, n_tasks, n_attn, seed, sizes, precision, tol):
    """fp32 context: SIMT FFMA everywhere (1e-5).  bf16 context: every dense
    layer / dgrad / wgrad on the tcgen05 tensor cores (bf16x3 split operands),
    attention / heads / LambdaRank SIMT fp32 (contract 1e-2)."""
    tokens, scale = tokscale
    ocfg = oracle_cfg(n_tasks=n_tasks, n_attn=n_attn, hidden=64, up=(32, 64), head_dim=32)
    flat = flat_params(ocfg, seed=seed)
    X, y, off = train_inputs(tokens, scale, n_tasks, sizes=sizes)
    p = OM.unflatten(ocfg, flat)
    s_ref, acts = OM.forward(ocfg, p, X, save=True)
    assert min_rel_gap(s_ref, off) > 2e-4
    loss_ref, g = OLR.mtl_lambdarank(s_ref, y.astype(np.float64), off)
    grads_ref = OM.backward(ocfg, p, acts, g)
    m = tp.TLP(product_cfg(ocfg, precision))
    m.set_params(flat.astype(np.float32))
    loss = m.compute_grads(torch.from_numpy(X).cuda(), torch.from_numpy(y).cuda(), off)
    m.sync()
    assert abs(float(loss.cpu()) - loss_ref) <= tol * abs(loss_ref)
    got = OM.unflatten(ocfg, m.get_grads().astype(np.float64))
    bad = grad_mismatches(ocfg, p, acts, g, got, grads_ref, tol)
    assert not bad, bad


def test_group_offsets_reused_and_changed(tp, tokscale):
    """The group offsets are uploaded only when they change (api.cu upload_goff):
    a step after a different layout, and the same layout again, give bitwise the
    gradients of a fresh context given that layout alone."""
    tokens, scale = tokscale
    ocfg = oracle_cfg(n_tasks=1, n_attn=1, hidden=64, up=(32, 64), head_dim=32)
    flat = flat_params(ocfg, seed=5).astype(np.float32)
    X, y, off = train_inputs(tokens, scale, 1, sizes=(9, 16, 12, 16, 11, 7))
    off2 = np.array([0, 20, 41, int(off[-1])], np.int64)
    Xd, yd = torch.from_numpy(X).cuda(), torch.from_numpy(y).cuda()

    def fresh(o):
        r = tp.TLP(product_cfg(ocfg, "fp32"))
        r.set_params(flat)
        r.compute_grads(Xd, yd, o)
        r.sync()
        return r.get_grads()

    want = {1: fresh(off), 2: fresh(off2)}
    m = tp.TLP(product_cfg(ocfg, "fp32"))
    m.set_params(flat)
    for which in (1, 1, 2, 1, 2, 2):
        o = off if which == 1 else off2
        m.compute_grads(Xd, yd, o.copy())
        m.sync()
        assert np.array_equal(m.get_grads().view(np.uint32), want[which].view(np.uint32)), which


def test_mse_unit_parity(tp):
    """NEXT-3 MSE unit (tlp_mse) vs oracle mtl_mse on MTL labels with absent tasks."""
    rng = np.random.default_rng(4)
    s = rng.normal(size=(777, 3)).astype(np.float32)
    y = rng.uniform(0.05, 1.0, (777, 3)).astype(np.float32)
    y[rng.random((777, 3)) < 0.3] = np.nan
    y[:, 2] = np.nan  # a task with no labels contributes nothing (R41)
    loss_ref, g_ref = OLR.mtl_mse(s.astype(np.float64), y.astype(np.float64))
    m = tp.TLP(tp.TLPConfig(precision="fp32", n_tasks=3, loss="mse"))
    loss, g = m.mse(torch.from_numpy(s).cuda(), torch.from_numpy(y).cuda())
    m.sync()
    assert abs(float(loss.cpu()) - loss_ref) <= 1e-6 * loss_ref
    assert rel_err(g.cpu().numpy(), g_ref) <= 1e-6
    assert not g.cpu().numpy()[np.isnan(y)].any()


@pytest.mark.parametrize("precision,tol", [("fp32", 1e-5), ("bf16", 1e-2)])
def test_grads_parity_mse(tp, tokscale, precision, tol):
    """NEXT-3: the whole training gradient with the MSE loss (cfg.loss = MSE),
    MTL with absent labels.  Only attn*.bk is identically zero here (softmax
    shift invariance, R32); c1 / c2 carry real MSE gradients."""
    tokens, scale = tokscale
    ocfg = oracle_cfg(n_tasks=2, n_attn=1, hidden=64, up=(32, 64), head_dim=32)
    flat = flat_params(ocfg, seed=23)
    X, y, off = train_inputs(tokens, scale, 2, sizes=(9, 16, 12, 16, 11, 7))
    p = OM.unflatten(ocfg, flat)
    s_ref, acts = OM.forward(ocfg, p, X, save=True)
    loss_ref, g = OLR.mtl_mse(s_ref, y.astype(np.float64))
    grads_ref = OM.backward(ocfg, p, acts, g)
    cfg = product_cfg(ocfg, precision)
    cfg.loss = "mse"
    m = tp.TLP(cfg)
    m.set_params(flat.astype(np.float32))
    loss = m.compute_grads(torch.from_numpy(X).cuda(), torch.from_numpy(y).cuda(), off)
    m.sync()
    assert abs(float(loss.cpu()) - loss_ref) <= tol * abs(loss_ref)
    got = OM.unflatten(ocfg, m.get_grads().astype(np.float64))
    bad = grad_mismatches(ocfg, p, acts, g, got, grads_ref, tol, lambdarank=False)
    assert not bad, bad


# ---------------------------------------------------------------- NEXT-3: padding mask (R42)
@pytest.mark.parametrize("precision,tol", [("fp32", 1e-5), ("bf16", 1e-2)])
def test_forward_parity_attn_mask(tp, tokscale, precision, tol):
    """Encoded TenSet-shaped candidates (most shorter than 25 primitives, so
    with padding rows) scored with the padding-key mask, 2 layers."""
    tokens, scale = tokscale
    ocfg = oracle_cfg(n_attn=2)
    ocfg.attn_mask = True
    flat = flat_params(ocfg, seed=31)
    _, X = encoded_batch(33, 301, tokens, scale)
    assert ((X == 0).all(axis=2).any(axis=1)).mean() > 0.3  # padding present
    ref = OM.forward(ocfg, OM.unflatten(ocfg, flat), X)
    cfg = product_cfg(ocfg, precision)
    cfg.attn_mask = True
    m = tp.TLP(cfg)
    m.set_params(flat.astype(np.float32))
    Xd = torch.from_numpy(X).cuda()
    s = m.score(Xd)
    m.sync()
    assert rel_err(s.cpu().numpy(), ref) <= tol
    # the mask changes the result (it is not a no-op on padded inputs)
    unmasked = OM.forward(oracle_cfg(n_attn=2), OM.unflatten(ocfg, flat), X)
    assert rel_err(unmasked, ref) > 1e-3
    if precision == "bf16":  # batch invariance holds with the mask
        part = m.score(Xd[7:300].contiguous()).cpu().numpy()
        assert np.array_equal(s.cpu().numpy()[7:300].view(np.uint32), part.view(np.uint32))


@pytest.mark.parametrize("precision,tol", [("fp32", 1e-5), ("bf16", 1e-2)])
def test_grads_parity_attn_mask(tp, tokscale, precision, tol):
    tokens, scale = tokscale
    ocfg = oracle_cfg(n_tasks=1, n_attn=1, hidden=64, up=(32, 64), head_dim=32)
    ocfg.attn_mask = True
    flat = flat_params(ocfg, seed=25)  # seed with within-group score gaps > 2e-4 (R26)
    X, y, off = train_inputs(tokens, scale, 1, sizes=(9, 16, 12, 16, 11, 7))
    p = OM.unflatten(ocfg, flat)
    s_ref, acts = OM.forward(ocfg, p, X, save=True)
    assert min_rel_gap(s_ref, off) > 2e-4
    loss_ref, g = OLR.mtl_lambdarank(s_ref, y.astype(np.float64), off)
    grads_ref = OM.backward(ocfg, p, acts, g)
    cfg = product_cfg(ocfg, precision)
    cfg.attn_mask = True
    m = tp.TLP(cfg)
    m.set_params(flat.astype(np.float32))
    loss = m.compute_grads(torch.from_numpy(X).cuda(), torch.from_numpy(y).cuda(), off)
    m.sync()
    assert abs(float(loss.cpu()) - loss_ref) <= tol * abs(loss_ref)
    got = OM.unflatten(ocfg, m.get_grads().astype(np.float64))
    bad = grad_mismatches(ocfg, p, acts, g, got, grads_ref, tol)
    assert not bad, bad


# ---------------------------------------------------------------- NEXT-3: learned positional table (R43)
@pytest.mark.parametrize("precision,tol", [("fp32", 1e-5), ("bf16", 1e-2)])
def test_forward_parity_pos_enc(tp, tokscale, precision, tol):
    tokens, scale = tokscale
    ocfg = oracle_cfg(n_attn=2)
    ocfg.pos_enc = True
    flat = flat_params(ocfg, seed=41)
    _, X = encoded_batch(43, 301, tokens, scale)
    ref = OM.forward(ocfg, OM.unflatten(ocfg, flat), X)
    m = tp.TLP(product_cfg(ocfg, precision))
    assert m.num_params == OM.n_params(ocfg)
    m.set_params(flat.astype(np.float32))
    s = m.score(torch.from_numpy(X).cuda())
    m.sync()
    assert rel_err(s.cpu().numpy(), ref) <= tol


@pytest.mark.parametrize("precision,tol", [("fp32", 1e-5), ("bf16", 1e-2)])
def test_grads_parity_pos_enc(tp, tokscale, precision, tol):
    tokens, scale = tokscale
    ocfg = oracle_cfg(n_tasks=1, n_attn=1, hidden=64, up=(32, 64), head_dim=32)
    ocfg.pos_enc = True
    ocfg.attn_mask = True
    X, y, off = train_inputs(tokens, scale, 1, sizes=(9, 16, 12, 16, 11, 7))
    for seed in range(40, 80):  # a seed with within-group score gaps > 2e-4 (R26)
        flat = flat_params(ocfg, seed=seed)
        p = OM.unflatten(ocfg, flat)
        s_ref, acts = OM.forward(ocfg, p, X, save=True)
        if min_rel_gap(s_ref, off) > 2e-4:
            break
    loss_ref, g = OLR.mtl_lambdarank(s_ref, y.astype(np.float64), off)
    grads_ref = OM.backward(ocfg, p, acts, g)
    m = tp.TLP(product_cfg(ocfg, precision))
    m.set_params(flat.astype(np.float32))
    loss = m.compute_grads(torch.from_numpy(X).cuda(), torch.from_numpy(y).cuda(), off)
    m.sync()
    assert abs(float(loss.cpu()) - loss_ref) <= tol * abs(loss_ref)
    got = OM.unflatten(ocfg, m.get_grads().astype(np.float64))
    bad = grad_mismatches(ocfg, p, acts, g, got, grads_ref, tol)
    assert not bad, bad


@pytest.mark.parametrize("mask", [False, True])
def test_grads_parity_bf16_paper_shape(tp, tokscale, mask):
    """bf16 context at the paper shape (d_h = 32): the training attention core
    runs on the tensor cores (tf32 mma.sync, k_attn_tc.cu), the dense layers on
    tcgen05 (bf16x3); the whole gradient against the fp64 oracle at 1e-2."""
    tokens, scale = tokscale
    ocfg = oracle_cfg(n_attn=1)
    ocfg.attn_mask = mask
    X, y, off = train_inputs(tokens, scale, 1, sizes=(9, 16, 12, 16, 11, 7))
    for seed in range(50, 90):  # within-group score gaps > 2e-4 (R26)
        flat = flat_params(ocfg, seed=seed)
        p = OM.unflatten(ocfg, flat)
        s_ref, acts = OM.forward(ocfg, p, X, save=True)
        if min_rel_gap(s_ref, off) > 2e-4:
            break
    loss_ref, g = OLR.mtl_lambdarank(s_ref, y.astype(np.float64), off)
    grads_ref = OM.backward(ocfg, p, acts, g)
    m = tp.TLP(product_cfg(ocfg, "bf16"))
    m.set_params(flat.astype(np.float32))
    loss = m.compute_grads(torch.from_numpy(X).cuda(), torch.from_numpy(y).cuda(), off)
    m.sync()
    assert abs(float(loss.cpu()) - loss_ref) <= 1e-2 * abs(loss_ref)
    got = OM.unflatten(ocfg, m.get_grads().astype(np.float64))
    bad = grad_mismatches(ocfg, p, acts, g, got, grads_ref, 1e-2)
    assert not bad, bad


def test_finetune_from_checkpoint(tp, tokscale):
    """NEXT-3 fine-tuning (P:518 transfer): parameters saved from one ctx
    (tlp_get_params) and loaded into a fresh ctx (tlp_set_params) continue
    training exactly like the original ctx after a re-load of the same state
    (Adam restarts, R23)."""
    tokens, scale = tokscale
    ocfg = oracle_cfg(hidden=64, up=(32, 64), head_dim=32)
    X, y, off = train_inputs(tokens, scale)
    Xd, yd = torch.from_numpy(X).cuda(), torch.from_numpy(y).cuda()
    a = tp.TLP(product_cfg(ocfg, "fp32"))
    a.set_params(flat_params(ocfg, seed=17).astype(np.float32))
    for _ in range(3):
        a.train_step(Xd, yd, off)
    ckpt = a.get_params()
    b = tp.TLP(product_cfg(ocfg, "fp32"))
    b.set_params(ckpt)
    a.set_params(ckpt)  # both restart Adam from the checkpoint
    for _ in range(2):
        a.train_step(Xd, yd, off)
        b.train_step(Xd, yd, off)
    a.sync(); b.sync()
    assert np.array_equal(a.get_params().view(np.uint32), b.get_params().view(np.uint32))
    assert not np.array_equal(a.get_params(), ckpt)


def test_train_step_adam_parity(tp, tokscale):
    tokens, scale = tokscale
    ocfg = oracle_cfg(hidden=64, up=(32, 64), head_dim=32)
    flat = flat_params(ocfg, seed=17)
    X, y, off = train_inputs(tokens, scale, 1)
    m = tp.TLP(product_cfg(ocfg, "fp32"))
    m.set_params(flat.astype(np.float32))
    st = AdamState.zeros(flat.size)
    p_ref = flat.copy()
    Xd, yd = torch.from_numpy(X).cuda(), torch.from_numpy(y).cuda()
    for _ in range(3):
        s_ref, acts = OM.forward(ocfg, OM.unflatten(ocfg, p_ref), X, save=True)
        _, g = OLR.mtl_lambdarank(s_ref, y.astype(np.float64), off)
        gflat = OM.flatten(ocfg, OM.backward(ocfg, OM.unflatten(ocfg, p_ref), acts, g))
        p_ref = adam_step(p_ref, gflat, st)
        m.train_step(Xd, yd, off)
    m.sync()
    got = m.get_params().astype(np.float64)
    # parameter change after 3 steps within 1e-5 of the oracle's change, per tensor
    d_ref = OM.unflatten(ocfg, p_ref - flat)
    d_got = OM.unflatten(ocfg, got - flat)
    bad = {}
    for name, _ in OM.param_shapes(ocfg):
        if ZERO_GRAD.search(name) or CANCEL_GRAD.search(name):
            # Adam maps a (near-)zero gradient's rounding noise to +-lr updates:
            # no meaningful comparison; bounded by 3 steps of lr.
            # |Adam step| <= lr (1-b1)/sqrt(1-b2) ~ 3.17 lr per step
            assert np.abs(d_got[name]).max() <= 3 * 3.17e-3, name
            continue
        e = rel_err(d_got[name], d_ref[name])
        if e > 1e-3:
            bad[name] = e
    assert not bad, bad


# ---------------------------------------------------------------- bf16 tcgen05 path
@pytest.mark.parametrize("N,K,a_tmem", [(16, 32, 0), (96, 64, 0), (160, 32, 0), (32, 160, 0),
                                         (256, 256, 0), (32, 160, 1), (256, 128, 1), (16, 32, 1)])
def test_umma_building_block(tp, N, K, a_tmem):
    """One tcgen05.mma chain (descriptors, TMEM, tcgen05.ld) vs an fp64 matmul of
    the same bf16-rounded operands: products are exact, accumulation fp32."""
    rng = np.random.default_rng(N * 1000 + K)
    A = synth.bf16_round(rng.normal(size=(128, K))).astype(np.float32)
    B = synth.bf16_round(rng.normal(size=(N, K))).astype(np.float32)
    D = torch.zeros((128, N), dtype=torch.float32, device="cuda")
    lib = tp._lib.load()
    Ad, Bd = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()  # keep alive until sync
    st = lib.tlp_debug_umma(Ad.data_ptr(), Bd.data_ptr(), D.data_ptr(), N, K, a_tmem,
                            torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    assert st == 0
    ref = A.astype(np.float64) @ B.astype(np.float64).T
    assert rel_err(D.cpu().numpy(), ref) <= 1e-5


BF16_CASES = {"paper_1layer": dict(), "paper_2layer": dict(n_attn=2), "mtl4": dict(n_tasks=4),
              "no_res": dict(n_res=0), "no_attn": dict(n_attn=0)}


@pytest.mark.parametrize("name", list(BF16_CASES))
def test_forward_bf16_parity(tp, tokscale, name):
    tokens, scale = tokscale
    ocfg = oracle_cfg(**BF16_CASES[name])
    flat = flat_params(ocfg, seed=11)
    _, X = encoded_batch(23, 301, tokens, scale)  # 61 tiles of 5 candidates, last one ragged
    ref = OM.forward(ocfg, OM.unflatten(ocfg, flat), X)
    m = tp.TLP(product_cfg(ocfg, "bf16"))
    m.set_params(flat.astype(np.float32))
    s = m.score(torch.from_numpy(X).cuda())
    m.sync()
    assert rel_err(s.cpu().numpy(), ref) <= 1e-2


def test_bf16_batch_invariance_and_retrain_refresh(tp, tokscale):
    tokens, scale = tokscale
    ocfg = oracle_cfg(n_attn=2)
    flat = flat_params(ocfg, seed=12)
    _, X = encoded_batch(24, 300, tokens, scale)
    m = tp.TLP(product_cfg(ocfg, "bf16"))
    m.set_params(flat.astype(np.float32))
    Xd = torch.from_numpy(X).cuda()
    full = m.score(Xd).cpu().numpy()
    for lo, hi in ((113, 250), (1, 2), (7, 300)):  # slots shift by lo mod 5
        part = m.score(Xd[lo:hi].contiguous()).cpu().numpy()
        assert np.array_equal(full[lo:hi].view(np.uint32), part.view(np.uint32)), (lo, hi)
    # new parameters must re-pack the bf16 weight stream
    flat2 = flat_params(ocfg, seed=13)
    m.set_params(flat2.astype(np.float32))
    s2 = m.score(Xd).cpu().numpy()
    m.sync()
    assert rel_err(s2, OM.forward(ocfg, OM.unflatten(ocfg, flat2), X)) <= 1e-2


def test_bf16_full_size_sampled(tp, tokscale):
    """C2 at full size in bench.py's launch configuration: 409,600 candidates
    (100 tasks x 4096), 2 layers, one tlp_score call; a seeded sample of 64
    candidates is checked against the oracle one by one; top-16 of every task
    equals the oracle top-k of the GPU's own scores (bit-exact selection)."""
    tokens, scale = tokscale
    ocfg = oracle_cfg(n_attn=2)
    flat = flat_params(ocfg, seed=7)
    N = 100 * 4096
    b = synth.generate(1000, N)
    m = tp.TLP(product_cfg(ocfg, "bf16"))
    m.set_token_table(sorted(tokens, key=tokens.get))
    m.set_norm_scales(scale)
    m.set_params(flat.astype(np.float32))
    X = m.encode(tp.DeviceBatch.from_packed(b))
    s = m.score(X)
    off = synth.uniform_task_off(100, 4096)
    idx, val = m.topk(s, off, 16)
    m.sync()
    s_h = s.cpu().numpy()
    rng = np.random.default_rng(0)
    pick = np.sort(rng.choice(N, 64, replace=False))
    Xs = oracle.encode([b.slice(int(i), int(i) + 1).to_lists()[0] for i in pick], tokens, scale)
    assert np.array_equal(X[torch.from_numpy(pick).cuda()].cpu().numpy().view(np.uint32), Xs.view(np.uint32))
    ref = OM.forward(ocfg, OM.unflatten(ocfg, flat), Xs)
    assert rel_err(s_h[pick], ref) <= 1e-2
    idx_ref, val_ref = oracle.topk(s_h[:, 0], off, 16)
    assert np.array_equal(idx.cpu().numpy(), idx_ref)


# ---------------------------------------------------------------- bf16 tcgen05 GEMM (training, bf16 ctx)
@pytest.mark.parametrize("ta,tb", [(0, 0), (0, 1), (1, 0), (1, 1)])
@pytest.mark.parametrize("M,N,K,splits", [(300, 200, 72, 1), (128, 128, 32, 1), (1000, 96, 516, 3),
                                          (64, 256, 4096, 8), (37, 22, 22, 1), (130, 30, 50, 2),
                                          (256, 256, 3000, 5), (200, 136, 777, 3),
                                          # ta = 0, splits = 1, 128 < N <= 256, N % 16 == 0: the
                                          # TMA-fed persistent kernel (k_tc_tma.cu), ragged M / K
                                          (300, 256, 72, 1), (1000, 144, 256, 1), (40000, 256, 768, 1),
                                          (5000, 128, 256, 1), (5000, 96, 128, 1),
                                          # N > 256, N % 256 == 0: 256-wide column blocks
                                          # (fused Q/K/V, LSTM gates), ragged M / K
                                          (5000, 768, 256, 1), (40000, 1024, 256, 1), (4097, 512, 100, 1)])
def test_train_gemm_building_block(tp, ta, tb, M, N, K, splits):
    rng = np.random.default_rng(M + N + K + 10 * ta + tb)
    A = rng.normal(size=(K, M) if ta else (M, K)).astype(np.float32)
    B = rng.normal(size=(N, K) if tb else (K, N)).astype(np.float32)
    opA = A.T if ta else A
    opB = B.T if tb else B
    m = tp.TLP(tp.TLPConfig(precision="bf16"))
    Ad, Bd = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
    ldc = N + (4 - N % 4) % 4
    C = torch.zeros((splits, M, ldc), dtype=torch.float32, device="cuda")
    st = m.lib.tlp_debug_gemm(m.h, ta, tb, M, N, K, Ad.data_ptr(), A.shape[1], Bd.data_ptr(),
                              B.shape[1], C.data_ptr(), ldc, splits, torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    assert st == 0
    got = C.cpu().numpy().sum(axis=0)[:, :N]
    # bf16x3 split precision (hi.hi + hi.lo + lo.hi): ~2^-16 per product + fp32 sums
    ref = opA.astype(np.float64) @ opB.astype(np.float64)
    assert rel_err(got, ref) <= 1e-4


@pytest.mark.parametrize("M,K,N,J", [(204800, 256, 256, 1), (64000, 256, 128, 1), (64000, 128, 256, 1),
                                     (3001, 256, 256, 1), (1775, 64, 64, 1), (70000, 256, 256, 3),
                                     (2500, 22, 128, 1), (204800, 22, 128, 1), (9000, 17, 256, 1)])
def test_wgrad_bias_building_block(tp, M, K, N, J):
    """The weight + bias gradient of one training layer (tlp_debug_wgrad; J = 3:
    three products sharing X, the Q/K/V case) vs fp64: dW = X^T dY within the
    tf32 operand rounding (R52: each operand truncated to 10 mantissa bits,
    <= 2 x 2^-10 per product), db = 1^T dY summed in fp32 (1e-5); covers ragged
    slices, the 256 x 128 head and 128 x 256 upsample shapes, shapes the TMA
    kernel does not take (K = 22 / 17) and the bench's 204,800 rows."""
    rng = np.random.default_rng(M + K + N)
    X = rng.normal(size=(M, K)).astype(np.float32)
    dY = rng.normal(size=(M, J * N)).astype(np.float32) * (rng.random((M, 1)) < 0.7)
    m = tp.TLP(tp.TLPConfig(precision="bf16"))
    Xd, Yd = torch.from_numpy(X).cuda(), torch.from_numpy(dY).cuda()
    for j in range(J):
        out = torch.zeros(K * N + N, dtype=torch.float32, device="cuda")
        st = m.lib.tlp_debug_wgrad(m.h, M, K, N, Xd.data_ptr(), K, Yd[:, j * N:].data_ptr(), J * N,
                                   out.data_ptr(), torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()
        assert st == 0
        got = out.cpu().numpy()
        Y = dY[:, j * N:(j + 1) * N].astype(np.float64)
        ref_w = X.astype(np.float64).T @ Y
        assert rel_err(got[:K * N].reshape(K, N), ref_w) <= 3e-3
        assert rel_err(got[K * N:], Y.sum(axis=0)) <= 1e-5


def test_bf16_scoring_needs_paper_shape(tp):
    m = tp.TLP(tp.tiny_config(precision="bf16"))  # training works at any shape
    m.set_params(np.zeros(m.num_params, np.float32))
    with pytest.raises(tp.TLPError) as e:
        m.score(torch.zeros((5, 25, 22), device="cuda"))
    assert e.value.code == "ERR_UNSUPPORTED"


def test_sharded_topk_merge_bitwise(tp, tokscale):
    """C-2 on one GPU: 4 shards (5-aligned, paper.dist.shard_range) scored and
    selected separately with their shard_base, then tlp_topk_merge == the
    unsharded tlp_topk bit for bit (needs batch-invariant bf16 scoring, R34)."""
    from paper_2211_03578_b200 import dist as D
    tokens, scale = tokscale
    ocfg = oracle_cfg(n_attn=2)
    flat = flat_params(ocfg, seed=9)
    _, X = encoded_batch(26, 2003, tokens, scale)
    off = np.array([0, 400, 401, 1500, 2003], np.int64)
    m = tp.TLP(product_cfg(ocfg, "bf16"))
    m.set_params(flat.astype(np.float32))
    Xd = torch.from_numpy(X).cuda()
    full = m.score(Xd)
    idx_ref, val_ref = m.topk(full, off, 16)
    vs, is_ = [], []
    for r in range(4):
        lo, hi = D.shard_range(2003, 4, r)
        s = m.score(Xd[lo:hi].contiguous())
        i, v = m.topk(s, D.local_task_off(off, lo, hi), 16, shard_base=lo)
        vs.append(v); is_.append(i)
    idx, val = m.topk_merge(torch.stack(vs), torch.stack(is_))
    m.sync()
    assert np.array_equal(idx.cpu().numpy(), idx_ref.cpu().numpy())
    assert np.array_equal(val.cpu().numpy().view(np.uint32), val_ref.cpu().numpy().view(np.uint32))


# ---------------------------------------------------------------- one search round from host memory
ROUND_OFF = np.array([0, 400, 401, 401, 1500, 2003], np.int64)  # an empty and a 1-candidate task


def _round_model(tp, tokens, scale, precision):
    ocfg = oracle_cfg(n_attn=2, n_tasks=2)
    flat = flat_params(ocfg, seed=21)
    m = tp.TLP(product_cfg(ocfg, precision))
    m.set_token_table(sorted(tokens, key=tokens.get))
    m.set_norm_scales(scale)
    m.set_params(flat.astype(np.float32))
    return m, ocfg, flat


@pytest.mark.parametrize("precision", ["fp32", "bf16"])
def test_search_round_host_pipeline(tp, tokscale, precision):
    """tlp_search_round (host batch; chunked host->device copy overlapped with
    encode + score) equals tlp_encode -> tlp_score -> tlp_topk on a device copy
    bit for bit, for every chunk count and for pinned and pageable host memory;
    its top-k is the oracle top-k of the GPU's scores and sampled scores match
    the oracle forward."""
    tokens, scale = tokscale
    m, ocfg, flat = _round_model(tp, tokens, scale, precision)
    N = 2003
    b = synth.generate(41, N)
    X = m.encode(tp.DeviceBatch.from_packed(b))
    s = m.score(X)
    idx_ref, val_ref = m.topk(s, ROUND_OFF, 16, head=1, shard_base=7)
    m.sync()
    idx_ref, val_ref = idx_ref.cpu().numpy(), val_ref.cpu().numpy()
    s_h = s.cpu().numpy()
    o_idx, o_val = oracle.topk(s_h[:, 1], ROUND_OFF, 16)
    assert np.array_equal(idx_ref, np.where(o_idx >= 0, o_idx + 7, o_idx))
    pick = np.array([0, 1, 399, 400, 1004, 2002])
    Xs = oracle.encode([b.slice(int(i), int(i) + 1).to_lists()[0] for i in pick], tokens, scale)
    tol = 1e-5 if precision == "fp32" else 1e-2
    assert rel_err(s_h[pick], OM.forward(ocfg, OM.unflatten(ocfg, flat), Xs)) <= tol
    for pin in (True, False):
        hb = tp.DeviceBatch.from_packed(b, pin=True) if pin else tp.DeviceBatch.from_packed(b, device="cpu")
        for chunks in ((1, 2, 7, 64) if pin else (3,)):
            idx, val = m.search_round(hb, ROUND_OFF, 16, head=1, shard_base=7, chunks=chunks)
            m.sync()
            assert np.array_equal(idx.numpy(), idx_ref), (pin, chunks)
            assert np.array_equal(val.numpy().view(np.uint32), val_ref.view(np.uint32)), (pin, chunks)


def test_search_round_errors(tp, tokscale):
    tokens, scale = tokscale
    m, _, _ = _round_model(tp, tokens, scale, "bf16")
    b = synth.generate(42, 50)
    hb = tp.DeviceBatch.from_packed(b, device="cpu")
    off = np.array([0, 20, 50], np.int64)
    for kw, code in ((dict(chunks=0), "ERR_ARG"), (dict(chunks=65), "ERR_ARG"),
                     (dict(head=2), "ERR_ARG")):
        with pytest.raises(tp.TLPError) as e:
            m.search_round(hb, off, 4, **kw)
        assert e.value.code == code
    with pytest.raises(tp.TLPError) as e:
        m.search_round(hb, np.array([0, 20, 51], np.int64), 4)
    assert e.value.code == "ERR_SHAPE"
    bad = hb.seq_off.clone()
    bad[3] = bad[2] - 1
    hb_bad = tp.DeviceBatch(bad, hb.prim_type, hb.arg_off, hb.arg_kind, hb.arg_num, hb.arg_name,
                            hb.str_blob, hb.str_off, hb.N, hb.P, hb.A, hb.U)
    with pytest.raises(tp.TLPError) as e:
        m.search_round(hb_bad, off, 4)
    assert e.value.code == "ERR_SHAPE"
    idx, _ = m.search_round(hb, off, 4)  # the ctx is still usable after the refusals
    m.sync()
    assert (idx.numpy()[:, :4] >= 0).all()


# ---------------------------------------------------------------- edge cases
def test_empty_and_single_candidate(tp, tokscale):
    """N = 0 is a no-op for encode / score / top-k (segments empty -> padding);
    N = 1 scores like the oracle on both paths (one ragged tile)."""
    tokens, scale = tokscale
    ocfg = oracle_cfg(n_attn=2)
    flat = flat_params(ocfg, seed=61)
    for prec, tol in (("fp32", 1e-5), ("bf16", 1e-2)):
        m = tp.TLP(product_cfg(ocfg, prec))
        m.set_token_table(sorted(tokens, key=tokens.get))
        m.set_norm_scales(scale)
        m.set_params(flat.astype(np.float32))
        empty = torch.empty((0, 25, 22), device="cuda")
        s0 = m.score(empty)
        assert s0.shape == (0, 1)
        idx, val = m.topk(s0, np.array([0, 0], np.int64), 4)
        m.sync()
        assert (idx.cpu().numpy() == -1).all() and np.isneginf(val.cpu().numpy()).all()
        b, X = encoded_batch(62, 1, tokens, scale)
        Xd = m.encode(tp.DeviceBatch.from_packed(b))
        assert np.array_equal(Xd.cpu().numpy().view(np.uint32), X.view(np.uint32))
        s1 = m.score(Xd)
        m.sync()
        assert rel_err(s1.cpu().numpy(), OM.forward(ocfg, OM.unflatten(ocfg, flat), X)) <= tol


def test_crop_boundaries_bit_exact(tp, tokscale):
    """Sequences of exactly 24 / 25 / 26 / 54 primitives and primitives with
    exactly 10 / 11 / 12 arguments: the crop boundaries of R4 (rows >= 25 and
    argument slots >= 11 are dropped) are bit-exact against the oracle."""
    tokens, scale = tokscale
    b = synth.generate(63, 400)
    seqs = b.to_lists()
    lens = np.array([len(sq) for sq in seqs])
    picked = [int(np.flatnonzero(lens == k)[0]) for k in (24, 25, 26) if (lens == k).any()]
    picked += [int(np.argmax(lens))]
    nargs = [max(len(p[1]) for p in sq) for sq in seqs]
    for k in (10, 11, 12):
        hits = [i for i, a in enumerate(nargs) if a == k]
        if hits:
            picked.append(hits[0])
    sub = [seqs[i] for i in picked]
    assert max(lens[picked]) > 25 and any(nargs[i] > 11 for i in picked)
    ref = oracle.encode(sub, tokens, scale)
    m = make_encoder(tp, tokens, scale)
    X = m.encode(tp.DeviceBatch.from_packed(synth.pack(sub)))
    m.sync()
    assert np.array_equal(X.cpu().numpy().view(np.uint32), ref.view(np.uint32))


# ---------------------------------------------------------------- R1 / R3 fitted by the library
def test_fit_token_table_and_scales_bit_exact(tp):
    """tlp_fit_token_table (R1: first occurrence over the training stream's name
    arguments) and tlp_fit_norm_scales (R3: per-column max |x| over the kept,
    un-normalised rows, 1.0 for all-zero columns) against oracle.build_token_table
    / oracle.fit_scales on the same seeded training split; then tlp_encode with
    the fitted state equals oracle.encode bit for bit."""
    train = synth.generate(12345, 2000, unseen_rate=0.0)
    tokens = oracle.build_token_table(synth.training_stream(12345, 2000))
    raw = np.stack([oracle.extract_rows(s, tokens, 25, 22, 11) for s in train.to_lists()])
    scale_ref = oracle.fit_scales(raw)
    assert (np.diff(train.seq_off) > 25).any() and (np.diff(train.arg_off) > 11).any()  # crops exercised
    m = tp.TLP(tp.TLPConfig(precision="fp32"))
    m.fit_token_table(train)
    scale = m.fit_norm_scales(tp.DeviceBatch.from_packed(train))
    m.sync()
    assert np.array_equal(scale.view(np.uint32), scale_ref.view(np.uint32)), (scale, scale_ref)
    b = synth.generate(5, 777)  # includes 1% unseen names -> token 1
    X = m.encode(tp.DeviceBatch.from_packed(b))
    m.sync()
    X_ref = oracle.encode(b.to_lists(), tokens, scale_ref)
    assert np.array_equal(X.cpu().numpy().view(np.uint32), X_ref.view(np.uint32))


def test_fit_scales_errors_and_empty(tp):
    """Device errors of the fit follow tlp_encode's (kept data only); an empty
    batch gives scale 1.0 everywhere."""
    m = tp.TLP(tp.TLPConfig(precision="fp32"))
    empty = synth.pack([])
    assert np.array_equal(m.fit_norm_scales(tp.DeviceBatch.from_packed(empty)), np.ones(22, np.float32))
    bad = synth.pack([[(3, [1.0, float("inf")])]])
    m.fit_norm_scales(tp.DeviceBatch.from_packed(bad))
    with pytest.raises(tp.TLPError) as e:
        m.sync()
    assert e.value.code == "ERR_NONFINITE"
