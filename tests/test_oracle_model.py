"""Pins for oracle O2 (forward) and O3 (backward)."""
import numpy as np
import pytest
import torch

import synth
from oracle import model as M

SMALL = M.Config(L=6, E=8, T=3, hidden=16, up_dims=(12, 16), attn_heads=4, n_attn=1,
                 n_res=2, head_dim=8, n_tasks=2)


def rand_params(cfg, seed, scale=1.0):
    vals = synth.init_params(seed, M.param_shapes(cfg), bf16=False, scale=scale)
    return {n: v for (n, _), v in zip(M.param_shapes(cfg), vals)}


def rand_X(cfg, n, seed, n_real=None):
    rng = np.random.default_rng(seed)
    X = rng.normal(size=(n, cfg.L, cfg.E))
    if n_real is not None:
        X[:, n_real:] = 0
    return X


class TorchTLP(torch.nn.Module):
    """Independent fp64 re-implementation from standard torch layers (test only)."""

    def __init__(self, cfg, p):
        super().__init__()
        self.cfg = cfg
        self.ups = torch.nn.ModuleList()
        d = cfg.E
        for i, w in enumerate(cfg.up_dims):
            lin = torch.nn.Linear(d, w, dtype=torch.float64)
            lin.weight.data = torch.tensor(p["up%d.W" % i].T.copy())
            lin.bias.data = torch.tensor(p["up%d.b" % i])
            self.ups.append(lin)
            d = w
        H = cfg.hidden
        self.attn = torch.nn.ModuleList()
        for l in range(cfg.n_attn):
            mha = torch.nn.MultiheadAttention(H, cfg.attn_heads, bias=True, batch_first=True,
                                              dtype=torch.float64)
            pre = "attn%d." % l
            mha.in_proj_weight.data = torch.tensor(np.concatenate(
                [p[pre + "Wq"].T, p[pre + "Wk"].T, p[pre + "Wv"].T]))
            mha.in_proj_bias.data = torch.tensor(np.concatenate([p[pre + "bq"], p[pre + "bk"], p[pre + "bv"]]))
            mha.out_proj.weight.data = torch.tensor(p[pre + "Wo"].T.copy())
            mha.out_proj.bias.data = torch.tensor(p[pre + "bo"])
            self.attn.append(mha)
        self.pos = (torch.nn.Parameter(torch.tensor(p["pos"].copy()))
                    if getattr(cfg, "pos_enc", False) else None)
        self.res = torch.nn.ModuleList()
        for r in range(cfg.n_res):
            a = torch.nn.Linear(H, H, dtype=torch.float64)
            b = torch.nn.Linear(H, H, dtype=torch.float64)
            a.weight.data = torch.tensor(p["res%d.Wa" % r].T.copy()); a.bias.data = torch.tensor(p["res%d.a" % r])
            b.weight.data = torch.tensor(p["res%d.Wb" % r].T.copy()); b.bias.data = torch.tensor(p["res%d.b" % r])
            self.res.append(torch.nn.ModuleList([a, b]))
        self.heads = torch.nn.ModuleList()
        for t in range(cfg.n_tasks):
            a = torch.nn.Linear(H, cfg.head_dim, dtype=torch.float64)
            b = torch.nn.Linear(cfg.head_dim, 1, dtype=torch.float64)
            a.weight.data = torch.tensor(p["head%d.W1" % t].T.copy()); a.bias.data = torch.tensor(p["head%d.c1" % t])
            b.weight.data = torch.tensor(p["head%d.w2" % t].T.copy()); b.bias.data = torch.tensor(p["head%d.c2" % t])
            self.heads.append(torch.nn.ModuleList([a, b]))

    def forward(self, x):
        h = x
        pad = (x == 0).all(dim=-1) if getattr(self.cfg, "attn_mask", False) else None
        for lin in self.ups:
            h = torch.relu(lin(h))
        if self.pos is not None:
            h = h + self.pos
        for mha in self.attn:
            h = h + mha(h, h, h, key_padding_mask=pad, need_weights=False)[0]
        for a, b in self.res:
            h = h + b(torch.relu(a(h)))
        return torch.stack([b(torch.relu(a(h)))[..., 0].sum(dim=1) for a, b in self.heads], dim=1)

    def named_grads(self):
        g = {}
        for i, lin in enumerate(self.ups):
            g["up%d.W" % i] = lin.weight.grad.T; g["up%d.b" % i] = lin.bias.grad
        H = self.cfg.hidden
        for l, mha in enumerate(self.attn):
            pre = "attn%d." % l
            W, b = mha.in_proj_weight.grad, mha.in_proj_bias.grad
            for j, nm in enumerate("qkv"):
                g[pre + "W" + nm] = W[j * H:(j + 1) * H].T
                g[pre + "b" + nm] = b[j * H:(j + 1) * H]
            g[pre + "Wo"] = mha.out_proj.weight.grad.T; g[pre + "bo"] = mha.out_proj.bias.grad
        for r, (a, b) in enumerate(self.res):
            g["res%d.Wa" % r] = a.weight.grad.T; g["res%d.a" % r] = a.bias.grad
            g["res%d.Wb" % r] = b.weight.grad.T; g["res%d.b" % r] = b.bias.grad
        for t, (a, b) in enumerate(self.heads):
            g["head%d.W1" % t] = a.weight.grad.T; g["head%d.c1" % t] = a.bias.grad
            g["head%d.w2" % t] = b.weight.grad.T; g["head%d.c2" % t] = b.bias.grad
        if self.pos is not None:
            g["pos"] = self.pos.grad
        return {k: v.detach().numpy() for k, v in g.items()}


@pytest.mark.parametrize("cfg", [SMALL, M.Config(hidden=64, up_dims=(32, 64), head_dim=32, n_attn=2, n_tasks=1)])
def test_forward_matches_torch_layers(cfg):
    p = rand_params(cfg, 1)
    X = rand_X(cfg, 7, 2, n_real=cfg.L - 2)
    s = M.forward(cfg, p, X)
    ref = TorchTLP(cfg, p)(torch.tensor(X)).detach().numpy()
    assert np.abs(s - ref).max() <= 1e-12 * max(1.0, np.abs(ref).max())


def test_backward_matches_torch_autograd():
    cfg = SMALL
    p = rand_params(cfg, 3)
    X = rand_X(cfg, 5, 4, n_real=4)
    g = np.random.default_rng(5).normal(size=(5, cfg.n_tasks))
    s, acts = M.forward(cfg, p, X, save=True)
    grads = M.backward(cfg, p, acts, g)
    tm = TorchTLP(cfg, p)
    out = tm(torch.tensor(X))
    (out * torch.tensor(g)).sum().backward()
    tg = tm.named_grads()
    for name, _ in M.param_shapes(cfg):
        a, b = grads[name].reshape(tg[name].shape), tg[name]
        assert np.abs(a - b).max() <= 1e-12 * max(1.0, np.abs(b).max()), name


def test_backward_finite_differences():
    """S:346 / S:597: central differences, h=1e-5, relative error < 1e-4 (fp64)."""
    cfg = SMALL
    p = rand_params(cfg, 6)
    X = rand_X(cfg, 3, 7, n_real=5)
    g = np.random.default_rng(8).normal(size=(3, cfg.n_tasks))
    s, acts = M.forward(cfg, p, X, save=True)
    grads = M.backward(cfg, p, acts, g)
    flat = M.flatten(cfg, p)
    ga = M.flatten(cfg, grads)
    rng = np.random.default_rng(9)
    h = 1e-5
    f = lambda v: float((M.forward(cfg, M.unflatten(cfg, v), X) * g).sum())  # noqa: E731
    # every parameter tensor gets probed
    o = 0
    for name, shp in M.param_shapes(cfg):
        k = int(np.prod(shp))
        for i in rng.choice(k, size=min(k, 4), replace=False):
            e = np.zeros_like(flat); e[o + i] = h
            fd = (f(flat + e) - f(flat - e)) / (2 * h)
            assert abs(fd - ga[o + i]) <= 1e-4 * max(abs(fd), 1e-3), (name, i, fd, ga[o + i])
        o += k


def test_zero_weights_give_zero():
    cfg = SMALL
    p = {n: np.zeros(s) for n, s in M.param_shapes(cfg)}
    assert not M.forward(cfg, p, np.zeros((2, cfg.L, cfg.E))).any()


def test_row_permutation_invariance():
    cfg = M.Config(hidden=64, up_dims=(32, 64), head_dim=32)
    p = rand_params(cfg, 11)
    X = rand_X(cfg, 4, 12)
    perm = np.random.default_rng(13).permutation(cfg.L)
    a, b = M.forward(cfg, p, X), M.forward(cfg, p, X[:, perm])
    assert np.abs(a - b).max() <= 1e-12 * np.abs(a).max()  # R9 + sum pooling


def test_wq_wk_zero_gives_row_mean_of_v():
    cfg = SMALL
    p = rand_params(cfg, 14)
    p["attn0.Wq"][:] = 0; p["attn0.bq"][:] = 0
    p["attn0.Wk"][:] = 0; p["attn0.bk"][:] = 0
    X = rand_X(cfg, 3, 15)
    _, acts = M.forward(cfg, p, X, save=True)
    a = acts["attn"][0]
    V = a["h"] @ p["attn0.Wv"] + p["attn0.bv"]
    expect = np.repeat(V.mean(axis=1, keepdims=True), cfg.L, axis=1)  # uniform softmax
    assert np.abs(a["O"] - expect).max() < 1e-13


def test_single_row_softmax_is_one():
    cfg = M.Config(L=1, E=8, T=3, hidden=16, up_dims=(16,), attn_heads=4, head_dim=8)
    p = rand_params(cfg, 16)
    X = rand_X(cfg, 3, 17)
    _, acts = M.forward(cfg, p, X, save=True)
    a = acts["attn"][0]
    assert np.all(a["A"] == 1.0)
    V = a["h"] @ p["attn0.Wv"] + p["attn0.bv"]
    assert np.abs(a["O"] - V).max() < 1e-13


def test_head_order_identity_r13():
    """R13: per-position head then sum == sum-pool after ReLU, then affine with L*c2."""
    cfg = M.Config(hidden=64, up_dims=(32, 64), head_dim=32, n_tasks=3)
    p = rand_params(cfg, 18)
    X = rand_X(cfg, 5, 19, n_real=17)
    s, acts = M.forward(cfg, p, X, save=True)
    for t in range(cfg.n_tasks):
        z = acts["heads"][t]["z"]
        alt = z.sum(axis=1) @ p["head%d.w2" % t][:, 0] + cfg.L * p["head%d.c2" % t][0]
        assert np.abs(alt - s[:, t]).max() <= 1e-13 * np.abs(s[:, t]).max()


def test_pad_rows_share_one_head_value():
    cfg = M.Config(hidden=64, up_dims=(32, 64), head_dim=32)
    p = rand_params(cfg, 20)
    X = rand_X(cfg, 3, 21, n_real=17)
    _, acts = M.forward(cfg, p, X, save=True)
    z = acts["heads"][0]["z"]
    per_pos = z @ p["head0.w2"][:, 0]
    pads = per_pos[:, 17:]
    assert np.abs(pads - pads[:, :1]).max() <= 1e-14 * np.abs(per_pos).max()


def test_param_count_paper_config():
    # 595,329 / 858,497 / 694,404 params.
    assert M.n_params(M.Config(n_attn=1)) == 595329
    assert M.n_params(M.Config(n_attn=2)) == 858497
    assert M.n_params(M.Config(n_attn=1, n_tasks=4)) == 694404
    assert M.n_params(M.Config(hidden=64, up_dims=(32, 64), head_dim=32)) == 38241


# ---------------------------------------------------------------- NEXT-3: padding mask (R42)
MASKED = M.Config(L=6, E=8, T=3, hidden=16, up_dims=(8, 16), attn_heads=2, n_attn=2, n_res=1,
                  head_dim=8, n_tasks=2, attn_mask=True)


def _ragged_X(cfg, n, seed):
    X = rand_X(cfg, n, seed, n_real=cfg.L)
    lens = np.random.default_rng(seed).integers(1, cfg.L + 1, n)
    for i, ln in enumerate(lens):
        X[i, ln:] = 0.0
    return X, lens


def test_masked_forward_matches_torch_key_padding_mask():
    """nn.MultiheadAttention(key_padding_mask = all-zero rows): independent."""
    p = rand_params(MASKED, 11)
    X, _ = _ragged_X(MASKED, 9, 12)
    s = M.forward(MASKED, p, X)
    ref = TorchTLP(MASKED, p)(torch.tensor(X)).detach().numpy()
    assert np.abs(s - ref).max() <= 1e-12 * max(1.0, np.abs(ref).max())


def test_masked_equals_unmasked_without_padding():
    p = rand_params(MASKED, 13)
    X = rand_X(MASKED, 4, 14, n_real=MASKED.L)
    import dataclasses
    plain = dataclasses.replace(MASKED, attn_mask=False)
    assert np.array_equal(M.forward(MASKED, p, X), M.forward(plain, p, X))


def test_masked_keys_do_not_matter():
    """Changing the hidden state of a padding key (through the upsample bias)
    cannot change any output other than through that row itself: scores of a
    candidate with padding equal those of the same candidate whose padding keys
    are dropped from every softmax (re-computed with the keys sliced off)."""
    p = rand_params(MASKED, 15)
    X, lens = _ragged_X(MASKED, 6, 16)
    s = M.forward(MASKED, p, X, save=True)[1]
    for i, ln in enumerate(lens):
        for l, a in enumerate(s["attn"]):
            A = a["A"][i]                       # [heads, L, L]
            assert np.all(A[:, :, ln:] == 0.0)  # no weight on padding keys
            assert np.allclose(A[:, :, :ln].sum(-1), 1.0)


def test_masked_backward_matches_torch_autograd():
    cfg = MASKED
    p = rand_params(cfg, 17)
    X, _ = _ragged_X(cfg, 5, 18)
    g = np.random.default_rng(19).normal(size=(5, cfg.n_tasks))
    s, acts = M.forward(cfg, p, X, save=True)
    grads = M.backward(cfg, p, acts, g)
    tm = TorchTLP(cfg, p)
    out = tm(torch.tensor(X))
    (out * torch.tensor(g)).sum().backward()
    tg = tm.named_grads()
    for name, _ in M.param_shapes(cfg):
        a, b = grads[name].reshape(tg[name].shape), tg[name]
        assert np.abs(a - b).max() <= 1e-12 * max(1.0, np.abs(b).max()), name


# ---------------------------------------------------------------- NEXT-3: learned positional table (R43)
POSENC = M.Config(L=6, E=8, T=3, hidden=16, up_dims=(8, 16), attn_heads=2, n_attn=2, n_res=1,
                  head_dim=8, n_tasks=2, pos_enc=True)


def test_posenc_forward_backward_match_torch():
    cfg = POSENC
    p = rand_params(cfg, 21)
    X, _ = _ragged_X(cfg, 5, 22)
    g = np.random.default_rng(23).normal(size=(5, cfg.n_tasks))
    s, acts = M.forward(cfg, p, X, save=True)
    tm = TorchTLP(cfg, p)
    out = tm(torch.tensor(X))
    assert np.abs(s - out.detach().numpy()).max() <= 1e-12 * max(1.0, np.abs(s).max())
    (out * torch.tensor(g)).sum().backward()
    tg = tm.named_grads()
    grads = M.backward(cfg, p, acts, g)
    for name, _ in M.param_shapes(cfg):
        a, b = grads[name].reshape(tg[name].shape), tg[name]
        assert np.abs(a - b).max() <= 1e-12 * max(1.0, np.abs(b).max()), name


def test_posenc_breaks_permutation_invariance_and_zero_table_is_identity():
    """with positional encoding off a row-permuted input gives the same
    score; with a nonzero table it does not; a zero table equals no table."""
    import dataclasses
    cfg = POSENC
    p = rand_params(cfg, 24)
    X = rand_X(cfg, 3, 25, n_real=cfg.L)
    perm = np.random.default_rng(26).permutation(cfg.L)
    assert np.abs(M.forward(cfg, p, X) - M.forward(cfg, p, X[:, perm])).max() > 1e-6
    plain = dataclasses.replace(cfg, pos_enc=False)
    q = {k: v for k, v in p.items() if k != "pos"}
    assert np.allclose(M.forward(plain, q, X), M.forward(plain, q, X[:, perm]), rtol=0, atol=1e-12)
    p0 = dict(p, pos=np.zeros_like(p["pos"]))
    assert np.array_equal(M.forward(cfg, p0, X), M.forward(plain, q, X))


# ---------------------------------------------------------------- R50: per-term RMS of each gradient
@pytest.mark.parametrize("backbone", ["attn", "lstm"])
def test_term_rms_brute_force_single_row(backbone):
    """With L = 1 every candidate contributes exactly one row term to each
    parameter gradient, so backward(..., rms=) must equal the root of the sum of
    the squared per-candidate gradients, each computed alone by brute force;
    and passing ``rms`` leaves the gradients bitwise unchanged."""
    cfg = M.Config(L=1, E=8, T=3, hidden=16, up_dims=(12, 16), attn_heads=4, n_attn=1,
                   n_res=2, head_dim=8, n_tasks=2, backbone=backbone, pos_enc=True)
    p = rand_params(cfg, 3)
    X = rand_X(cfg, 7, 4)
    g = np.random.default_rng(5).normal(size=(7, 2))
    s, acts = M.forward(cfg, p, X, save=True)
    plain = M.backward(cfg, p, acts, g)
    rms = {}
    grads = M.backward(cfg, p, acts, g, rms=rms)
    assert set(rms) == set(grads)
    for k in grads:
        assert np.array_equal(grads[k], plain[k]), k
    sq = {k: np.zeros_like(v) for k, v in grads.items()}
    for n in range(7):
        _, a_n = M.forward(cfg, p, X[n:n + 1], save=True)
        for k, v in M.backward(cfg, p, a_n, g[n:n + 1]).items():
            sq[k] += v * v
    for k in grads:
        np.testing.assert_allclose(rms[k], np.sqrt(sq[k]), rtol=1e-12, atol=1e-300, err_msg=k)


def test_term_rms_cauchy_schwarz():
    """|grad| <= sqrt(#terms) * rms elementwise (N*L row terms), rms >= 0."""
    p = rand_params(SMALL, 6)
    X = rand_X(SMALL, 5, 7, n_real=4)
    g = np.random.default_rng(8).normal(size=(5, 2))
    _, acts = M.forward(SMALL, p, X, save=True)
    rms = {}
    grads = M.backward(SMALL, p, acts, g, rms=rms)
    nt = 5 * SMALL.L
    for k in grads:
        assert np.all(rms[k] >= 0)
        assert np.all(np.abs(grads[k]) <= np.sqrt(nt) * rms[k] * (1 + 1e-12) + 1e-300), k
