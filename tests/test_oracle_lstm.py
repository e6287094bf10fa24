"""Pins of the NEXT-4 LSTM backbone of oracle/model.py (R49): the forward and
the hand-written backpropagation-through-time against torch.nn.LSTM (fp64,
gate order i, f, g, o) and autograd, central finite differences, and the SPEC
anti-test: with an LSTM backbone the score is NOT invariant
under a permutation of the rows (it is for attention without positional
encoding)."""
import numpy as np
import pytest
import torch

from oracle import model as M

from test_oracle_model import TorchTLP, rand_X, rand_params

SMALL = M.Config(L=6, E=8, T=3, hidden=16, up_dims=(12, 16), attn_heads=4, n_attn=1,
                 n_res=2, head_dim=8, n_tasks=2, backbone="lstm")


class TorchLSTMTLP(TorchTLP):
    """TorchTLP with its attention layers replaced by torch.nn.LSTM layers and
    the identity residual of R49."""

    def __init__(self, cfg, p):
        base = M.Config(**{**cfg.__dict__, "backbone": "attn", "n_attn": 0})
        super().__init__(base, p)
        self.cfg = cfg
        H = cfg.hidden
        self.lstm = torch.nn.ModuleList()
        for l in range(cfg.n_attn):
            m = torch.nn.LSTM(H, H, batch_first=True, dtype=torch.float64)
            pre = "lstm%d." % l
            m.weight_ih_l0.data = torch.tensor(p[pre + "Wih"].T.copy())
            m.weight_hh_l0.data = torch.tensor(p[pre + "Whh"].T.copy())
            m.bias_ih_l0.data = torch.tensor(p[pre + "bih"].copy())
            m.bias_hh_l0.data = torch.tensor(p[pre + "bhh"].copy())
            self.lstm.append(m)

    def forward(self, x):
        h = x
        for lin in self.ups:
            h = torch.relu(lin(h))
        if self.pos is not None:
            h = h + self.pos
        for m in self.lstm:
            h = h + m(h)[0]
        for a, b in self.res:
            h = h + b(torch.relu(a(h)))
        return torch.stack([b(torch.relu(a(h)))[..., 0].sum(dim=1) for a, b in self.heads], dim=1)

    def named_grads(self):
        g = super().named_grads()
        for l, m in enumerate(self.lstm):
            pre = "lstm%d." % l
            g[pre + "Wih"] = m.weight_ih_l0.grad.T.numpy()
            g[pre + "Whh"] = m.weight_hh_l0.grad.T.numpy()
            g[pre + "bih"] = m.bias_ih_l0.grad.numpy()
            g[pre + "bhh"] = m.bias_hh_l0.grad.numpy()
        return g


CFGS = [SMALL, M.Config(hidden=64, up_dims=(32, 64), head_dim=32, n_attn=2, n_tasks=1, backbone="lstm"),
        M.Config(L=6, E=8, T=3, hidden=16, up_dims=(12, 16), attn_heads=4, n_attn=1, n_res=1, head_dim=8,
                 backbone="lstm", pos_enc=True)]


@pytest.mark.parametrize("cfg", CFGS)
def test_lstm_forward_matches_torch(cfg):
    p = rand_params(cfg, 1)
    X = rand_X(cfg, 7, 2, n_real=cfg.L - 2)
    s = M.forward(cfg, p, X)
    ref = TorchLSTMTLP(cfg, p)(torch.tensor(X)).detach().numpy()
    assert np.abs(s - ref).max() <= 1e-12 * max(1.0, np.abs(ref).max())


@pytest.mark.parametrize("cfg", CFGS)
def test_lstm_backward_matches_torch_autograd(cfg):
    p = rand_params(cfg, 3)
    X = rand_X(cfg, 5, 4, n_real=cfg.L - 3)
    g = np.random.default_rng(5).normal(size=(5, cfg.n_tasks))
    s, acts = M.forward(cfg, p, X, save=True)
    grads = M.backward(cfg, p, acts, g)
    tm = TorchLSTMTLP(cfg, p)
    (tm(torch.tensor(X)) * torch.tensor(g)).sum().backward()
    tg = tm.named_grads()
    for name, _ in M.param_shapes(cfg):
        a, b = grads[name].reshape(tg[name].shape), tg[name]
        assert np.abs(a - b).max() <= 1e-12 * max(1.0, np.abs(b).max()), name


def test_lstm_backward_finite_differences():
    cfg = SMALL
    p = rand_params(cfg, 6)
    X = rand_X(cfg, 3, 7, n_real=5)
    g = np.random.default_rng(8).normal(size=(3, cfg.n_tasks))
    _, acts = M.forward(cfg, p, X, save=True)
    ga = M.flatten(cfg, M.backward(cfg, p, acts, g))
    flat = M.flatten(cfg, p)
    f = lambda v: float((M.forward(cfg, M.unflatten(cfg, v), X) * g).sum())  # noqa: E731
    rng = np.random.default_rng(9)
    o = 0
    for name, shp in M.param_shapes(cfg):
        k = int(np.prod(shp))
        if name.startswith("lstm"):
            for i in rng.choice(k, size=6, replace=False):
                e = np.zeros_like(flat); e[o + i] = 1e-5
                fd = (f(flat + e) - f(flat - e)) / 2e-5
                assert abs(fd - ga[o + i]) <= 1e-4 * max(abs(fd), 1e-3), (name, i, fd, ga[o + i])
        o += k


def test_lstm_is_not_permutation_invariant_but_attention_is():
    """SPEC S:347 anti-test."""
    for backbone, invariant in (("lstm", False), ("attn", True)):
        cfg = M.Config(**{**SMALL.__dict__, "backbone": backbone})
        p = rand_params(cfg, 11)
        X = rand_X(cfg, 4, 12)
        perm = np.random.default_rng(0).permutation(cfg.L)
        a, b = M.forward(cfg, p, X), M.forward(cfg, p, X[:, perm])
        assert np.allclose(a, b, rtol=1e-12, atol=1e-12) == invariant


def test_lstm_single_row_closed_form():
    """L = 1: h_0 = c_0 = 0 gives c = sig(z_i) tanh(z_g), h = sig(z_o) tanh(c)
    with z = x Wih + bih + bhh -- written out from the LSTM equations."""
    cfg = M.Config(L=1, E=4, T=2, hidden=8, up_dims=(8,), attn_heads=2, n_attn=1, n_res=0,
                   head_dim=4, n_tasks=1, backbone="lstm")
    p = rand_params(cfg, 13)
    X = rand_X(cfg, 3, 14)
    _, acts = M.forward(cfg, p, X, save=True)
    x = acts["attn"][0]["h"][:, 0]
    z = x @ p["lstm0.Wih"] + p["lstm0.bih"] + p["lstm0.bhh"]
    H = 8
    sg = lambda v: 1.0 / (1.0 + np.exp(-v))  # noqa: E731
    c = sg(z[:, :H]) * np.tanh(z[:, 2 * H:3 * H])
    want = x + sg(z[:, 3 * H:]) * np.tanh(c)
    assert np.allclose(acts["h"][:, 0], want, rtol=0, atol=1e-14)


def test_lstm_param_count():
    assert M.n_params(M.Config(backbone="lstm")) == 595329 - 4 * (256 * 256 + 256) + 2 * (256 * 1024 + 1024)
