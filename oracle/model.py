"""O2/O3: the TLP / MTL-TLP network, forward and manual backward, float64.
TEST INFRASTRUCTURE.

Paper (P:295 [§4.4], P:431 [§6.1.3], P:355 [§5.2]):
  "The model first upsamples the dimension to 256 or more through multiple
   linear layers" -> upsample (R11: 22->128->256, ReLU after each).
  "we use the self-attention ... module ... to capture contextual features"
   with "8 heads", "one layer of the self-attention module is enough"
   -> n_attn layers of 8-head self-attention; R8 no mask, R9 no positional
   encoding, R10 identity residual and no LayerNorm, R14 scale 1/sqrt(d_h).
   NEXT-3 variant (cfg.attn_mask, R42): keys that are padding rows (all-zero
   rows of X, R7) are masked out of every softmax; queries are unchanged.
   NEXT-3 variant (cfg.pos_enc, R43): a learned positional table pos [L, H]
   is added to the upsampled rows before the first attention layer.
  NEXT-4 variant (cfg.backbone = "lstm", R49): "we use the self-attention or
   LSTM module, which we call the backbone basic module" -- n_attn layers of a
   single-direction LSTM (hidden -> hidden, gates i, f, g, o, h_0 = c_0 = 0,
   rows in sequence order, pads included) in place of the attention layers,
   with the same identity residual h <- h + LSTM(h) (R10).
  "Then two residual blocks follow" -> R12: h + relu(h Wa + a) Wb + b.
  "Finally, multiple linear layers and a sum operation are used to obtain a
   prediction score" -> R13: per position relu(h W1 + c1) w2 + c2, summed over
   the L rows (pads included).
  MTL-TLP: one such head per task on a shared backbone.

Parameter order R24: upsample (W, b)...; per attention layer Wq, bq, Wk, bk,
Wv, bv, Wo, bo (or per LSTM layer Wih [H, 4H], bih, Whh [H, 4H], bhh); per residual block Wa, a, Wb, b; per task head W1, c1, w2, c2.
W is [in, out].
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Dict, List, Optional, Tuple

import numpy as np


@dataclass
class Config:
    L: int = 25
    E: int = 22
    T: int = 11
    hidden: int = 256
    up_dims: Tuple[int, ...] = (128, 256)
    attn_heads: int = 8
    n_attn: int = 1
    n_res: int = 2
    head_dim: int = 128
    n_tasks: int = 1
    attn_mask: bool = False  # NEXT-3 / R42: mask padding keys (the paper: no mask, R8)
    pos_enc: bool = False    # NEXT-3 / R43: learned positional table (the paper: none, R9)
    backbone: str = "attn"   # NEXT-4 / R49: "attn" (the paper's choice) or "lstm"

    def __post_init__(self):
        self.up_dims = tuple(self.up_dims)
        assert self.up_dims[-1] == self.hidden
        assert self.hidden % self.attn_heads == 0
        assert self.backbone in ("attn", "lstm")

    @property
    def d_h(self) -> int:
        return self.hidden // self.attn_heads


def param_shapes(cfg: Config) -> List[Tuple[str, Tuple[int, ...]]]:
    """R24 flat order."""
    out: List[Tuple[str, Tuple[int, ...]]] = []
    d_in = cfg.E
    for i, d in enumerate(cfg.up_dims):
        out += [("up%d.W" % i, (d_in, d)), ("up%d.b" % i, (d,))]
        d_in = d
    H = cfg.hidden
    if cfg.pos_enc:
        out += [("pos", (cfg.L, H))]  # R43: right after the upsample (R24 order)
    for l in range(cfg.n_attn):
        if cfg.backbone == "lstm":
            out += [("lstm%d.Wih" % l, (H, 4 * H)), ("lstm%d.bih" % l, (4 * H,)),
                    ("lstm%d.Whh" % l, (H, 4 * H)), ("lstm%d.bhh" % l, (4 * H,))]
            continue
        for nm in ("q", "k", "v", "o"):
            out += [("attn%d.W%s" % (l, nm), (H, H)), ("attn%d.b%s" % (l, nm), (H,))]
    for r in range(cfg.n_res):
        out += [("res%d.Wa" % r, (H, H)), ("res%d.a" % r, (H,)),
                ("res%d.Wb" % r, (H, H)), ("res%d.b" % r, (H,))]
    for t in range(cfg.n_tasks):
        out += [("head%d.W1" % t, (H, cfg.head_dim)), ("head%d.c1" % t, (cfg.head_dim,)),
                ("head%d.w2" % t, (cfg.head_dim, 1)), ("head%d.c2" % t, (1,))]
    return out


def n_params(cfg: Config) -> int:
    return int(sum(np.prod(s) for _, s in param_shapes(cfg)))


def unflatten(cfg: Config, flat: np.ndarray) -> Dict[str, np.ndarray]:
    flat = np.asarray(flat, np.float64)
    p, o = {}, 0
    for name, shp in param_shapes(cfg):
        k = int(np.prod(shp))
        p[name] = flat[o:o + k].reshape(shp).copy()
        o += k
    assert o == flat.size, "flat parameter vector has the wrong length"
    return p


def flatten(cfg: Config, p: Dict[str, np.ndarray]) -> np.ndarray:
    return np.concatenate([np.asarray(p[n], np.float64).ravel() for n, _ in param_shapes(cfg)])


def relu(x):
    return np.maximum(x, 0.0)


def softmax_rows(S):
    """Row softmax, max-subtracted (O2)."""
    m = S.max(axis=-1, keepdims=True)
    e = np.exp(S - m)
    return e / e.sum(axis=-1, keepdims=True)


def sigmoid(x):
    return 0.5 * (1.0 + np.tanh(0.5 * x))


def lstm_forward(p: Dict[str, np.ndarray], pre: str, h: np.ndarray):
    """R49: one LSTM layer over the L rows of every candidate, in order.
    z_t = h_t Wih + bih + hprev Whh + bhh; [i, f, g, o] = [sig, sig, tanh, sig](z_t);
    c_t = f c_{t-1} + i g; hl_t = o tanh(c_t); returns the sequence hl and the
    per-step values backward needs."""
    N, L, H = h.shape
    hp = np.zeros((N, H))
    cp = np.zeros((N, H))
    out = np.zeros((N, L, H))
    steps = []
    for t in range(L):
        z = h[:, t] @ p[pre + "Wih"] + p[pre + "bih"] + hp @ p[pre + "Whh"] + p[pre + "bhh"]
        i, f = sigmoid(z[:, :H]), sigmoid(z[:, H:2 * H])
        g, o = np.tanh(z[:, 2 * H:3 * H]), sigmoid(z[:, 3 * H:])
        c = f * cp + i * g
        hl = o * np.tanh(c)
        steps.append(dict(i=i, f=f, g=g, o=o, c=c, cp=cp, hp=hp))
        out[:, t] = hl
        hp, cp = hl, c
    return out, steps


def lstm_backward(p: Dict[str, np.ndarray], pre: str, h: np.ndarray, steps, dout: np.ndarray,
                  grads: Dict[str, np.ndarray], rms: Optional[Dict[str, np.ndarray]] = None) -> np.ndarray:
    """Backpropagation through time of lstm_forward; returns d h (the input).
    ``rms``: as in backward() (R50)."""
    N, L, H = h.shape
    dh_in = np.zeros_like(h)
    dWih = np.zeros((H, 4 * H)); dWhh = np.zeros((H, 4 * H)); db = np.zeros(4 * H)
    sWih = np.zeros((H, 4 * H)); sWhh = np.zeros((H, 4 * H)); sb = np.zeros(4 * H)
    dhn = np.zeros((N, H))
    dcn = np.zeros((N, H))
    for t in reversed(range(L)):
        st = steps[t]
        dht = dout[:, t] + dhn
        tc = np.tanh(st["c"])
        do = dht * tc
        dc = dcn + dht * st["o"] * (1.0 - tc * tc)
        di, dg, df = dc * st["g"], dc * st["i"], dc * st["cp"]
        dcn = dc * st["f"]
        dz = np.concatenate([di * st["i"] * (1 - st["i"]), df * st["f"] * (1 - st["f"]),
                             dg * (1 - st["g"] ** 2), do * st["o"] * (1 - st["o"])], axis=1)
        dWih += h[:, t].T @ dz
        dWhh += st["hp"].T @ dz
        db += dz.sum(axis=0)
        if rms is not None:
            sWih += (h[:, t] ** 2).T @ dz ** 2
            sWhh += (st["hp"] ** 2).T @ dz ** 2
            sb += (dz ** 2).sum(axis=0)
        dhn = dz @ p[pre + "Whh"].T
        dh_in[:, t] = dz @ p[pre + "Wih"].T
    grads[pre + "Wih"], grads[pre + "Whh"] = dWih, dWhh
    grads[pre + "bih"], grads[pre + "bhh"] = db, db.copy()
    if rms is not None:
        rms[pre + "Wih"], rms[pre + "Whh"] = np.sqrt(sWih), np.sqrt(sWhh)
        rms[pre + "bih"], rms[pre + "bhh"] = np.sqrt(sb), np.sqrt(sb)
    return dh_in


def forward(cfg: Config, p: Dict[str, np.ndarray], X: np.ndarray, save: bool = False):
    """O2.  X [N, L, E] -> scores [N, n_tasks] (float64).  With ``save`` also
    returns the activations backward() needs."""
    h = np.asarray(X, np.float64)
    N, L = h.shape[0], h.shape[1]
    nh, dh, H = cfg.attn_heads, cfg.d_h, cfg.hidden
    # R42: a key is valid unless its input row is all zeros (a padding row)
    key_valid = (h != 0).any(axis=2) if cfg.attn_mask else None
    acts = {"up_in": [], "up_pre": [], "attn": [], "res": []}
    for i in range(len(cfg.up_dims)):
        acts["up_in"].append(h)
        pre = h @ p["up%d.W" % i] + p["up%d.b" % i]
        acts["up_pre"].append(pre)
        h = relu(pre)
    if cfg.pos_enc:
        h = h + p["pos"][None, :L, :]                           # R43
    for l in range(cfg.n_attn if cfg.backbone == "lstm" else 0):
        out, steps = lstm_forward(p, "lstm%d." % l, h)
        acts["attn"].append(dict(h=h, steps=steps))
        h = h + out                                            # R49 (as R10)
    for l in range(cfg.n_attn if cfg.backbone == "attn" else 0):
        pre = "attn%d." % l
        Q = h @ p[pre + "Wq"] + p[pre + "bq"]
        K = h @ p[pre + "Wk"] + p[pre + "bk"]
        V = h @ p[pre + "Wv"] + p[pre + "bv"]
        Qh = Q.reshape(N, L, nh, dh).transpose(0, 2, 1, 3)
        Kh = K.reshape(N, L, nh, dh).transpose(0, 2, 1, 3)
        Vh = V.reshape(N, L, nh, dh).transpose(0, 2, 1, 3)
        S = Qh @ Kh.transpose(0, 1, 3, 2) / np.sqrt(dh)      # R14
        if key_valid is not None:
            S = np.where(key_valid[:, None, None, :], S, -np.inf)
        A = softmax_rows(S)                                    # R8: no mask (R42 optional)
        Oh = A @ Vh
        O = Oh.transpose(0, 2, 1, 3).reshape(N, L, H)
        acts["attn"].append(dict(h=h, Qh=Qh, Kh=Kh, Vh=Vh, A=A, O=O))
        h = h + O @ p[pre + "Wo"] + p[pre + "bo"]             # R10
    for r in range(cfg.n_res):
        pre = "res%d." % r
        v = h @ p[pre + "Wa"] + p[pre + "a"]
        rr = relu(v)
        acts["res"].append(dict(h=h, v=v, r=rr))
        h = h + rr @ p[pre + "Wb"] + p[pre + "b"]              # R12
    acts["h"] = h
    scores = np.zeros((N, cfg.n_tasks))
    heads = []
    for t in range(cfg.n_tasks):
        pre = "head%d." % t
        u = h @ p[pre + "W1"] + p[pre + "c1"]
        z = relu(u)
        per_pos = z @ p[pre + "w2"] + p[pre + "c2"]           # [N, L, 1]
        scores[:, t] = per_pos[..., 0].sum(axis=1)             # R13: sum over L rows
        heads.append(dict(u=u, z=z))
    acts["heads"] = heads
    return (scores, acts) if save else scores


def _w_rms(x, d):
    """sqrt(sum_rows x_r^2 (x) d_r^2): RMS scale of the per-row terms x_r^T d_r of
    a weight gradient sum_r x_r^T d_r (R50)."""
    return np.sqrt(np.einsum("nli,nlo->io", x * x, d * d))


def _b_rms(d):
    return np.sqrt((d * d).sum(axis=(0, 1)))


def backward(cfg: Config, p: Dict[str, np.ndarray], acts, g: np.ndarray,
             rms: Optional[Dict[str, np.ndarray]] = None) -> Dict[str, np.ndarray]:
    """O3.  g = dLoss/dscores [N, n_tasks] -> gradient for every parameter.
    relu'(0) := 0.  Sums over l run over all L rows, pads included.

    Every parameter gradient is a sum over the N*L rows of per-row terms.  If a
    dict is passed as ``rms``, it also receives, per parameter, the root of the
    sum of the squared terms (elementwise) -- the scale at which independent
    per-term rounding errors accumulate, used by the tests to state fp32 error
    bounds for cancelling sums (R50).  The gradients are unaffected."""
    g = np.asarray(g, np.float64)
    R = rms if rms is not None else {}
    track = rms is not None
    nh, dh, H = cfg.attn_heads, cfg.d_h, cfg.hidden
    N, L = acts["h"].shape[0], acts["h"].shape[1]
    grads: Dict[str, np.ndarray] = {}
    h = acts["h"]
    dh_ = np.zeros_like(h)
    for t in range(cfg.n_tasks):
        pre = "head%d." % t
        u, z = acts["heads"][t]["u"], acts["heads"][t]["z"]
        gt = g[:, t][:, None, None]                            # d s_t / d per_pos = 1
        grads[pre + "w2"] = np.einsum("nlk,n->k", z, g[:, t])[:, None]
        grads[pre + "c2"] = np.array([L * g[:, t].sum()])
        du = gt * p[pre + "w2"][:, 0][None, None, :] * (u > 0)
        grads[pre + "W1"] = np.einsum("nli,nlo->io", h, du)
        grads[pre + "c1"] = du.sum(axis=(0, 1))
        if track:
            R[pre + "w2"] = np.sqrt(np.einsum("nlk,n->k", z * z, g[:, t] ** 2))[:, None]
            R[pre + "c2"] = np.array([np.sqrt(L * (g[:, t] ** 2).sum())])
            R[pre + "W1"], R[pre + "c1"] = _w_rms(h, du), _b_rms(du)
        dh_ += du @ p[pre + "W1"].T
    for r in reversed(range(cfg.n_res)):
        pre = "res%d." % r
        a = acts["res"][r]
        grads[pre + "Wb"] = np.einsum("nli,nlo->io", a["r"], dh_)
        grads[pre + "b"] = dh_.sum(axis=(0, 1))
        dv = (dh_ @ p[pre + "Wb"].T) * (a["v"] > 0)
        grads[pre + "Wa"] = np.einsum("nli,nlo->io", a["h"], dv)
        grads[pre + "a"] = dv.sum(axis=(0, 1))
        if track:
            R[pre + "Wb"], R[pre + "b"] = _w_rms(a["r"], dh_), _b_rms(dh_)
            R[pre + "Wa"], R[pre + "a"] = _w_rms(a["h"], dv), _b_rms(dv)
        dh_ = dh_ + dv @ p[pre + "Wa"].T
    for l in reversed(range(cfg.n_attn if cfg.backbone == "lstm" else 0)):
        a = acts["attn"][l]
        dh_ = dh_ + lstm_backward(p, "lstm%d." % l, a["h"], a["steps"], dh_, grads,
                                  R if track else None)
    for l in reversed(range(cfg.n_attn if cfg.backbone == "attn" else 0)):
        pre = "attn%d." % l
        a = acts["attn"][l]
        grads[pre + "Wo"] = np.einsum("nli,nlo->io", a["O"], dh_)
        grads[pre + "bo"] = dh_.sum(axis=(0, 1))
        if track:
            R[pre + "Wo"], R[pre + "bo"] = _w_rms(a["O"], dh_), _b_rms(dh_)
        dO = dh_ @ p[pre + "Wo"].T
        dOh = dO.reshape(N, L, nh, dh).transpose(0, 2, 1, 3)
        A, Qh, Kh, Vh = a["A"], a["Qh"], a["Kh"], a["Vh"]
        dA = dOh @ Vh.transpose(0, 1, 3, 2)
        dVh = A.transpose(0, 1, 3, 2) @ dOh
        dS = A * (dA - (dA * A).sum(axis=-1, keepdims=True))
        dQh = dS @ Kh / np.sqrt(dh)
        dKh = dS.transpose(0, 1, 3, 2) @ Qh / np.sqrt(dh)
        dQ = dQh.transpose(0, 2, 1, 3).reshape(N, L, H)
        dK = dKh.transpose(0, 2, 1, 3).reshape(N, L, H)
        dV = dVh.transpose(0, 2, 1, 3).reshape(N, L, H)
        hin = a["h"]
        for nm, d in (("q", dQ), ("k", dK), ("v", dV)):
            grads[pre + "W" + nm] = np.einsum("nli,nlo->io", hin, d)
            grads[pre + "b" + nm] = d.sum(axis=(0, 1))
            if track:
                R[pre + "W" + nm], R[pre + "b" + nm] = _w_rms(hin, d), _b_rms(d)
        dh_ = dh_ + dQ @ p[pre + "Wq"].T + dK @ p[pre + "Wk"].T + dV @ p[pre + "Wv"].T
    if cfg.pos_enc:
        grads["pos"] = dh_.sum(axis=0)                         # R43: d h / d pos = identity per row
        if track:
            R["pos"] = np.sqrt((dh_ * dh_).sum(axis=0))
    for i in reversed(range(len(cfg.up_dims))):
        pre_ = "up%d." % i
        dpre = dh_ * (acts["up_pre"][i] > 0)
        grads[pre_ + "W"] = np.einsum("nli,nlo->io", acts["up_in"][i], dpre)
        grads[pre_ + "b"] = dpre.sum(axis=(0, 1))
        if track:
            R[pre_ + "W"], R[pre_ + "b"] = _w_rms(acts["up_in"][i], dpre), _b_rms(dpre)
        if i > 0:
            dh_ = dpre @ p[pre_ + "W"].T
    return grads
