"""Small end-to-end run of every kernel for compute-sanitizer (memcheck /
racecheck / synccheck): encode -> score (fp32 + bf16 fused, with and without the
padding mask / positional table) -> top-k -> labels -> train steps (LambdaRank
and MSE; fp32 and bf16 contexts, incl. the B-image and wgrad GEMMs) -> top-k
merge -> tlp_search_round -> tlp_dedup -> tlp_topk_score; a 2,500-row bf16
train step (fused wgrad + bias kernels, 1 and 4 heads); token-table / scale
fitting; NEXT-1 device tuning rounds (fp32 and bf16 scoring) and NEXT-4 LSTM
contexts (score + train)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import synth
import oracle
from oracle import model as OM
import paper_2211_03578_b200 as tp

tokens = oracle.build_token_table(synth.training_stream(n=200))
names = sorted(tokens, key=tokens.get)
b = synth.generate(3, 23)
off = np.array([0, 7, 15, 23], np.int64)
lat = torch.from_numpy(synth.latencies(b, off, 1).astype(np.float32)).cuda()
cases = [("fp32", OM.Config(hidden=64, up_dims=(32, 64), head_dim=32), {}),
         ("bf16", OM.Config(n_attn=2, n_tasks=2), {}),
         ("bf16", OM.Config(n_attn=1, n_tasks=1, attn_mask=True, pos_enc=True), {"loss": "mse"})]
for prec, cfg, extra in cases:
    m = tp.TLP(tp.TLPConfig(hidden=cfg.hidden, up_dims=cfg.up_dims, head_dim=cfg.head_dim,
                            n_attn=cfg.n_attn, n_tasks=cfg.n_tasks, precision=prec,
                            attn_mask=cfg.attn_mask, pos_enc=cfg.pos_enc, **extra))
    m.set_token_table(names)
    m.set_norm_scales(np.full(22, 8.0, np.float32))
    m.set_params(np.concatenate([v.ravel() for v in synth.init_params(1, OM.param_shapes(cfg))]).astype(np.float32))
    db = tp.DeviceBatch.from_packed(b)
    X = m.encode(db)
    s = m.score(X)
    idx, val = m.topk(s, off, 4)
    y = m.normalize_labels(lat, off).view(-1, 1).repeat(1, cfg.n_tasks).contiguous()
    m.train_step(X, y, off)
    m.topk_merge(torch.stack([val, val]), torch.stack([idx, idx]))
    if prec == "bf16":
        m.search_round(tp.DeviceBatch.from_packed(b, pin=True), off, 4, chunks=3)
    m.dedup(X, off, y[:, 0].contiguous())
    m.topk_score(s, lat, off, [1.0, 2.0, 1.0], 2)
    m.sync()
# the training GEMM variants at their real shapes (N = 256 tiles, 256 x 256
# wgrad): 100 samples = 2,500 rows > one 2,048-row slice, so the fused
# wgrad + bias-sum kernel (J = 1 and the J = 3 Q/K/V launch) and the slice
# reduction run, as in the benched step; MTL-4 heads
for nt in (1, 4):
    bcfg = OM.Config(n_tasks=nt)
    big = tp.TLP(tp.TLPConfig(n_attn=1, n_tasks=nt))
    big.set_params(np.concatenate([v.ravel() for v in synth.init_params(2, OM.param_shapes(bcfg))]).astype(np.float32))
    Xb = torch.rand((100, 25, 22), device="cuda")
    yb = torch.rand((100, nt), device="cuda") + 0.01
    big.train_step(Xb, yb, np.array([0, 50, 100], np.int64))
    big.sync()
# R1 / R3 fitted on the device
fit = tp.TLP(tp.TLPConfig(precision="fp32"))
tb = synth.generate(9, 50, unseen_rate=0.0)
fit.fit_token_table(tb)
fit.fit_norm_scales(tp.DeviceBatch.from_packed(tb))
fit.sync()
# NEXT-1: device tuning rounds (GA kernels + dedup + materialise -> encode -> score -> top-k)
ts = [synth.make_template(5, s) for s in range(3)] + [synth.small_template((2, 3))]
for prec, cfg in (("fp32", OM.Config(hidden=64, up_dims=(32, 64), head_dim=32)), ("bf16", OM.Config(n_attn=2))):
    m = tp.TLP(tp.TLPConfig(hidden=cfg.hidden, up_dims=cfg.up_dims, head_dim=cfg.head_dim,
                            n_attn=cfg.n_attn, precision=prec))
    m.set_token_table(names)
    m.set_norm_scales(np.full(22, 8.0, np.float32))
    m.set_params(np.concatenate([v.ravel() for v in synth.init_params(3, OM.param_shapes(cfg))]).astype(np.float32))
    m.ga_set_space(synth.pack_space(ts), id_base=2)
    m.ga_round(8, 24, 2, 0.5, 0.3, seed=1, rnd=0)
    m.sync()
# NEXT-4: LSTM contexts
for prec in ("fp32", "bf16"):
    cfg = OM.Config(hidden=64, up_dims=(32, 64), head_dim=32, n_attn=2, backbone="lstm")
    m = tp.TLP(tp.TLPConfig(hidden=64, up_dims=(32, 64), head_dim=32, n_attn=2, precision=prec,
                            backbone="lstm"))
    m.set_params(np.concatenate([v.ravel() for v in synth.init_params(4, OM.param_shapes(cfg))]).astype(np.float32))
    Xl = torch.rand((23, 25, 22), device="cuda")
    m.score(Xl)
    m.train_step(Xl, torch.rand((23, 1), device="cuda") + 0.01, off)
    m.sync()
print("sanitize smoke ok")
