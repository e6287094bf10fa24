"""Small end-to-end run of every kernel for compute-sanitizer (memcheck /
racecheck / synccheck):  encode -> score (fp32 + bf16 fused) -> top-k ->
labels -> LambdaRank train step (fp32 and bf16 contexts) -> top-k merge."""
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
for prec, cfg in (("fp32", OM.Config(hidden=64, up_dims=(32, 64), head_dim=32)),
                  ("bf16", OM.Config(n_attn=2, n_tasks=2))):
    m = tp.TLP(tp.TLPConfig(hidden=cfg.hidden, up_dims=cfg.up_dims, head_dim=cfg.head_dim,
                            n_attn=cfg.n_attn, n_tasks=cfg.n_tasks, precision=prec))
    m.set_token_table(names)
    m.set_norm_scales(np.full(22, 8.0, np.float32))
    m.set_params(np.concatenate([v.ravel() for v in synth.init_params(1, OM.param_shapes(cfg))]).astype(np.float32))
    X = m.encode(tp.DeviceBatch.from_packed(b))
    s = m.score(X)
    idx, val = m.topk(s, off, 4)
    y = m.normalize_labels(lat, off).view(-1, 1).repeat(1, cfg.n_tasks).contiguous()
    m.train_step(X, y, off)
    m.topk_merge(torch.stack([val, val]), torch.stack([idx, idx]))
    m.sync()
print("sanitize smoke ok")
