"""Run a few C3-shape training steps (16 groups x 512) for ncu launch lists."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth, oracle
import paper_2211_03578_b200 as tp
from oracle import model as OM
prec = sys.argv[1] if len(sys.argv) > 1 else "bf16"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
m = tp.TLP(tp.TLPConfig(n_attn=1, precision=prec))
flat = np.concatenate([v.ravel() for v in synth.init_params(8, OM.param_shapes(OM.Config()))]).astype(np.float32)
m.set_params(flat)
G, P = 16, 512
b = synth.generate(5, G * P)
goff = np.arange(G + 1, dtype=np.int64) * P
tokens = oracle.build_token_table(synth.training_stream())
m.set_token_table(sorted(tokens, key=tokens.get))
m.set_norm_scales(np.ones(22, np.float32) * 8)
X = m.encode(tp.DeviceBatch.from_packed(b))
lat = torch.from_numpy(synth.latencies(b, goff, 3).astype(np.float32)).cuda()
y = m.normalize_labels(lat, goff).view(-1, 1).contiguous()
for _ in range(steps):
    m.train_step(X, y, goff)
m.sync()
print("ok")
