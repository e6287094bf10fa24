"""C3-shape training step timing (16 groups x 512 = 8,192 samples, 1 attention
layer, bf16 tensor-core path) with CUDA events: python tools/time_train.py [reps]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth, oracle
import paper_2211_03578_b200 as tp
from oracle import model as OM
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
m = tp.TLP(tp.TLPConfig(n_attn=1, precision="bf16"))
m.set_params(np.concatenate([v.ravel() for v in synth.init_params(8, OM.param_shapes(OM.Config()))]).astype(np.float32))
G, P = 16, 512
b = synth.generate(5, G * P)
goff = np.arange(G + 1, dtype=np.int64) * P
tokens = oracle.build_token_table(synth.training_stream())
m.set_token_table(sorted(tokens, key=tokens.get))
m.set_norm_scales(np.ones(22, np.float32) * 8)
X = m.encode(tp.DeviceBatch.from_packed(b))
lat = torch.from_numpy(synth.latencies(b, goff, 3).astype(np.float32)).cuda()
y = m.normalize_labels(lat, goff).view(-1, 1).contiguous()
for _ in range(3):
    loss = m.train_step(X, y, goff)
m.sync()
ts = []
for _ in range(reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); loss = m.train_step(X, y, goff); e1.record(); e1.synchronize()
    ts.append(e0.elapsed_time(e1))
ts.sort()
print("train ms: median %.3f min %.3f  (%.0f K samples/s)  loss %.6f" % (ts[len(ts) // 2], ts[0], G * P / ts[len(ts) // 2], float(loss)))
