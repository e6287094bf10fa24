"""C4-shape MTL training step timing (4 heads, 1 attention layer, 16 groups x 512,
target-head labels on 7%, bf16): python tools/time_c4.py [reps]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth, oracle
import paper_2211_03578_b200 as tp
from oracle import model as OM
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
cfg = tp.TLPConfig(n_attn=1, n_tasks=4, precision="bf16")
m = tp.TLP(cfg)
m.set_params(np.concatenate([v.ravel() for v in synth.init_params(10, cfg.param_shapes())]).astype(np.float32))
tokens = oracle.build_token_table(synth.training_stream())
m.set_token_table(sorted(tokens, key=tokens.get))
m.set_norm_scales(np.ones(22, np.float32) * 8)
G, P = 16, 512
b = synth.generate(3000, G * P)
goff = np.arange(G + 1, dtype=np.int64) * P
X = m.encode(tp.DeviceBatch.from_packed(b))
lab = np.stack([synth.latencies(b, goff, 40, task_noise=0.3 * (t > 0)) for t in range(4)], 1)
y = np.stack([oracle.normalize_labels(lab[:, t], goff) for t in range(4)], 1).astype(np.float32)
y[np.random.default_rng(41).random(G * P) >= 0.07, 0] = np.nan
yd = torch.from_numpy(y).cuda()
for _ in range(3):
    m.train_step(X, yd, goff)
m.sync()
ts = []
for _ in range(reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); m.train_step(X, yd, goff); e1.record(); e1.synchronize()
    ts.append(e0.elapsed_time(e1))
ts.sort()
print("c4 train ms: median %.3f min %.3f" % (ts[len(ts) // 2], ts[0]))
