"""tlp_encode timing on the C2 round (409,600 synthetic TenSet-shaped candidates)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth, oracle
import paper_2211_03578_b200 as tp
m = tp.TLP(tp.TLPConfig(n_attn=2, precision="bf16"))
tokens = oracle.build_token_table(synth.training_stream())
m.set_token_table(sorted(tokens, key=tokens.get))
m.set_norm_scales(np.ones(22, np.float32) * 8)
db = tp.DeviceBatch.from_packed(synth.generate(11, 409600))
for _ in range(3):
    X = m.encode(db)
m.sync()
ts = []
for _ in range(20):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); X = m.encode(db); e1.record(); e1.synchronize()
    ts.append(e0.elapsed_time(e1))
ts.sort()
print("encode ms: median %.4f min %.4f" % (ts[len(ts) // 2], ts[0]))
