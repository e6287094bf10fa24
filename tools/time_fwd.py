"""Score-only timing of the C2 round (409,600 candidates, 2 layers, bf16) with
CUDA events: python tools/time_fwd.py [reps].  TLP_TC_PAIR / TLP_TC_TRACE are
read by the library at the first launch."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, synth
import paper_2211_03578_b200 as tp
from oracle import model as OM
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
m = tp.TLP(tp.TLPConfig(n_attn=2, precision="bf16"))
m.set_params(np.concatenate([v.ravel() for v in synth.init_params(7, OM.param_shapes(OM.Config(n_attn=2)))]).astype(np.float32))
X = torch.rand((409600, 25, 22), device="cuda")
for _ in range(3):
    s = m.score(X)
m.sync()
ts = []
for _ in range(reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); s = m.score(X); e1.record(); e1.synchronize()
    ts.append(e0.elapsed_time(e1))
ts.sort()
print("score ms: median %.3f min %.3f  (%.2f M cand/s)  pair=%s" % (ts[len(ts) // 2], ts[0], 409600 / ts[len(ts) // 2] / 1e3, os.environ.get("TLP_TC_PAIR", "0")))
