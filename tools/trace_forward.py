import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["TLP_TC_TRACE"] = "1"
import numpy as np, torch, synth
import paper_2211_03578_b200 as tp
from oracle import model as OM
n_attn = int(sys.argv[1]) if len(sys.argv) > 1 else 2
m = tp.TLP(tp.TLPConfig(n_attn=n_attn))
m.set_params(np.concatenate([v.ravel() for v in synth.init_params(7, OM.param_shapes(OM.Config(n_attn=n_attn)))]).astype(np.float32))
X = torch.rand((409600, 25, 22), device="cuda")
for _ in range(2):
    m.score(X)
m.sync()
