"""Two tlp_score launches of the C2 round (409,600 candidates, 2 layers) for ncu:
    ncu --set full -k regex:tc_forward -s 1 -c 1 -o OUT python tools/profile_fwd.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, synth
import paper_2211_03578_b200 as tp
from oracle import model as OM
m = tp.TLP(tp.TLPConfig(n_attn=2))
m.set_params(np.concatenate([v.ravel() for v in synth.init_params(7, OM.param_shapes(OM.Config(n_attn=2)))]).astype(np.float32))
X = torch.rand((409600, 25, 22), device="cuda")
for _ in range(2):
    m.score(X)
m.sync()
