"""Kernel timeline of C3 training steps (torch.profiler / CUPTI activity
records): per-kernel device time and the idle gaps between consecutive kernels
of a step (diagnostics): python tools/gap_train.py"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth, oracle
import paper_2211_03578_b200 as tp
from oracle import model as OM
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
for _ in range(5):
    m.train_step(X, y, goff)
m.sync()
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(3):
        m.train_step(X, y, goff)
    m.sync()
prof.export_chrome_trace("/tmp/tr.json")
ev = [e for e in json.load(open("/tmp/tr.json"))["traceEvents"] if e.get("cat") == "kernel"]
ev.sort(key=lambda e: e["ts"])
# last step: from the last pair_count_kernel on
starts = [i for i, e in enumerate(ev) if e["name"].startswith("pair_count") or "pair_count" in e["name"]]
seg = ev[starts[-1]:]
t0 = seg[0]["ts"]; t1 = seg[-1]["ts"] + seg[-1]["dur"]
busy = sum(e["dur"] for e in seg)
print("kernels %d  span %.1f us  busy %.1f us  gaps %.1f us" % (len(seg), t1 - t0, busy, t1 - t0 - busy))
prev = None
for e in seg:
    gap = e["ts"] - (prev["ts"] + prev["dur"]) if prev else 0.0
    print("%7.1f gap %5.1f  %s" % (e["dur"], gap, e["name"].split("(")[0][-40:]))
    prev = e
