"""Summarise a round's ncu captures (gpurun_out/<tag>_*) into profiles/<tag>_*.

    python tools/summarize_profiles.py r01

Writes profiles/<tag>_launches.csv (kernel, ms, share of the step) and
profiles/<tag>_kernels.md (per kernel: duration, DRAM bytes, tensor-pipe %,
achieved occupancy, top stall reasons) and profiles/<tag>_traffic.json (DRAM
bytes per launch of each captured kernel, read by bench.py's roofline).
"""
from __future__ import annotations

import collections
import csv
import io
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GO = os.path.join(ROOT, "gpurun_out")
PR = os.path.join(ROOT, "profiles")


def short(name: str) -> str:
    m = re.search(r"(\w+_kernel\w*|\w+_partial\w*|reduce_partials|label_kernel|finalize_\w+|sum_counts|resolve_tokens|pack_kernel|lstm_cell_\w+)", name)
    k = m.group(1) if m else name.split("(")[0][:40]
    t = re.search(r"<([^>]*)>", name)
    if t and ("gemm" in k or "attn" in k or "encode" in k):
        k += "<" + t.group(1) + ">"
    return k


def launches(tag: str):
    path = os.path.join(GO, tag + "_launches.csv")
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[start]
    ik, iv = hdr.index("Kernel Name"), hdr.index("Metric Value")
    data = rows[start + 1:]
    agg, cnt = collections.OrderedDict(), collections.Counter()
    # the bench does 3 warm-up steps + 1 timed step (+ the e2e passes); take
    # the launches of the timed step: from the encode (resolve_tokens /
    # encode_*) that starts the round of the 4th tc_forward to the launch
    # before the next step's encode -- the round (encode, fused forward, top-k)
    # and the training step that follows it
    fwd = [i for i, r in enumerate(data) if "tc_forward_kernel" in r[ik]]
    k4 = fwd[3] if len(fwd) > 3 else (fwd[-1] if fwd else 0)
    starts = [i for i, r in enumerate(data) if "resolve_tokens" in r[ik] or "encode_" in r[ik]]
    lo = max([i for i in starts if i < k4] or [0])
    while lo > 0 and ("resolve_tokens" in data[lo - 1][ik]):
        lo -= 1
    hi = min([i for i in starts if i > k4] or [len(data)])
    for r in data[lo:hi]:
        k = short(r[ik])
        agg[k] = agg.get(k, 0.0) + float(r[iv].replace(",", ""))
        cnt[k] += 1
    tot = sum(agg.values())
    out = io.StringIO()
    w = csv.writer(out)
    w.writerow(["kernel", "launches", "total_ms", "share_of_step"])
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1]):
        w.writerow([k, cnt[k], "%.4f" % (v / 1e6), "%.4f" % (v / tot)])
    return out.getvalue(), tot


def tune_round_launches(tag: str):
    """Launch list of one NEXT-1 device tuning round (tlp_ga_round): the
    launches between the last two ga_init_kernel launches of the bench."""
    path = os.path.join(GO, tag + "_launches.csv")
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[start]
    ik, iv = hdr.index("Kernel Name"), hdr.index("Metric Value")
    data = rows[start + 1:]
    inits = [i for i, r in enumerate(data) if "ga_init_kernel" in r[ik]]
    if len(inits) < 2:
        return None
    agg, cnt = collections.OrderedDict(), collections.Counter()
    for r in data[inits[-2]:inits[-1]]:
        k = short(r[ik])
        agg[k] = agg.get(k, 0.0) + float(r[iv].replace(",", ""))
        cnt[k] += 1
    tot = sum(agg.values())
    out = io.StringIO()
    w = csv.writer(out)
    w.writerow(["kernel", "launches", "total_ms", "share_of_round"])
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1]):
        w.writerow([k, cnt[k], "%.4f" % (v / 1e6), "%.4f" % (v / tot)])
    return out.getvalue()


def raw_metrics(rep: str):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    if len(rows) < 3:
        return {}
    return {h: (u, v) for h, u, v in zip(rows[0], rows[1], rows[2])}


def to_bytes(u, v):
    x = float(v.replace(",", ""))
    return x * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)


def kernels(tag: str):
    md = ["# %s ncu --set full summaries (one launch each, --clock-control none)\n" % tag,
          "| kernel | duration | DRAM read | DRAM write | DRAM GB/s | tensor pipe % | occupancy % | top stalls |",
          "|---|---|---|---|---|---|---|---|"]
    traffic = {}
    for f in sorted(os.listdir(GO)):
        if not (f.startswith(tag + "_prof_") and f.endswith(".ncu-rep")):
            continue
        k = f[len(tag + "_prof_"):-len(".ncu-rep")]
        m = raw_metrics(os.path.join(GO, f))
        if not m:
            continue
        dur_u, dur_v = m.get("gpu__time_duration.sum", ("", "0"))
        dur_s = float(dur_v.replace(",", "")) * {"ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3}.get(dur_u, 1e-9)
        rd = to_bytes(*m.get("dram__bytes_read.sum", ("byte", "0")))
        wr = to_bytes(*m.get("dram__bytes_write.sum", ("byte", "0")))
        tp = m.get("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", ("", "n/a"))[1]
        occ = m.get("sm__warps_active.avg.pct_of_peak_sustained_active", ("", "n/a"))[1]
        st = [(h.replace("smsp__pcsamp_warps_issue_stalled_", ""), float(v[1] or 0)) for h, v in m.items()
              if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued")]
        tots = sum(x for _, x in st) or 1.0
        top = ", ".join("%s %.0f%%" % (a, 100 * b / tots) for a, b in sorted(st, key=lambda x: -x[1])[:3])
        md.append("| %s | %.3f ms | %.1f MB | %.1f MB | %.0f | %s | %s | %s |" % (
            k, dur_s * 1e3, rd / 1e6, wr / 1e6, (rd + wr) / max(dur_s, 1e-12) / 1e9, tp, occ, top))
        traffic[k] = {"dram_read_bytes": rd, "dram_write_bytes": wr, "duration_s": dur_s}
    return "\n".join(md) + "\n", traffic


def main():
    tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
    os.makedirs(PR, exist_ok=True)
    csv_txt, tot = launches(tag)
    open(os.path.join(PR, tag + "_launches.csv"), "w").write(csv_txt)
    tr = tune_round_launches(tag)
    if tr:
        open(os.path.join(PR, tag + "_tune_round_launches.csv"), "w").write(tr)
        print(tr)
    md, traffic = kernels(tag)
    open(os.path.join(PR, tag + "_kernels.md"), "w").write(md)
    json.dump(traffic, open(os.path.join(PR, tag + "_traffic.json"), "w"), indent=1)
    print(csv_txt)
    print(md)


if __name__ == "__main__":
    main()
