"""Summarise an ncu --set full report of one kernel: stall reasons and the
hottest SASS lines with their source line (diagnostics).
    python tools/ncu_hot.py REPORT.ncu-rep [N] [sass|cuda] [LAUNCH_INDEX]"""
import csv, io, subprocess, sys
rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
sel = ["--launch-skip", sys.argv[4], "--launch-count", "1"] if len(sys.argv) > 4 else []
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source",
                      sys.argv[3] if len(sys.argv) > 3 else "sass"] + sel,
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr_i = next(i for i, r in enumerate(rows) if r and r[0] == "Address" or (len(r) > 1 and r[1] == "Source"))
h = rows[hdr_i]
idx = {k: i for i, k in enumerate(h)}
data = [r for r in rows[hdr_i + 1:] if len(r) == len(h)]
S = "Warp Stall Sampling (All Samples)"
stalls = [k for k in h if k.startswith("stall_") and "Not Issued" not in k]
tot = {k: 0 for k in stalls}
allS = 0
def iv(x):
    try: return int(float(x))
    except Exception: return 0
for r in data:
    allS += iv(r[idx[S]])
    for k in stalls: tot[k] += iv(r[idx[k]])
print("samples", allS)
for k, v in sorted(tot.items(), key=lambda x: -x[1])[:10]:
    print("  %-28s %5.1f%%" % (k, 100.0 * v / max(allS, 1)))
for r in sorted(data, key=lambda r: -iv(r[idx[S]]))[:n]:
    best = max(stalls, key=lambda k: iv(r[idx[k]]))
    print("%6.2f%% %-24s %s" % (100.0 * iv(r[idx[S]]) / max(allS, 1), best, r[idx["Source"]][:100]))
