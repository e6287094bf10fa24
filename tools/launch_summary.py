"""Summarise an ncu --metrics gpu__time_duration.sum[,dram__bytes_*] launch list CSV:
python tools/launch_summary.py gpurun_out/x.csv [--each]"""
import csv, sys
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 5]
hdr = rows[0]
ki, mi, vi, ii = (hdr.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "ID"))
d = {}
for r in rows[1:]:
    d.setdefault(r[ii], {})[r[mi]] = float(r[vi].replace(",", ""))
    d[r[ii]]["k"] = r[ki].split("(")[0].replace("<unnamed>::", "").replace("void ", "")[:34]
tot = {}
for v in d.values():
    t = tot.setdefault(v["k"], [0.0, 0, 0.0])
    t[0] += v["gpu__time_duration.sum"]; t[1] += 1
    t[2] += v.get("dram__bytes_read.sum", 0) + v.get("dram__bytes_write.sum", 0)
print("sum %.3f ms over %d launches" % (sum(t[0] for t in tot.values()) / 1e6, len(d)))
for k, t in sorted(tot.items(), key=lambda kv: -kv[1][0]):
    print("  %-36s %9.1f us  n=%-3d %6.2f TB/s" % (k, t[0] / 1e3, t[1], t[2] / t[0] / 1e3 if t[0] else 0))
if "--each" in sys.argv:
    for v in d.values():
        print("    %-36s %9.1f us" % (v["k"], v["gpu__time_duration.sum"] / 1e3))
