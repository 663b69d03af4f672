"""Summarise an `ncu --metrics gpu__time_duration.sum,dram__bytes_* --csv` launch
list of N identical pipeline steps: per-kernel launches, time, share, DRAM MB
(per step).  Usage: launch_summary.py launches.csv steps title > out.txt"""
import csv
import sys
from collections import defaultdict

path, steps, title = sys.argv[1], int(sys.argv[2]), sys.argv[3]
rows = [r for r in csv.reader(l for l in open(path) if l.startswith('"'))]
h = rows[0]
ix = {k: i for i, k in enumerate(h)}
launch = defaultdict(dict)
for r in rows[1:]:
    launch[r[ix["ID"]]][r[ix["Metric Name"]]] = (r[ix["Kernel Name"]], float(r[ix["Metric Value"]].replace(",", "")),
                                                 r[ix["Metric Unit"]])
agg = defaultdict(lambda: [0, 0.0, 0.0])
for lid, m in launch.items():
    name, t, unit = m["gpu__time_duration.sum"]
    scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "nsecond": 1e-6}.get(unit, 1e-6)
    by = sum(m[k][1] * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(m[k][2], 1)
             for k in ("dram__bytes_read.sum", "dram__bytes_write.sum") if k in m)
    name = name.split("(")[0].replace("void ", "").replace("bltc::", "").replace("<unnamed>::", "")
    a = agg[name]
    a[0] += 1
    a[1] += t * scale
    a[2] += by
tot = sum(a[1] for a in agg.values())
print(f"# {title}")
print("# ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none")
print("# (cold-cache, serialised launches: compare SHARES, not absolute times); per-step figures")
print(f"# launches per step: {sum(a[0] for a in agg.values()) / steps:.0f}   kernel time per step: {tot / steps:.1f} ms")
print(f"{'kernel':60s} {'n':>5s} {'ms':>10s} {'share':>7s} {'dram MB':>9s}")
for name, a in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{name[:60]:60s} {a[0] / steps:5.0f} {a[1] / steps:10.3f} {100 * a[1] / tot:6.2f}% {a[2] / steps / 1e6:9.1f}")
