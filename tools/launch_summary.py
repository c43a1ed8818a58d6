"""Summarise an ncu --csv launch list (gpu__time_duration, dram bytes) per kernel name (dev tool)."""
import csv
import sys
from collections import defaultdict

lines = open(sys.argv[1]).read().splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
rows = list(csv.DictReader(lines[start:]))
per = defaultdict(dict)
for r in rows:
    per[(int(r["ID"]), r["Kernel Name"])][r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
agg = defaultdict(lambda: [0, 0.0, 0.0, 0.0])
for (_i, name), m in per.items():
    a = agg[name[:70]]
    a[0] += 1
    a[1] += m.get("gpu__time_duration.sum", 0.0)
    a[2] += m.get("dram__bytes_read.sum", 0.0)
    a[3] += m.get("dram__bytes_write.sum", 0.0)
tot = sum(a[1] for a in agg.values())
for name, a in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{name:70s} n={a[0]:3d} avg_us={a[1] / a[0] / 1e3:9.2f} share={100 * a[1] / tot:5.1f}% "
          f"dram_rd_MB={a[2] / a[0] / 1e6:8.2f} dram_wr_MB={a[3] / a[0] / 1e6:8.2f} (per launch)")
