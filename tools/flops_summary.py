"""Executed FP64 work per kernel from an ncu --metrics CSV (DFMA x2 + DMUL + DADD per thread instruction, DMMA
warp instructions x 512 flops) next to its duration (dev tool)."""
import csv
import sys
from collections import defaultdict

for path in sys.argv[1:]:
    lines = open(path).read().splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
    per = defaultdict(dict)
    for r in csv.DictReader(lines[start:]):
        per[(int(r["ID"]), r["Kernel Name"])][r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
    print("==", path)
    for (i, name), m in sorted(per.items()):
        t = m.get("gpu__time_duration.sum", 0.0) * 1e-9
        fl = (2 * m.get("smsp__sass_thread_inst_executed_op_dfma_pred_on.sum", 0)
              + m.get("smsp__sass_thread_inst_executed_op_dmul_pred_on.sum", 0)
              + m.get("smsp__sass_thread_inst_executed_op_dadd_pred_on.sum", 0))
        dm = 512 * m.get("sm__inst_executed_pipe_tensor_subpipe_dmma.sum", 0)
        print(f"  {name[:48]:48s} {t * 1e3:9.3f} ms  exec {(fl + dm) / 1e9:9.3f} GFLOP (dmma {dm / max(fl + dm, 1):4.0%})"
              f"  {(fl + dm) / max(t, 1e-12) / 1e12:6.2f} TF/s  fp64 pipe {m.get('sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active', 0):5.1f}%"
              f"  tensor {m.get('sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active', 0):5.1f}%"
              f"  dram {(m.get('dram__bytes_read.sum', 0) + m.get('dram__bytes_write.sum', 0)) / 1e6:8.2f} MB")
