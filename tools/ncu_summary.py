"""Summarise an ncu report: key metrics, stall reasons, and SASS opcode mix (dev tool)."""
import csv, subprocess, sys
from collections import Counter

rep = sys.argv[1]
kfilter = sys.argv[2] if len(sys.argv) > 2 else None
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
hdr = rows[0]
for r in rows[2:]:
    d = dict(zip(hdr, r))
    if kfilter and kfilter not in d.get("Kernel Name", ""):
        continue
    print("==", d.get("Kernel Name", "")[:80])
    for k in ["gpu__time_duration.sum", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
              "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
              "smsp__thread_inst_executed_per_inst_executed.ratio", "sm__warps_active.avg.per_cycle_active",
              "launch__registers_per_thread", "dram__bytes_read.sum", "dram__bytes_write.sum",
              "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
              "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"]:
        if k in d:
            print(f"  {k:70s} {d[k]}")
    st = []
    for k, v in d.items():
        if "warps_issue_stalled" in k and k.endswith("per_issue_active.ratio"):
            try:
                st.append((float(v.replace(",", "")), k.split("stalled_")[1].split("_per")[0]))
            except ValueError:
                pass
    print("  stalls/issue:", ", ".join(f"{n}={v:.2f}" for v, n in sorted(st, reverse=True) if v > 0.05))
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"] +
                     (["-k", kfilter] if kfilter else []), capture_output=True, text=True).stdout
rows = list(csv.reader(src.splitlines()))
if len(rows) > 2:
    hdr = rows[1]
    ie = hdr.index("Instructions Executed")
    ss = hdr.index("Warp Stall Sampling (All Samples)")
    c, s = Counter(), Counter()
    tot = 0
    for r in rows[2:]:
        if len(r) <= ie or not r[ie].isdigit():
            continue
        t = r[1].strip().split()
        if not t:
            continue
        op = t[1] if t[0].startswith("@") else t[0]
        op = op.split(".")[0]
        c[op] += int(r[ie]); s[op] += int(r[ss]) if r[ss].isdigit() else 0
        tot += int(r[ie])
    stot = sum(s.values()) or 1
    print("  opcode mix (executed %, stall-sample %):")
    print("   " + ", ".join(f"{op}={n/tot*100:.1f}/{s[op]/stot*100:.0f}" for op, n in c.most_common(18)))
