"""Warp-state samples of one kernel attributed to its phases through the inline call chain (dev tool).

  python tools/ncu_phase.py REP.ncu-rep OBJECT.o MANGLED_SUBSTRING [ncu -k filter]

ncu's source page gives per-SASS-instruction samples but only the innermost source line, which for a kernel made of
inlined device functions (cfms, dmma, ...) says nothing about the phase.  nvdisasm -gi on the same object gives the
whole "inlined at" chain per instruction; the two are joined by instruction offset.  The report groups samples and
executed instructions by the line of the outermost call inside the per-frequency lambda (column_tile / panel<2> /
panel<1> / finish) and by the line one level below."""
import csv
import os
import re
import subprocess
import sys
import tempfile
from collections import Counter

rep, obj, sub = sys.argv[1:4]
kfilt = sys.argv[4] if len(sys.argv) > 4 else None
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=tmp, check=True, capture_output=True)
cubin = [f for f in os.listdir(tmp) if f.endswith(".cubin")][0]
dis = subprocess.run(["nvdisasm", "-gi", cubin], cwd=tmp, capture_output=True, text=True).stdout.splitlines()
start = next(i for i, l in enumerate(dis) if l.startswith(".text.") and sub in l)
end = next((i for i in range(start + 1, len(dis)) if dis[i].startswith("//--------------------- .text")), len(dis))
off2chain, cur, new = {}, [], True
for ln in dis[start:end]:
    m = re.match(r'\s*//## File "([^"]+)", line (\d+)', ln)
    if m:
        if new:
            cur, new = [], False
        cur.append(int(m.group(2)))
        continue
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?);", ln)
    if m:
        new = True
        off2chain[int(m.group(1), 16)] = list(cur)
outer = Counter(c[-1] for c in off2chain.values() if c).most_common(1)[0][0]  # the per-frequency lambda's call
src_lines = open(next(l for l in dis[start:end] if "//## File" in l).split('"')[1]).read().splitlines()
cmd = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"] + (["-k", kfilt] if kfilt else [])
rows = list(csv.reader(subprocess.run(cmd, capture_output=True, text=True).stdout.splitlines()))
h = rows[1]
ix = {n: i for i, n in enumerate(h)}
body = [r for r in rows[2:] if len(r) >= len(h)]
base = int(body[0][0], 16)
S, I, S2, I2 = Counter(), Counter(), Counter(), Counter()
for r in body:
    ch = off2chain.get(int(r[0], 16) - base, [])
    s, n = int(r[ix["Warp Stall Sampling (All Samples)"]]), int(r[ix["Instructions Executed"]])
    if ch and ch[-1] == outer and len(ch) >= 2:
        k, k2 = ch[-2], (ch[-3] if len(ch) > 2 else None)
    else:
        k, k2 = "outside", (ch[-1] if ch else None)
    S[k] += s
    I[k] += n
    S2[(k, k2)] += s
    I2[(k, k2)] += n
T = sum(S.values())


def text(line):
    return src_lines[line - 1].strip()[:90] if isinstance(line, int) and 0 < line <= len(src_lines) else ""


print(f"kernel {sub}: {T} samples, {sum(I.values())} warp instructions; per-frequency call at line {outer}")
for k, v in S.most_common(10):
    print(f"{100 * v / T:5.1f} %  inst {I[k]:>12d}  L{k}  {text(k)}")
print("-- one level below")
for (k, k2), v in S2.most_common(40):
    print(f"{100 * v / T:5.1f} %  inst {I2[(k, k2)]:>12d}  L{k} > L{k2}  {text(k2)}")
