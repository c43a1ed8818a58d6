"""Per-CUDA-source-line warp-stall samples from an ncu report (dev tool): python tools/ncu_lines.py rep [top]."""
import re
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
src = {}
res = []
tot = 0
for ln in out.splitlines():
    m = re.match(r'^"(\d+)","(.*)$', ln)
    if not m:
        continue
    parts = m.group(2).split('","')
    try:
        k = parts.index("-")
    except ValueError:
        continue
    if k + 2 >= len(parts) or parts[k + 1] != "-":
        continue
    try:
        samples = int(parts[k + 2])
        inst = int(parts[k + 5])
    except ValueError:
        continue
    code = '","'.join(parts[:k])
    res.append((samples, int(m.group(1)), inst, code.strip()[:90]))
    tot += samples
res.sort(reverse=True)
print(f"total samples {tot}")
for s, line, inst, code in res[:top]:
    print(f"{100.0 * s / max(tot, 1):5.1f}%  L{line:<4d} inst={inst:>11d}  {code}")
