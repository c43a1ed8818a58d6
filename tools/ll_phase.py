"""Dev: solve-kernel time of the left-looking LU (PODP_FLAG_LU_LL) at one r, with and without pivoting, for the
library named by PODP_LIB_NAME (ablation builds from tools/ablate_build.sh)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import podp_inputs as g
from paper_2307_05590_b200 import FLAG_LU_LL, FLAG_NO_PIVOT, Evaluator, profile_enable, profile_read
r = int(sys.argv[1]) if len(sys.argv) > 1 else 48
F = int(float(os.environ.get("LU_AB_F", "1e5")))
w = torch.tensor(g.omega_grid(F), device="cuda")
ev = Evaluator(g.make_operators(r))
out = ev.alloc_outputs(F)
for name, fl in (("pivot", FLAG_LU_LL), ("nopivot", FLAG_LU_LL | FLAG_NO_PIVOT)):
    for _ in range(3):
        ev.eval(w, out=out, flags=fl)
    torch.cuda.synchronize()
    profile_enable(True); profile_read(reset=True)
    for _ in range(10):
        ev.eval(w, out=out, flags=fl)
    torch.cuda.synchronize()
    p = profile_read(reset=True); profile_enable(False)
    print(f"{os.environ.get('PODP_LIB_NAME', 'libpodp.so'):22s} r={r} {name:8s} solve {p['solve'][0]/p['solve'][1]:.4f} ms", flush=True)
