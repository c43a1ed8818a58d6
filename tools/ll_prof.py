"""Dev: two podp_eval calls with the left-looking LU forced (for ncu on a dev library via PODP_LIB_NAME)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import podp_inputs as g
from paper_2307_05590_b200 import FLAG_LU_LL, Evaluator
r = int(sys.argv[1]) if len(sys.argv) > 1 else 48
F = int(sys.argv[2]) if len(sys.argv) > 2 else 20000
ev = Evaluator(g.make_operators(r))
w = torch.tensor(g.omega_grid(F), device="cuda")
out = ev.alloc_outputs(F)
for _ in range(2):
    ev.eval(w, out=out, flags=FLAG_LU_LL)
torch.cuda.synchronize()
print("ok")
