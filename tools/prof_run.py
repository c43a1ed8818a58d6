"""Small driver for ncu: a few podp_eval calls on one BASELINE config (dev tool)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import podp_inputs as g
from paper_2307_05590_b200 import Evaluator

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 2
F = int(sys.argv[3]) if len(sys.argv) > 3 else None
c = g.make_config(cfg, F=F)
ev = Evaluator(c["ops"])
w = torch.tensor(c["omega"], device="cuda")
out = ev.alloc_outputs(len(c["omega"]))
for _ in range(iters):
    ev.eval(w, out=out)
torch.cuda.synchronize()
print("ok")
