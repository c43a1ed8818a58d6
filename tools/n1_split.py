"""Dev: kernel split of the literal per-direction path (N1) vs the embedding, F = 1e5."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import podp_inputs as g
import paper_2307_05590_b200 as pb
from paper_2307_05590_b200 import perdir as pdir
F = 100_000
w = torch.tensor(g.omega_grid(F), device="cuda")
for mm in ((16, 16, 16), (24, 16, 8), (8, 8, 8), (32, 32, 32)):
    b = g.make_perdir_blocks(mm)
    args = (b["Kb"], b["Cb"], b["b0"], b["b1"], b["Hb"], b["N0"], b["S"], b["Gx"], b["nu"], b["alpha"], b["alpha_lb"])
    for name, ev in (("literal", pb.Evaluator.per_direction(*args)), ("embedding", pb.Evaluator(pdir.embed(*args)))):
        out = ev.alloc_outputs(F)
        for _ in range(3):
            ev.eval(w, out=out)
        torch.cuda.synchronize()
        pb.profile_enable(True); pb.profile_read(reset=True)
        for _ in range(5):
            ev.eval(w, out=out)
        torch.cuda.synchronize()
        p = pb.profile_read(reset=True); pb.profile_enable(False)
        print(mm, f"{name:9s}", {k: round(v[0] / 5, 4) for k, v in p.items()}, flush=True)
        ev.close()
