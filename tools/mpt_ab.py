"""Dev: contraction kernel A/B -- default operator-stationary DFMA kernel vs PODP_FLAG_MPT_GEMM (DMMA + bulk copy)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import podp_inputs as g
from paper_2307_05590_b200 import FLAG_MPT_GEMM, Evaluator, profile_enable, profile_read
F = int(float(os.environ.get("LU_AB_F", "1e5")))
w = torch.tensor(g.omega_grid(F), device="cuda")
for r in [int(x) for x in sys.argv[1:]] or [24, 48, 96]:
    ev = Evaluator(g.make_operators(r))
    out = ev.alloc_outputs(F)
    flop = 80 * r * r + 190 * r
    for name, fl in (("tile(DFMA)", 0), ("gemm(DMMA)", FLAG_MPT_GEMM)):
        ev.eval(w, out=out, flags=fl)
        torch.cuda.synchronize()
        profile_enable(True); profile_read(reset=True)
        for _ in range(5):
            ev.eval(w, out=out, flags=fl)
        torch.cuda.synchronize()
        p = profile_read(reset=True); profile_enable(False)
        ms = p["mpt"][0] / p["mpt"][1]
        print(f"r={r} {name:11s} mpt {ms:8.4f} ms  ({flop * F / ms / 1e9:6.2f} TF/s of the 80 r^2 + 190 r F_alg share)", flush=True)
    ev.close()
