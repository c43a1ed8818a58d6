"""Small driver for compute-sanitizer (racecheck / synccheck / memcheck): every LU kernel the library instantiates
(left-looking, lock-step, dynamically scheduled with and without the L2 right-hand-side mode, generic), the
pencil path, the MPT/certificate kernel, select and the N4 epilogues, on small F with ragged tails, on the BASELINE
generators and on the pivot-forcing input (dev tool; results in profiles/r02_sanitizer.txt)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import podp_inputs as g
import paper_2307_05590_b200 as pb
from paper_2307_05590_b200 import (FLAG_LU_BLK, FLAG_LU_DYN, FLAG_LU_GENERIC, FLAG_LU_LL, FLAG_OUT_R, FLAG_PENCIL,
                                   Evaluator)

F = int(os.environ.get("SAN_F", "37"))
w = torch.tensor(g.omega_grid(F), device="cuda")
cases = [("c0", g.make_config0()[0])] + [(f"r{r}", g.make_operators(r)) for r in (48, 56, 96)] + \
        [("pivot48", g.make_pivot_forcing(48, seed=1))]
for name, ops in cases:
    R = (ops.r + 7) // 8 * 8
    flags = [("default", 0), ("blk", FLAG_LU_BLK), ("dyn", FLAG_LU_DYN), ("generic", FLAG_LU_GENERIC)]
    if R <= 64:
        flags.append(("ll", FLAG_LU_LL))
    if not name.startswith("pivot"):
        flags.append(("pencil", FLAG_PENCIL))
    ev = Evaluator(ops)
    for fn, fl in flags:
        out = ev.eval(w, flags=FLAG_OUT_R | fl)
        torch.cuda.synchronize()
        print(name, fn, "info0" if bool((out["info"] == 0).all()) else "info!=0", flush=True)
    out = ev.eval(w)
    ev.select(w, out["Delta"][0], g.snapshot_grid(5), n_star=2)
    pb.invariants(out["T1"], out["I"])
    torch.cuda.synchronize()
    ev.close()
print("sanitize_run ok")
