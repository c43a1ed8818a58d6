"""A/B timing of the LU kernels over r (dev tool): python tools/lu_ab.py [r ...]  (env LU_AB_F, default 1e5).

Times the "solve" and "mpt" phases of podp_eval (CUDA events via the podp_profile API) for every LU kernel the
library instantiates at that r (PODP_FLAG_LU_*), on the BASELINE generators (make_operators(r)).
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import podp_inputs as g
from paper_2307_05590_b200 import (FLAG_LU_BLK, FLAG_LU_DYN, FLAG_LU_GENERIC, FLAG_LU_LL, Evaluator,
                                   profile_enable, profile_read)


def falg_solve(r):
    return (8.0 / 3.0) * r ** 3 + 27 * r ** 2


def main():
    rs = [int(x) for x in sys.argv[1:]] or [24, 32, 48, 64, 96]
    F = int(float(os.environ.get("LU_AB_F", "1e5")))
    w = torch.tensor(g.omega_grid(F), device="cuda")
    for r in rs:
        ev = Evaluator(g.make_operators(r))
        out = ev.alloc_outputs(F)
        R = (r + 7) // 8 * 8
        variants = [("ll", FLAG_LU_LL)] if R <= 96 else []
        if R <= 96:
            variants += [("blk", FLAG_LU_BLK), ("dyn", FLAG_LU_DYN)]
        if os.environ.get("LU_AB_GENERIC"):
            variants.append(("generic", FLAG_LU_GENERIC))
        for name, flags in variants:
            ev.eval(w, out=out, flags=flags)
            torch.cuda.synchronize()
            profile_enable(True)
            profile_read(reset=True)
            n = 5
            for _ in range(n):
                ev.eval(w, out=out, flags=flags)
            torch.cuda.synchronize()
            prof = profile_read(reset=True)
            profile_enable(False)
            ms = prof["solve"][0] / n
            tf = falg_solve(r) * F / ms / 1e9
            print(f"r={r} {name:8s} solve {ms:8.4f} ms  ({tf:6.2f} TF/s F_alg, {tf / 36.95:6.1%} of FP64)  "
                  f"mpt {prof['mpt'][0] / n:7.4f} ms", flush=True)
        ev.close()


main()
