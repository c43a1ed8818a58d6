"""A/B timing of the LU kernels over r (dev tool): python tools/lu_ab.py [r ...]; variants via PODP_LU_IMPL and PODP_LU_W."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import podp_inputs as g
from paper_2307_05590_b200 import Evaluator, profile_enable, profile_read
import numpy as np


def ops_for(r):
    if r % 2 == 0:
        return g.make_operators(r)
    o = g.make_operators(r + 1)
    keep = np.r_[0:6, 6:6 + r, 6 + r + 1:6 + 2 * r + 1]
    return g.Operators(K=o.K[:r, :r], M=o.M[:r, :r], b0=o.b0[:r], b1=o.b1[:r], N0=o.N0, S=o.S, H=o.H[:, :r],
                       G=o.G[np.ix_(keep, keep)], nu=o.nu, alpha=o.alpha, alpha_lb=o.alpha_lb)

VARIANTS = [("blk", {"PODP_LU_IMPL": "b"}), ("dyn", {"PODP_LU_IMPL": "d"}), ("dyn-w1", {"PODP_LU_IMPL": "d", "PODP_LU_W": "1"}),
            ("dyn-w2", {"PODP_LU_IMPL": "d", "PODP_LU_W": "2"}), ("dyn-w4", {"PODP_LU_IMPL": "d", "PODP_LU_W": "4"}),
            ]


def main():
    rs = [int(x) for x in sys.argv[1:]] or [8, 16, 24, 32, 40, 48, 56, 64, 72, 80, 88, 96]
    F = int(os.environ.get("AB_F", "100000"))
    w = torch.tensor(g.omega_grid(F), device="cuda")
    for r in rs:
        ev = Evaluator(ops_for(r))
        out = ev.alloc_outputs(F)
        line = [f"r={r:3d}"]
        for name, env in VARIANTS:
            for k in ("PODP_LU_IMPL", "PODP_LU_W"):
                os.environ.pop(k, None)
            os.environ.update(env)
            try:
                ev.eval(w, out=out)
                torch.cuda.synchronize()
                profile_enable(True)
                profile_read(reset=True)
                for _ in range(3):
                    ev.eval(w, out=out)
                torch.cuda.synchronize()
                prof = profile_read(reset=True)
                profile_enable(False)
                line.append(f"{name} {prof['solve'][0] / 3:.3f}")
            except Exception as e:  # noqa: BLE001 (dev tool: report and continue)
                line.append(f"{name} ERR({str(e)[:30]})")
        print("  ".join(line), flush=True)
        ev.close()


main()
