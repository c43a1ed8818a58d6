"""Time podp_eval (default LU path and pencil) over a range of r at F = 1e5 (dev tool)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import podp_inputs as g
from paper_2307_05590_b200 import FLAG_PENCIL, Evaluator, profile_enable, profile_read


def ops_for(r):
    if r % 2 == 0:
        return g.make_operators(r)
    o = g.make_operators(r + 1)
    R = r + 1
    keep = np.r_[0:6, 6:6 + r, 6 + R:6 + R + r]
    return g.Operators(K=o.K[:r, :r], M=o.M[:r, :r], b0=o.b0[:r], b1=o.b1[:r], N0=o.N0, S=o.S, H=o.H[:, :r],
                       G=o.G[np.ix_(keep, keep)], nu=o.nu, alpha=o.alpha, alpha_lb=o.alpha_lb)


def main():
    rs = [int(x) for x in sys.argv[1:]] or [24, 32, 39, 40, 45, 48, 51, 56, 57, 64, 96]
    F = int(os.environ.get("RS_F", "100000"))
    w = torch.tensor(g.omega_grid(F), device="cuda")
    for r in rs:
        ev = Evaluator(ops_for(r))
        out = ev.alloc_outputs(F)
        res = []
        split = []
        for flags in (0, FLAG_PENCIL):
            for _ in range(2):
                ev.eval(w, out=out, flags=flags)
            torch.cuda.synchronize()
            profile_enable(True)
            profile_read(reset=True)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(3):
                ev.eval(w, out=out, flags=flags)
            e1.record()
            torch.cuda.synchronize()
            res.append(e0.elapsed_time(e1) / 3)
            pr = profile_read(reset=True)
            profile_enable(False)
            split.append("/".join(f"{k}={v[0] / max(v[1], 1):.3f}" for k, v in pr.items()))
        print(f"r={r:3d} lu_ms={res[0]:8.3f} pencil_ms={res[1]:8.3f}   [{split[0]}] [{split[1]}]", flush=True)
        ev.close()


main()
