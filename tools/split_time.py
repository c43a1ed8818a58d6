"""Per-kernel split (solve / mpt) of podp_eval over r at F = 1e5 (dev tool): python tools/split_time.py [r ...]."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import podp_inputs as g
from paper_2307_05590_b200 import FLAG_PENCIL, Evaluator, profile_enable, profile_read


def main():
    rs = [int(x) for x in sys.argv[1:]] or [24, 32, 48, 96]
    F = int(os.environ.get("ST_F", "100000"))
    w = torch.tensor(g.omega_grid(F), device="cuda")
    for r in rs:
        ev = Evaluator(g.make_operators(r))
        out = ev.alloc_outputs(F)
        for name, flags in (("lu", 0), ("pencil", FLAG_PENCIL)):
            ev.eval(w, out=out, flags=flags)
            torch.cuda.synchronize()
            profile_enable(True)
            profile_read(reset=True)
            for _ in range(5):
                ev.eval(w, out=out, flags=flags)
            torch.cuda.synchronize()
            prof = profile_read(reset=True)
            profile_enable(False)
            print(f"r={r} {name}: " + "  ".join(f"{k} {v[0] / 5:.4f} ms" for k, v in prof.items()), flush=True)
        ev.close()


main()
