"""Quick CUDA-event timing of podp_eval on a BASELINE config (dev tool; bench.py is the contract)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import podp_inputs as g
from paper_2307_05590_b200 import Evaluator, FLAG_OUT_R

def main():
    cfgs = [int(x) for x in (sys.argv[1:] or ["2"])]
    for cfg in cfgs:
        c = g.make_config(cfg)
        ev = Evaluator(c["ops"])
        w = torch.tensor(c["omega"], device="cuda")
        out = ev.alloc_outputs(len(c["omega"]))
        flags = int(os.environ.get("QT_FLAGS", "0"))
        for _ in range(3):
            ev.eval(w, out=out, flags=flags)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        n = 5
        e0.record()
        for _ in range(n):
            ev.eval(w, out=out, flags=flags)
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / n
        nf = len(c["omega"]) * len(c["ops"])
        r = c["spec"]["r"]
        falg = (8 / 3) * r ** 3 + 107 * r ** 2 + 190 * r
        print(f"cfg{cfg} r={r} evals={nf} ms={ms:.3f} freq/s={nf/ms*1e3:.4g} TFLOP/s(F_alg)={falg*nf/ms/1e9:.3f}", flush=True)
        ev.close()

main()
