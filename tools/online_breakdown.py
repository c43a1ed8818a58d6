"""Dev: host-clock breakdown of one on-line certification (podp_create + podp_eval + podp_select + destroy) at r, F,
as the Algorithm-1 driver does per iteration (fresh context each time)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import podp_inputs as g
import paper_2307_05590_b200 as pb
r = int(sys.argv[1]) if len(sys.argv) > 1 else 48
F = int(float(sys.argv[2])) if len(sys.argv) > 2 else 100000
ops = g.make_operators(r)
w = torch.tensor(g.omega_grid(F), device="cuda")
snap = g.snapshot_grid(13)
for it in range(4):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ev = pb.Evaluator(ops)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    out = ev.eval(w)
    torch.cuda.synchronize(); t2 = time.perf_counter()
    ev.select(w, out["Delta"][0], snap, n_star=2)
    t3 = time.perf_counter()
    ev.close()
    torch.cuda.synchronize(); t4 = time.perf_counter()
    print(f"iter {it}: create {1e3*(t1-t0):7.2f} ms  eval {1e3*(t2-t1):7.2f}  select {1e3*(t3-t2):6.2f}  destroy {1e3*(t4-t3):6.2f}", flush=True)
