"""Parity report per BASELINE config (SURVEY 8(c) "Parity metric"): runs on the GPU box.

For each config the GPU evaluates the full workload in the bench launch configuration; a deterministic, evenly
spaced sample of outputs (all of c0 and c1) is compared with the CPU oracle:
  * gate metric (normalised by the north_star tolerances, must be <= 1): e_R, e_I (1e-10 x term magnitude),
    e_Delta (1e-8 x max(Delta, 1e-6 mag^Delta));
  * "also report, not gate": plain per-entry relative error with a 1e-3 max|T(omega)| floor, the normwise
    max|dT| / max|T| per omega, and the count of entries above 1e-10 by the plain metric, each adjudicated at that
    omega by the 80-bit re-evaluation (oracle/extended.py): the GPU passes there if its error against the 80-bit
    value is <= 2x the FP64 oracle's.
Writes one JSON object per config to stdout.
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import oracle
from oracle.extended import evaluate_one_ld
from oracle.parity import TOL_DELTA, TOL_RI, errors
import podp_inputs as g
from paper_2307_05590_b200 import FLAG_OUT_R, Evaluator

SAMPLE = {0: None, 1: None, 2: 1500, 3: (32, 40), 4: 300}


def plain(gpu, ora):
    floor = 1e-3 * np.max(np.abs(ora))
    return np.abs(gpu - ora) / np.maximum(np.abs(ora), max(floor, 1e-300))


def main():
    cfgs = [int(x) for x in (sys.argv[1:] or ["0", "1", "2", "3", "4"])]
    for k in cfgs:
        t0 = time.time()
        c = g.make_config(k)
        ops_list, omega = c["ops"], c["omega"]
        F = len(omega)
        ev = Evaluator(ops_list)
        out = ev.eval(torch.tensor(omega, device="cuda"), flags=FLAG_OUT_R)
        torch.cuda.synchronize()
        T1, I, D = (out[x].cpu().numpy() for x in ("T1", "I", "Delta"))
        ev.close()
        s = SAMPLE[k]
        if k == 3:
            objs = np.linspace(0, len(ops_list) - 1, s[0]).astype(int)
            fs = np.linspace(0, F - 1, s[1]).astype(int)
            pairs = [(o, f) for o in objs for f in fs]
        else:
            fs = range(F) if s is None else np.linspace(0, F - 1, s).astype(int)
            pairs = [(0, f) for f in fs]
        gate = np.zeros(3)
        pl = np.zeros(3)
        normw = np.zeros(3)
        above, adjudicated_ok = 0, 0
        details = []
        for o, f in pairs:
            ops = ops_list[o]
            w = float(omega[f])
            ora = oracle.evaluate_one(ops, w, out_R=True)
            o6 = [oracle.to6(ora[x]) for x in ("R", "I", "Delta")]
            g6 = [T1[o, f], I[o, f], D[o, f]]
            e = errors(ops, w, *g6, *o6)
            gate = np.maximum(gate, [e[0].max() / TOL_RI, e[1].max() / TOL_RI, e[2].max() / TOL_DELTA])
            for q in range(3):
                pq = plain(g6[q], o6[q])
                pl[q] = max(pl[q], pq.max())
                normw[q] = max(normw[q], np.max(np.abs(g6[q] - o6[q])) / max(np.max(np.abs(o6[q])), 1e-300))
                bad = np.nonzero(pq > 1e-10)[0]
                if len(bad):
                    t = evaluate_one_ld(ops, w)
                    t6 = [t["R6"], t["I6"], t["D6"]][q]
                    for b in bad:
                        above += 1
                        floor = 1e-3 * np.max(np.abs(t6))
                        eg = abs(g6[q][b] - t6[b])
                        eo = abs(o6[q][b] - t6[b])
                        ok = eg <= 2.0 * eo or eg <= 1e-10 * max(abs(t6[b]), floor)
                        adjudicated_ok += int(ok)
                        from oracle.parity import magnitudes
                        mg = magnitudes(ops, w)[q][b]
                        if len(details) < 8:
                            details.append({"obj": int(o), "omega": w, "quantity": "RID"[q], "entry": int(b),
                                            "value_80bit": float(t6[b]), "gpu_err": float(eg),
                                            "fp64_oracle_err": float(eo), "term_magnitude": float(mg),
                                            "gpu_err_over_magnitude": float(eg / mg) if mg > 0 else None,
                                            "within_2x_oracle": bool(ok)})
        rec = {"config": c["spec"]["name"], "r": c["spec"]["r"], "evaluations": F * len(ops_list),
               "sampled": len(pairs), "gate_max_normalised": dict(zip(("R", "I", "Delta"), gate.tolist())),
               "gate_pass": bool(np.all(gate <= 1.0)),
               "plain_rel_1e-3_floor_max": dict(zip(("R", "I", "Delta"), pl.tolist())),
               "normwise_max": dict(zip(("R", "I", "Delta"), normw.tolist())),
               "plain_above_1e-10": above, "adjudicated_80bit_ok": adjudicated_ok, "above_details": details,
               "seconds": round(time.time() - t0, 1)}
        print(json.dumps(rec), flush=True)


if __name__ == "__main__":
    main()
