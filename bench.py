#!/usr/bin/env python
"""Benchmark of the PODP on-line hot path on B200 -- prints ONE JSON line.

Workload (BASELINE.json metric / configs[2]): r = 48 POD modes, F = 1e5 log-spaced output frequencies per GPU on
[1e1, 1e8] rad/s, seeded synthetic operators (podp_inputs.make_operators, seed 0).  One "step" = one pass of the
whole hot path over the F frequencies: podp_eval (shifted LU solve, MPT R/I, certificate Delta) + podp_select
(one Algorithm-1 argmax step over the 13 log-spaced snapshot intervals).  podp_create (row a1, packing) is
omega-independent and timed once, outside the steps.

Multi-GPU (torchrun, one rank per GPU): frequencies shard with no data-path collective (weak scaling: each rank
evaluates its own contiguous block of an N*F-point log grid); timing is the max over ranks.

--impl reference runs the CPU oracle (oracle/, the slow plain NumPy implementation) on the box's host cores on
a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "MPT frequencies/sec (3x3 R,I + error bound, FP64) at r=48; % FP64 peak"
UNIT = "freq/s"
R_HEAD = 48
F_HEAD = 100_000
# Measured FP64 peaks on this pool's B200 (tools/fp64_peak.cu, profiles/r01_fp64_peak.jsonl): DMMA (mma.sync f64)
# 36.95 TF/s sustained, DFMA 34.0 TF/s; both paths share the FP64 units (mixed run: 36.8 TF/s total).
FP64_PEAK_TFLOPS = 36.95


def falg(r: int) -> float:
    """Algorithmic FP64 flops per frequency: (8/3)r^3 + 107 r^2 + 190 r."""
    return (8.0 / 3.0) * r ** 3 + 107.0 * r ** 2 + 190.0 * r


def falg_solve(r: int) -> float:
    """Flops of the solve kernel's share of F_alg: LU (8/3 r^3 - r^2) + 3-RHS solves (24 r^2) + A assembly (4 r^2)."""
    return (8.0 / 3.0) * r ** 3 - r ** 2 + 24.0 * r ** 2 + 4.0 * r ** 2


def falg_mpt(r: int) -> float:
    """Flops of the MPT/certificate kernel's share: K_R P, M P, Q formation, Q P (80 r^2) + epilogues (~190 r)."""
    return falg(r) - falg_solve(r)


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 100 ms during the timed region (B200_PROFILING.md)."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.sw_power_cap,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except (OSError, FileNotFoundError):
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self) -> dict:
        sm, mx, reasons = [], None, set()
        names = ["sw_power_cap", "hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        sm.sort()
        med = sm[len(sm) // 2] if sm else None
        return {"sm_mhz": med, "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


def oracle_sample(ops, omega, workers: int):
    """Time the CPU oracle (as it stands) over `omega` on `workers` processes; returns (seconds, n)."""
    return oracle_tasks([(ops, omega)], workers)


def oracle_tasks(tasks, workers: int):
    """Time the CPU oracle over a list of (ops, omegas) tasks, frequencies dealt round-robin to `workers` spawned
    processes with single-threaded BLAS; returns (seconds, n_frequencies)."""
    import multiprocessing as mp
    env_keys = ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS")
    saved = {k: os.environ.get(k) for k in env_keys}
    for k in env_keys:
        os.environ[k] = "1"
    try:
        chunks = [[(o, om[i::workers]) for (o, om) in tasks] for i in range(workers)]
        ctx = mp.get_context("spawn")
        with ctx.Pool(workers) as pool:
            pool.map(_oracle_chunk, [[(tasks[0][0], tasks[0][1][:2])]] * workers)  # warm the workers (imports)
            t0 = time.perf_counter()
            pool.map(_oracle_chunk, chunks)
            dt = time.perf_counter() - t0
    finally:
        for k, v in saved.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    return dt, sum(len(om) for (_o, om) in tasks)


def _oracle_chunk(tasks):
    import oracle
    n = 0
    for ops, om in tasks:
        if len(om):
            oracle.evaluate(ops, om, out_R=False)
        n += len(om)
    return n


def host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1


def measure_config(k: int, steps: int, warmup: int, dev, flush, cpu_seconds: float, cpu: bool) -> dict:
    """Secondary BASELINE configs: one step = podp_eval over the config's frequencies (all
    objects for c3) + podp_select for single-object configs (c4: one Algorithm-1 iteration over 13 log-spaced
    snapshots, N* = 2).  Device-timed with CUDA events, L2 flushed between steps; kernel split from the library's
    event instrumentation; cpu_baseline = the oracle on a bounded evenly spaced sample of the same workload."""
    import numpy as np
    import torch
    import podp_inputs as g
    import paper_2307_05590_b200 as pb
    c = g.make_config(k)
    spec = c["spec"]
    r, F, n_obj = spec["r"], spec["F"], len(c["ops"])
    ev = pb.Evaluator(c["ops"], device=dev.index)
    w = torch.tensor(c["omega"], device=dev)
    out = ev.alloc_outputs(F)
    snap = c.get("snap", g.snapshot_grid(13))
    stream = torch.cuda.current_stream()

    def step():
        ev.eval(w, out=out)
        n = ev.launches_last_call()
        if n_obj == 1:
            ev.select(w, out["Delta"][0], snap, n_star=2)
            n += ev.launches_last_call()
        return n

    for _ in range(warmup):
        step()
    torch.cuda.synchronize()
    pb.profile_enable(True)
    pb.profile_read(reset=True)
    tot, launches = 0.0, 0
    for _ in range(steps):
        flush.zero_()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        launches += step()
        e1.record(stream)
        e1.synchronize()
        tot += e0.elapsed_time(e1)
    prof = pb.profile_read(reset=True)
    pb.profile_enable(False)
    ev.close()
    n_eval = F * n_obj
    value = n_eval * steps / (tot / 1e3)
    res = {"workload": spec["name"], "r": r, "F": F, "n_obj": n_obj, "evaluations_per_step": n_eval,
           "step": "podp_eval + podp_select" if n_obj == 1 else "podp_eval (batch of objects)",
           "value": value, "unit": UNIT, "ms_per_step": tot / steps, "steps": steps,
           "pct_fp64_peak_falg": 100.0 * falg(r) * value / 1e12 / FP64_PEAK_TFLOPS,
           "kernel_ms_per_step": {kk: v[0] / steps for kk, v in prof.items()},
           "gpu_launches": launches}
    if "solve" in prof:
        res["solve_frac_fp64_peak"] = falg_solve(r) * n_eval / (prof["solve"][0] / steps / 1e3) / 1e12 / FP64_PEAK_TFLOPS
    if cpu:
        cores = host_cores()
        # bounded sample: evenly spaced frequencies (and objects, c3) sized for ~cpu_seconds of oracle work
        rate = {8: 20000.0, 24: 4000.0, 32: 2500.0, 48: 1100.0, 96: 320.0}.get(r, 1000.0) * cores
        n_s = int(max(cores * 4, min(n_eval, rate * cpu_seconds)))
        if n_obj == 1:
            idx = np.linspace(0, F - 1, n_s).astype(int)
            tasks = [(c["ops"][0], c["omega"][idx])]
            what = f"{n_s} of the {F} frequencies, evenly spaced"
        else:
            n_o = min(n_obj, 32)
            objs = np.linspace(0, n_obj - 1, n_o).astype(int)
            per = max(1, n_s // n_o)
            fi = np.linspace(0, F - 1, per).astype(int)
            tasks = [(c["ops"][j], c["omega"][fi]) for j in objs]
            what = f"{per} evenly spaced frequencies x {n_o} evenly spaced objects"
        dt, n, passes = 0.0, 0, 0
        while dt < cpu_seconds and passes < 50:  # whole passes over the sample until >= cpu_seconds of CPU work
            d, k = oracle_tasks(tasks, cores)
            dt, n, passes = dt + d, n + k, passes + 1
        res["cpu_baseline"] = {"value": n / dt, "unit": UNIT, "cores": cores, "kind": "oracle",
                               "sample": f"{passes} pass(es) over {what} ({dt:.1f} s, {cores} worker processes x "
                                         f"1 BLAS thread)"}
    return res


def run_reference(args, rank: int, world: int):
    """--impl reference: the oracle on host cores (rank 0 only), bounded sample per step."""
    if rank != 0:
        return
    import numpy as np
    import podp_inputs as g
    ops = g.make_operators(R_HEAD, seed=0)
    omega_full = g.omega_grid(F_HEAD)
    cores = host_cores()
    n_per_step = int(os.environ.get("PODP_REF_SAMPLE", str(512 * cores)))
    idx = np.linspace(0, F_HEAD - 1, n_per_step).astype(int)
    sample = omega_full[idx]
    for _ in range(args.warmup):
        oracle_sample(ops, sample[: max(cores, 64)], cores)
    tot, n = 0.0, 0
    for _ in range(args.steps):
        dt, k = oracle_sample(ops, sample, cores)
        tot += dt
        n += k
    value = n / tot
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "c2_r48_F1e5 (BASELINE configs[2]); oracle on a bounded evenly-spaced sample",
                   "r": R_HEAD, "F_per_gpu": F_HEAD, "sample_per_step": n_per_step},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle",
                         "sample": f"{n_per_step} of the {F_HEAD} c2 frequencies (evenly spaced) per step"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="podp", choices=["podp", "reference"])
    ap.add_argument("--F", type=int, default=F_HEAD)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-adapt", action="store_true", help="skip the Algorithm-1 (N2) variant")
    ap.add_argument("--no-configs", action="store_true", help="skip the secondary BASELINE configs c0, c1, c3, c4")
    ap.add_argument("--configs", default="0,1,3,4", help="secondary BASELINE configs measured into 'configs'")
    args = ap.parse_args()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if args.warmup < 3:
        args.warmup = 3  # timing rule: >= 3 warm-up steps

    import numpy as np
    import torch
    import __graft_entry__
    __graft_entry__.build()
    import podp_inputs as g
    import paper_2307_05590_b200 as pb

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)

    F = args.F
    ops = g.make_operators(R_HEAD, seed=0)
    # weak scaling: rank r owns block r of an (world*F)-point log grid on [1e1, 1e8]
    omega_all = g.omega_grid(F * world)
    omega_h = np.ascontiguousarray(omega_all[rank * F:(rank + 1) * F])
    snap = g.snapshot_grid(13)
    stream = torch.cuda.current_stream()

    t0 = time.perf_counter()
    ev = pb.Evaluator(ops, device=local)
    torch.cuda.synchronize()
    create_ms = (time.perf_counter() - t0) * 1e3

    w_d = torch.tensor(omega_h, device=dev)
    out = ev.alloc_outputs(F, info=True)
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)  # > 126 MB L2

    def step():
        ev.eval(w_d, out=out)
        n = ev.launches_last_call()
        ev.select(w_d, out["Delta"][0], snap, n_star=2)
        return n + ev.launches_last_call()

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    pb.profile_enable(True)
    pb.profile_read(reset=True)
    launches = 0
    step_ms = []
    with ClockSampler(local) as clk:
        time.sleep(0.6)  # let nvidia-smi start sampling before the timed region
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()
        for _ in range(args.steps):
            flush.zero_()  # L2 flush between timed steps (untimed)
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            launches += step()  # select synchronises the stream at its end
            e1.record(stream)
            e1.synchronize()
            step_ms.append(e0.elapsed_time(e1))
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
    prof = pb.profile_read(reset=True)
    pb.profile_enable(False)
    # NEXT row N3 (pencil solver) measured the same way, reported as a separate variant (not the headline)
    variants = {}
    try:
        pb.profile_enable(True)
        pb.profile_read(reset=True)
        for _ in range(args.warmup):
            ev.eval(w_d, out=out, flags=pb.FLAG_PENCIL)
        torch.cuda.synchronize()
        pb.profile_read(reset=True)
        pen_ms = 0.0
        for _ in range(args.steps):
            flush.zero_()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            ev.eval(w_d, out=out, flags=pb.FLAG_PENCIL)
            e1.record(stream)
            e1.synchronize()
            pen_ms += e0.elapsed_time(e1)
        pprof = pb.profile_read(reset=True)
        pb.profile_enable(False)
        r = R_HEAD
        # executed per frequency on the y path: y = D (c0 + omega c1) (~30 r), Q~ = G~kk + s J~ + s^2 G~mm (8 r^2),
        # Q~ y for 3 columns (24 r^2), diagonal K_R / M_I forms + linear terms + epilogue (~190 r)
        exec_flops = 32.0 * r * r + 220.0 * r
        pen_val = F * args.steps / (pen_ms / 1e3)
        variants["pencil_N3"] = {
            "value": pen_val, "unit": UNIT, "ms_per_eval": pen_ms / args.steps,
            "executed_flop_per_freq": exec_flops,
            "executed_tflops": exec_flops * pen_val / 1e12,
            "frac_of_fp64_peak_executed": exec_flops * pen_val / 1e12 / FP64_PEAK_TFLOPS,
            "kernel_ms_per_eval": {k: v[0] / max(v[1], 1) for k, v in pprof.items()},
            "note": "exact reformulation (K = L L^H, L^-1 M L^-H = V Lambda V^H, y = (I + i s Lambda)^-1 Z^H B, MPT and "
                    "certificate in pencil coordinates); NEXT row N3, not the LU headline"}
    except Exception as exc:  # pragma: no cover
        variants["pencil_N3"] = {"error": str(exc)[:200]}
    # NEXT row N1: the literal per-direction form (three LU solves of size M_i per omega + cross-block contractions)
    # against the block-diagonal embedding of size sum M_i, on the same synthetic blocks and the step's omegas
    try:
        from paper_2307_05590_b200 import perdir as pdir
        res_n1 = {}
        for mm in ((16, 16, 16), (24, 16, 8)):
            blk = g.make_perdir_blocks(mm)
            ev_lit = pb.Evaluator.per_direction(blk["Kb"], blk["Cb"], blk["b0"], blk["b1"], blk["Hb"], blk["N0"],
                                                blk["S"], blk["Gx"], blk["nu"], blk["alpha"], blk["alpha_lb"],
                                                device=local)
            ev_emb = pb.Evaluator(pdir.embed(blk["Kb"], blk["Cb"], blk["b0"], blk["b1"], blk["Hb"], blk["N0"],
                                             blk["S"], blk["Gx"], blk["nu"], blk["alpha"], blk["alpha_lb"]),
                                  device=local)
            row = {}
            for name, evx in (("literal", ev_lit), ("embedding", ev_emb)):
                for _ in range(args.warmup):
                    evx.eval(w_d, out=out)
                torch.cuda.synchronize()
                ms = 0.0
                for _ in range(args.steps):
                    flush.zero_()
                    e0 = torch.cuda.Event(enable_timing=True)
                    e1 = torch.cuda.Event(enable_timing=True)
                    e0.record(stream)
                    evx.eval(w_d, out=out)
                    e1.record(stream)
                    e1.synchronize()
                    ms += e0.elapsed_time(e1)
                row[name] = {"value": F * args.steps / (ms / 1e3), "unit": UNIT, "ms_per_eval": ms / args.steps}
                evx.close()
            row["speedup_literal"] = row["embedding"]["ms_per_eval"] / row["literal"]["ms_per_eval"]
            res_n1["M=" + "+".join(str(x) for x in mm)] = row
        variants["perdir_N1"] = dict(res_n1, note="podp_eval only (no select); literal = podp_create_perdir "
                                                  "(3 batched LU solves of size M_i + placement + contraction), "
                                                  "embedding = one LU of size sum M_i (block-diagonal K, M)")
    except Exception as exc:  # pragma: no cover
        variants["perdir_N1"] = {"error": str(exc)[:200]}
    # NEXT row N2: one Algorithm-1 run (off-line cuSOLVER/cuBLAS + on-line libpodp certification on a 1e5 grid)
    if rank == 0 and not args.no_adapt:
        try:
            import math
            from paper_2307_05590_b200 import adapt
            fom = g.make_fullorder()
            vol = fom.alpha ** 3 * 4.0 * math.pi / 3.0
            om_ad = g.omega_grid(F, 1e1, 1e7)
            adapt.run_adaptive(fom, om_ad[::100], tol_delta=1e-3, max_k=2, vol=vol)   # warm-up (cuSOLVER init)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            _o, _x, hist = adapt.run_adaptive(fom, om_ad, tol_delta=1e-3, max_k=4, vol=vol)
            torch.cuda.synchronize()
            variants["adaptive_N2"] = {
                "full_order_N": fom.N, "output_grid": F, "window": [1e1, 1e7], "iterations": len(hist),
                "N_snapshots": [h["N"] for h in hist], "r": [h["r"] for h in hist],
                "Lambda_over_vol": [h["Lambda"] / vol for h in hist],
                "offline_ms": [round(h["t_offline"] * 1e3, 3) for h in hist],
                "online_ms": [round(h["t_online"] * 1e3, 3) for h in hist],
                "total_s": time.perf_counter() - t0,
                "note": "host clock around synchronised phases; online = podp_create + podp_eval + podp_select"}
        except Exception as exc:  # pragma: no cover
            variants["adaptive_N2"] = {"error": str(exc)[:200]}
    # secondary BASELINE configs (rank 0, N = 1 only: they are single-GPU workloads)
    configs = {}
    if rank == 0 and world == 1 and not args.no_configs:
        for k in [int(x) for x in args.configs.split(",") if x.strip()]:
            try:
                configs[f"c{k}"] = measure_config(k, min(args.steps, 5), 3, dev, flush,
                                                  float(os.environ.get("PODP_CPU_SECONDS_CFG", "3")),
                                                  not args.no_cpu_baseline)
            except Exception as exc:  # pragma: no cover
                configs[f"c{k}"] = {"error": str(exc)[:200]}
    total_ms = float(sum(step_ms))
    if dist is not None:
        t = torch.tensor([total_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    value = (F * world * args.steps) / (total_ms / 1e3)

    # end-to-end through the public host-buffer entry point (podp_eval_host): H2D omega, D2H outputs per step
    T1h = torch.empty((1, F, 6), dtype=torch.float64, pin_memory=True).numpy()
    Ih = torch.empty((1, F, 6), dtype=torch.float64, pin_memory=True).numpy()
    Dh = torch.empty((1, F, 6), dtype=torch.float64, pin_memory=True).numpy()
    infoh = torch.empty((1, F), dtype=torch.int32, pin_memory=True).numpy()
    om_pin = torch.empty(F, dtype=torch.float64, pin_memory=True).numpy()
    om_pin[:] = omega_h
    hout = dict(T1=T1h, I=Ih, Delta=Dh, info=infoh)
    for _ in range(2):
        ev.eval_host(om_pin, out=hout)
    e2e_ms = 0.0
    for _ in range(args.steps):
        flush.zero_()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        ev.eval_host(om_pin, out=hout)
        e1.record(stream)
        e1.synchronize()
        e2e_ms += e0.elapsed_time(e1)
    if dist is not None:
        t = torch.tensor([e2e_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())
    e2e_value = (F * world * args.steps) / (e2e_ms / 1e3)
    h2d = omega_h.nbytes
    d2h = T1h.nbytes + Ih.nbytes + Dh.nbytes + infoh.nbytes

    if rank == 0:
        solve_ms, solve_n = prof.get("solve", (0.0, 1))
        mpt_ms, mpt_n = prof.get("mpt", (0.0, 1))
        sel_ms, sel_n = prof.get("select", (0.0, 1))
        dom = "solve" if solve_ms >= mpt_ms else "mpt"
        dom_ms = (solve_ms / max(solve_n, 1)) if dom == "solve" else (mpt_ms / max(mpt_n, 1))
        dom_flops = F * (falg_solve(R_HEAD) if dom == "solve" else falg_mpt(R_HEAD))
        achieved = dom_flops / (dom_ms / 1e3) / 1e12
        traffic = None
        tpath = os.path.join(ROOT, "profiles", "r02_roofline_traffic.json")
        if os.path.exists(tpath):
            try:
                traffic = json.load(open(tpath)).get(dom, {}).get("dram_bytes_per_launch")
            except (ValueError, OSError):
                traffic = None
        step_flops = F * falg(R_HEAD)
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": "c2_r48_F1e5 (BASELINE configs[2]): podp_eval + podp_select per step",
                       "r": R_HEAD, "F_per_gpu": F, "omega": "logspace(1,8,N*F) block per rank",
                       "l2": "flushed between timed steps (256 MiB write, untimed)",
                       "parallelism": f"dp{world} (independent omega shards, no data-path collective)",
                       "podp_create_ms": round(create_ms, 3)},
            "pct_fp64_peak": 100.0 * step_flops / (total_ms / args.steps / 1e3) / 1e12 / FP64_PEAK_TFLOPS,
            "roofline": {"bound": "alu", "kernel": dom, "achieved": achieved, "peak": FP64_PEAK_TFLOPS,
                         "unit": "TFLOP/s", "frac": achieved / FP64_PEAK_TFLOPS, "traffic": traffic,
                         "peak_source": "measured FP64 (mma.sync f64 / DFMA share one pipe), tools/fp64_peak.cu",
                         "flops_per_launch": dom_flops},
            "kernel_ms_per_step": {k: v[0] / max(v[1], 1) * (v[1] / args.steps) for k, v in prof.items()},
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
            "gpu_launches": launches,
            "variants": variants,
        }
        if configs:
            line["configs"] = configs
        line["clocks"] = clk.summary()
        if not args.no_cpu_baseline:
            cores = host_cores()
            # bounded sample of ~10 s of CPU work: whole passes over the step's F frequencies, repeated until
            # >= PODP_CPU_SECONDS (default 10) have elapsed (max 30 passes)
            target = float(os.environ.get("PODP_CPU_SECONDS", "10"))
            dt, n, passes = 0.0, 0, 0
            while dt < target and passes < 30:
                d, k = oracle_sample(ops, omega_h, cores)
                dt, n, passes = dt + d, n + k, passes + 1
            line["cpu_baseline"] = {"value": n / dt, "unit": UNIT, "cores": cores, "kind": "oracle",
                                    "sample": f"{passes} full pass(es) over the {F} c2 frequencies of one step "
                                              f"({dt:.1f} s, {cores} worker processes x 1 BLAS thread)"}
        print(json.dumps(line), flush=True)
    ev.close()
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
