"""Multi-process (gloo, world_size 2, CPU) test of the sharded-selection plumbing: ranks reduce their omega
shard to per-interval maxima, all-gather, merge -- must equal the single-process selection."""
import os

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2307_05590_b200 import dist as pd
import oracle


def _local_maxima(omega, D, snap, lo, hi):
    """Reference per-interval reduction of a shard (oracle select rules) -> (lam, global arg)."""
    n_int = len(snap) - 1
    lam, arg = [None] * n_int, [None] * n_int
    sset = set(float(x) for x in snap)
    for f in range(lo, hi):
        w = float(omega[f])
        if w in sset or w < snap[0] or w > snap[-1]:
            continue
        n = max(k for k in range(n_int) if snap[k] <= w)
        v = max((d for d in D[f] if d == d), default=None)
        if v is None:
            continue
        if lam[n] is None or v > lam[n]:
            lam[n], arg[n] = v, f
    return lam, arg


def _worker(rank, world, port, omega, D, snap, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    lo, hi = pd.shard_range(len(omega), world, rank)
    res = _local_maxima(omega, D, snap, lo, hi)
    idx, Lam = pd.select_distributed(res, n_star=2)
    idx_t, Lam_t = pd.select_distributed(res, n_star=12, theta=0.5)
    out[rank] = (idx, Lam, idx_t, Lam_t)
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_sharded_selection_matches_single_process(world):
    rng = np.random.default_rng(7)
    omega = np.logspace(1, 8, 3001)
    D = rng.random((3001, 6)) ** 4
    D[1234, 2] = 5.0
    D[1235, 1] = 5.0        # tie inside an interval -> lowest index
    D[2000:2003, 0] = np.nan
    snap = np.logspace(1, 8, 13)
    mgr = mp.get_context("spawn").Manager()
    out = mgr.dict()
    port = 29500 + (os.getpid() % 1000)
    mp.start_processes(_worker, args=(world, port, omega, D, snap, out), nprocs=world, start_method="spawn")
    ow, oidx, oLam, _ = oracle.select(omega, D, snap, 2)
    _, oidx_t, _, _ = oracle.select(omega, D, snap, 12, theta=0.5)
    for r in range(world):
        idx, Lam, idx_t, Lam_t = out[r]
        assert idx == oidx and Lam == oLam
        assert idx_t == oidx_t


def test_shard_range_covers():
    for n in (0, 1, 7, 100, 101):
        for w in (1, 2, 3, 8):
            parts = [pd.shard_range(n, w, r) for r in range(w)]
            assert parts[0][0] == 0 and parts[-1][1] == n
            assert all(parts[i][1] == parts[i + 1][0] for i in range(w - 1))


@pytest.mark.gpu
def test_local_interval_maxima_zero_interval(torch_cuda):
    """an interval whose Lambda_n is exactly 0 must come back with a consistent (lam, arg) pair."""
    torch = torch_cuda
    import numpy as np
    import podp_inputs as g
    from paper_2307_05590_b200 import Evaluator
    from paper_2307_05590_b200.dist import local_interval_maxima_gpu
    ev = Evaluator(g.make_operators(8))
    om = g.omega_grid(100)
    snap = g.snapshot_grid(5)
    D = np.random.default_rng(0).uniform(0.5, 1.0, (100, 6))
    D[(om >= snap[1]) & (om < snap[2])] = 0.0          # interval 1: all zero
    lam, arg = local_interval_maxima_gpu(ev, torch.tensor(om, device="cuda"), torch.tensor(D, device="cuda"),
                                         snap, global_offset=1000)
    assert lam[1] == 0.0 and arg[1] is not None
    i = arg[1] - 1000
    assert snap[1] <= om[i] < snap[2] and om[i] not in set(snap)
    assert i == min(j for j in range(100) if snap[1] <= om[j] < snap[2] and om[j] not in set(snap))
    for n in range(4):
        assert (lam[n] is None) == (arg[n] is None)
    ev.close()
