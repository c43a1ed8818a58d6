"""Multi-GPU plumbing for the PODP on-line path (one process per GPU, torch.distributed).

Frequencies are independent ("computed once for all frequencies of interest"), so evaluation shards the
omega grid with no collective.  The only cross-rank exchange is Algorithm 1's selection: each rank
reduces its shard to per-interval (Lambda_n, argmax) pairs on its GPU (podp_select), the pairs are all-gathered
(a few hundred bytes) and merged on the host with the same tie rules as the single-GPU path (readings U12/U13).
"""
from __future__ import annotations

import math


def shard_range(n_total: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous block [start, end) of rank `rank` (block sizes differ by at most one)."""
    base, extra = divmod(n_total, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def merge_interval_maxima(per_rank):
    """per_rank: list over ranks (in rank order, shards ascending) of (lam_n, arg_n) where lam_n[n] is the local
    interval maximum (None / < 0 if empty) and arg_n[n] the GLOBAL grid index of its argmax.
    Returns (lam, arg): global maxima; ties resolve to the lowest global index."""
    n_int = len(per_rank[0][0])
    lam = [None] * n_int
    arg = [None] * n_int
    for lam_r, arg_r in per_rank:
        for n in range(n_int):
            v = lam_r[n]
            if v is None or v < 0:
                continue
            if lam[n] is None or v > lam[n] or (v == lam[n] and arg_r[n] < arg[n]):
                lam[n], arg[n] = v, arg_r[n]
    return lam, arg


def choose(lam, arg, n_star: int, theta: float = 0.0):
    """Top-N* intervals by (-Lambda_n, n), or Lambda_n >= theta*Lambda.  Returns
    (sorted chosen grid indices, Lambda)."""
    cands = [n for n in range(len(lam)) if lam[n] is not None]
    if not cands:
        raise ValueError("no candidates")
    Lam = max(lam[n] for n in cands)
    if theta > 0.0:
        cands = [n for n in cands if lam[n] >= theta * Lam]
    elif len(cands) < n_star:
        raise ValueError("fewer non-empty intervals than n_star")
    order = sorted(cands, key=lambda n: (-lam[n], n))[:n_star]
    return sorted(arg[n] for n in order), Lam


def local_interval_maxima_gpu(ev, omega_d, delta_d, snap, global_offset: int):
    """Per-interval (Lambda_n, global argmax) of this rank's shard, reduced on the GPU by podp_select."""
    n_int = len(snap) - 1
    if n_int > 64:
        raise ValueError("distributed selection supports <= 64 intervals")
    try:
        _, idx, _, lam_n = ev.select(omega_d, delta_d, snap, n_star=n_int, theta=1e-300)
    except Exception:  # no candidate on this shard
        return [None] * n_int, [None] * n_int
    om = omega_d.cpu().numpy()
    lam = [float(x) if x >= 0 else None for x in lam_n]
    arg = [None] * n_int
    s = list(snap)
    for i in idx:
        w = om[i]
        n = max(k for k in range(n_int) if s[k] <= w)
        arg[n] = int(i) + global_offset
    # an interval whose Lambda_n is exactly 0 is not returned by the theta = 1e-300 call above (0 < theta * Lambda);
    # its argmax is its lowest candidate grid index (all entries 0; NaN ignored), found here so lam and arg agree
    missing = [n for n in range(n_int) if lam[n] is not None and arg[n] is None]
    if missing:
        import numpy as np
        dmax = np.nanmax(delta_d.cpu().numpy(), axis=1)
        snapset = set(s)
        for n in missing:
            last = n == n_int - 1
            for i, w in enumerate(om):
                inside = s[n] <= w and (w < s[n + 1] or (last and w <= s[n + 1]))
                if inside and w not in snapset and dmax[i] == lam[n]:
                    arg[n] = int(i) + global_offset
                    break
            if arg[n] is None:  # pragma: no cover - cannot happen when lam[n] is a maximum over the interval
                lam[n] = None
    return lam, arg


def select_distributed(local_result, n_star: int, theta: float = 0.0, group=None):
    """All-gather per-rank (lam, arg) and merge (every rank returns the same answer)."""
    import torch.distributed as dist
    world = dist.get_world_size(group)
    gathered = [None] * world
    dist.all_gather_object(gathered, local_result, group=group)
    lam, arg = merge_interval_maxima(gathered)
    return choose(lam, arg, n_star, theta)
