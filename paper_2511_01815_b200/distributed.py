"""Multi-GPU plumbing (host side).  Conversations are independent, so the data
path has no collective; the only exchange is the calibration all-reduce of the
per-rank sufficient statistics (sum_x, X^T X, n) before the eigensolver
(DESIGN.md §9).  torch.distributed does the transport (NCCL on GPUs, gloo in the
CPU tests)."""
from __future__ import annotations

import numpy as np
import torch


def shard_samples(samples, rank: int, world: int) -> np.ndarray:
    """This rank's share of the calibration draw (round-robin, so every rank gets
    a representative slice and the union is exactly the draw)."""
    return np.asarray(samples)[rank::world]


def lpt_assign(lengths, world: int):
    """Longest-processing-time assignment of conversations to ranks (weak scaling
    with unequal lengths): longest first to the least-loaded rank."""
    order = sorted(range(len(lengths)), key=lambda i: (-lengths[i], i))
    load = [0] * world
    out = [[] for _ in range(world)]
    for i in order:
        r = min(range(world), key=lambda k: (load[k], k))
        out[r].append(i)
        load[r] += lengths[i]
    return out


def allreduce_calibration(sum_x: torch.Tensor, xtx: torch.Tensor, n_local: int, group=None) -> int:
    """Sum the calibration statistics over all ranks in place; returns the total
    row count.  These are exactly what kvtc_calibrate_accumulate adds."""
    import torch.distributed as dist
    dist.all_reduce(sum_x, group=group)
    dist.all_reduce(xtx, group=group)
    n = torch.tensor([n_local], dtype=torch.int64, device=sum_x.device)
    dist.all_reduce(n, group=group)
    return int(n.item())


def calibrate_distributed(K, views, samples, which: int, rank_cap: int, inv_freq=None, pairing: int = 0,
                          group=None, local: bool = False, device="cuda"):
    """kvtc_calibrate_accumulate on this rank's shard of the draw -> all-reduce
    (NCCL on GPUs) -> kvtc_calibrate_finalize: every rank finalises the same
    statistics, hence the same basis.  local=True: this rank's own draw only, no
    collective (a layer shard of a pipeline-parallel model keeps its own basis,
    P:L443).  K is the binding (kvtc); the CPU tests pass an object with the same
    two calls (calibrate_accumulate / calibrate_finalize) and device="cpu"."""
    import torch.distributed as dist
    world = dist.get_world_size(group) if (dist.is_initialized() and not local) else 1
    rank = dist.get_rank(group) if (dist.is_initialized() and not local) else 0
    mine = shard_samples(samples, rank, world)
    p = views[0].shape[0] * views[0].shape[1] * views[0].shape[2]
    sum_x = torch.zeros(p, dtype=torch.float64, device=device)
    xtx = torch.zeros(p, p, dtype=torch.float32, device=device)
    K.calibrate_accumulate(views, mine, which, sum_x, xtx, inv_freq=inv_freq, pairing=pairing)
    n = allreduce_calibration(sum_x, xtx, len(mine), group) if world > 1 else len(mine)
    return K.calibrate_finalize(views[0].shape, which, sum_x, xtx, n, rank_cap, inv_freq=inv_freq, pairing=pairing)
