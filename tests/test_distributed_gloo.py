"""World-size-2 gloo tests (CPU) of the multi-GPU host logic: sample sharding,
LPT assignment, and the calibration-statistics all-reduce, whose sum over ranks
must equal the single-process statistics of the whole draw."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2511_01815_b200.distributed import allreduce_calibration, lpt_assign, shard_samples


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, C, ret):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rows = shard_samples(np.arange(C.shape[0]), rank, world)
    X = torch.from_numpy(C[rows])                              # this rank's bf16-valued rows
    sum_x = X.double().sum(0)
    xtx = (X.float().T @ X.float())
    n = allreduce_calibration(sum_x, xtx, len(rows))
    ret[rank] = (n, sum_x.numpy().copy(), xtx.numpy().copy())
    dist.destroy_process_group()


def test_calibration_allreduce_world2():
    rng = np.random.default_rng(0)
    C = (rng.standard_normal((301, 24)) * 3).astype(np.float32)
    C = torch.from_numpy(C).bfloat16().float().numpy()         # bf16-representable, like the gathered rows
    port = _free_port()
    mgr = mp.Manager()
    ret = mgr.dict()
    mp.spawn(_worker, args=(2, port, C, ret), nprocs=2, join=True)
    full_sum = C.astype(np.float64).sum(0)
    full_xtx = C.astype(np.float64).T @ C.astype(np.float64)
    for r in range(2):
        n, s, x = ret[r]
        assert n == 301
        np.testing.assert_allclose(s, full_sum, rtol=1e-12)
        np.testing.assert_allclose(x, full_xtx, rtol=1e-5, atol=1e-6 * np.abs(full_xtx).max())   # fp32 sums
    np.testing.assert_array_equal(ret[0][2], ret[1][2])       # every rank finalises the same matrix


def test_shard_samples_partition():
    s = np.arange(1001 * 2).reshape(-1, 2)
    parts = [shard_samples(s, r, 3) for r in range(3)]
    allrows = np.concatenate(parts)
    assert len(allrows) == len(s)
    assert sorted(map(tuple, allrows)) == sorted(map(tuple, s))


def test_lpt_assignment_balances():
    from kvtc_inputs import lengths_for
    lens = lengths_for(256, 8192, 32768, seed=0)
    for world in (1, 2, 4, 8):
        a = lpt_assign(lens, world)
        assert sorted(i for part in a for i in part) == list(range(256))
        loads = [sum(lens[i] for i in part) for part in a]
        assert max(loads) - min(loads) <= max(lens)              # LPT bound
        assert max(loads) / (sum(lens) / world) < 1.02
