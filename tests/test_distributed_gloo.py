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


class _HostCalibration:
    """The two calls calibrate_distributed makes on the binding, computed on the
    host (the CPU stand-in for kvtc_calibrate_accumulate / _finalize): rows via
    the oracle's gather (keys un-RoPE'd, R1) rounded to bf16 like the GPU's
    gathered X; sum_x in fp64, X^T X in fp32; finalize = eigh of
    X^T X - n mu mu^T, descending, canonical sign (Q13)."""

    def __init__(self, caches):
        self.caches = caches

    def calibrate_accumulate(self, views, samples, which, sum_x, xtx, inv_freq=None, pairing=0):
        from oracle import numerics as ON
        from oracle import pca as OPCA
        C = OPCA.gather(self.caches, samples, which == 0, inv_freq, pairing)
        C = ON.bf16(C)
        sum_x += torch.from_numpy(C.sum(0))
        Xf = torch.from_numpy(C).float()
        xtx += Xf.T @ Xf

    def calibrate_finalize(self, shape, which, sum_x, xtx, n, rank_cap, inv_freq=None, pairing=0):
        mu = sum_x.numpy() / n
        S = xtx.double().numpy() - n * np.outer(mu, mu)
        w, V = np.linalg.eigh(S)
        order = np.argsort(-w, kind="stable")
        r = min(rank_cap, n - 1, len(mu))
        V = V[:, order[:r]]
        idx = np.argmax(np.abs(V), axis=0)
        V = V * np.sign(V[idx, np.arange(r)])
        return mu, V, np.sqrt(np.maximum(w[order[:r]], 0))


class _View:
    def __init__(self, shape):
        self.shape = shape


def _calib_worker(rank, world, port, caches, samples, invf, ret):
    from paper_2511_01815_b200.distributed import calibrate_distributed
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    l, t, h, d = caches[0][0][0].shape
    K = _HostCalibration(caches)
    out = {}
    for which in (0, 1):
        cs = [(c[which], p0) for c, p0 in caches]
        K.caches = cs
        out[which] = calibrate_distributed(K, [_View((l, h, d))], samples, which, 64, inv_freq=invf, device="cpu")
    # a layer shard (local=True) uses its own draw only, with no collective
    K.caches = [(c[1], p0) for c, p0 in caches]
    out["local"] = calibrate_distributed(K, [_View((l, h, d))], samples[rank::world], 1, 64, device="cpu", local=True)
    ret[rank] = out
    dist.destroy_process_group()


def test_calibrate_distributed_world2_equals_single_process():
    """The real orchestration (paper_2511_01815_b200.distributed.calibrate_distributed:
    shard the draw -> accumulate -> all-reduce sum_x, X^T X, n -> finalize) over
    gloo with world size 2: both ranks finalise the identical basis, equal to the
    oracle's fit of the whole draw."""
    from kvtc_inputs import generate, make_spec, sample_positions
    from oracle import numerics as ON
    from oracle import pca as OPCA
    spec = make_spec("toy")
    invf = spec.inv_freq().double().numpy()
    caches = [((generate(spec, 0, 700, conversation=c).double().numpy(),
                generate(spec, 1, 700, conversation=c).double().numpy()), 0) for c in (40, 41)]
    caches = [((k, v), p0) for (k, v), p0 in caches]
    samples = sample_positions([700, 700], 900, sinks=4, seed=3)
    port = _free_port()
    mgr = mp.Manager()
    ret = mgr.dict()
    mp.spawn(_calib_worker, args=(2, port, [((k, v), p0) for (k, v), p0 in caches], samples, invf, ret),
             nprocs=2, join=True)
    for which in (0, 1):
        mu0, V0, s0 = ret[0][which]
        mu1, V1, s1 = ret[1][which]
        np.testing.assert_array_equal(V0, V1)
        np.testing.assert_array_equal(mu0, mu1)
        C = ON.bf16(OPCA.gather([(c[which], p0) for c, p0 in caches], samples, which == 0, invf))
        ob = OPCA.fit(C, 64)
        np.testing.assert_allclose(mu0, ob.mu, rtol=1e-6, atol=1e-6)
        np.testing.assert_allclose(s0[:16], ob.sigma[:16], rtol=1e-4)
        cos = np.abs(np.sum(V0[:, :8] * ob.V[:, :8], axis=0))
        assert np.all(cos > 0.999), cos
    # local=True: each rank's basis is its own half of the draw (they differ)
    assert not np.array_equal(ret[0]["local"][1], ret[1]["local"][1])


# ---------------------------------------------------------------- joint cross-shard exchange
def _joint_worker(rank, world, port, Xs, V, ret):
    """Rank g holds the rows X_g of its layer shard and V_g (its rows of V): the
    reduce-scatter of the partial products must give each rank its tile-aligned
    slice of X V (block identity sum_g X_g V_g = X V), and the all-gather of the
    slices every row (joint.py; the kernels are replaced by torch matmuls here)."""
    from paper_2511_01815_b200.joint import all_gather_rows, reduce_scatter_rows, row_partition
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    f0 = sum(x.shape[1] for x in Xs[:rank])
    Xg = torch.from_numpy(Xs[rank])
    Vg = torch.from_numpy(V[f0:f0 + Xs[rank].shape[1]])
    P = Xg @ Vg
    mine = reduce_scatter_rows(P, world, rank)
    m = P.shape[0]
    full = all_gather_rows(mine, m, world, rank)
    ret[rank] = (mine.numpy().copy(), full.numpy().copy(), row_partition(m, world)[1][rank])
    dist.destroy_process_group()


@pytest.mark.parametrize("m", [1000, 100, 257])
def test_joint_exchange_world2(m):
    rng = np.random.default_rng(m)
    Xs = [rng.standard_normal((m, 48)), rng.standard_normal((m, 80))]       # two shards of 48 / 80 features
    V = rng.standard_normal((128, 24))
    port = _free_port()
    mgr = mp.Manager()
    ret = mgr.dict()
    mp.spawn(_joint_worker, args=(2, port, Xs, V, ret), nprocs=2, join=True)
    D = np.concatenate(Xs, axis=1) @ V                                       # the joint projection
    rows = []
    for r in range(2):
        mine, full, (r0, r1) = ret[r]
        assert (r0 % 128 == 0 or r0 == m) and mine.shape == (r1 - r0, 24)   # empty tail slices allowed
        np.testing.assert_allclose(mine, D[r0:r1], rtol=1e-12, atol=1e-12)
        np.testing.assert_allclose(full, D, rtol=1e-12, atol=1e-12)
        rows.append((r0, r1))
    assert rows[0][0] == 0 and rows[0][1] == rows[1][0] and rows[1][1] == m   # the slices tile the rows


def test_row_partition_properties():
    from paper_2511_01815_b200.joint import row_partition
    for m in (0, 1, 127, 128, 129, 1000, 32636):
        for world in (1, 2, 3, 8):
            per, parts = row_partition(m, world)
            assert per % 128 == 0 and world * per >= m
            assert parts[0][0] == 0 and parts[-1][1] == m
            for (a, b), (c, d) in zip(parts, parts[1:]):
                assert b == c and a <= b and (a % 128 == 0 or a == m)
