"""Pins for oracle/numerics.py against library routines and the format specs."""
import numpy as np
import torch

from oracle import numerics as nm


def _edge_values(rng):
    base = np.concatenate([
        rng.standard_normal(20000) * 10.0 ** rng.uniform(-9, 6, 20000),
        [0.0, -0.0, 1.0, -1.0, 65504.0, 65519.99, 65520.0, 1e-8, 2 ** -24, 2 ** -25,
         3 * 2 ** -26, 2 ** -14, 2 ** -15 + 2 ** -25, 1.0 + 2 ** -11, 1.0 + 3 * 2 ** -11],
    ])
    return base


def test_f16_matches_numpy_cast():
    rng = np.random.default_rng(0)
    x = _edge_values(rng)
    ref = x.astype(np.float16).astype(np.float64)
    got = nm.f16(x)
    np.testing.assert_array_equal(np.signbit(got), np.signbit(ref))
    np.testing.assert_array_equal(got, ref)


def test_f32_matches_numpy_cast():
    rng = np.random.default_rng(1)
    x = np.concatenate([_edge_values(rng), rng.standard_normal(1000) * 1e-40, [1e39, -1e39]])
    np.testing.assert_array_equal(nm.f32(x), x.astype(np.float32).astype(np.float64))


def test_bf16_matches_torch_cast_of_fp32():
    rng = np.random.default_rng(2)
    x32 = (rng.standard_normal(50000) * 10.0 ** rng.uniform(-30, 30, 50000)).astype(np.float32)
    x32 = np.concatenate([x32, np.array([1.0 + 2 ** -8, 1.0 + 3 * 2 ** -8, 1e-39, -1e-40], np.float32)])
    ref = torch.from_numpy(x32).to(torch.bfloat16).to(torch.float64).numpy()
    np.testing.assert_array_equal(nm.bf16(x32.astype(np.float64)), ref)


def test_bits_roundtrip():
    v = nm.f16(np.array([0.0, -1.5, 0.05, 10.0, 65504.0, 2 ** -24]))
    np.testing.assert_array_equal(nm.f16_from_bits(nm.f16_bits(v)), v)
    assert list(nm.f16_bits(np.array([-1.5, 10.0, 1.0]))) == [0xBE00, 0x4900, 0x3C00]
    b = nm.bf16(np.array([1.0, -2.5, 3.140625]))
    np.testing.assert_array_equal(nm.bf16_from_bits(nm.bf16_bits(b)), b)


def test_e4m3_table_from_spec():
    t = nm.E4M3_VALUES
    assert t[0x00] == 0.0 and np.signbit(t[0x80])
    assert t[0x7E] == 448.0 and t[0xFE] == -448.0
    assert np.isnan(t[0x7F]) and np.isnan(t[0xFF])
    assert t[0x01] == 2.0 ** -9            # smallest subnormal
    assert t[0x08] == 2.0 ** -6            # smallest normal
    assert t[0x38] == 1.0
    finite = ~np.isnan(t)
    assert finite.sum() == 254


def test_e4m3_exhaustive_roundtrip():
    for c in range(256):
        v = nm.E4M3_VALUES[c]
        if np.isnan(v):
            continue
        assert int(nm.e4m3_encode(np.array([v]))[0]) == c, hex(c)


def test_e4m3_rne_and_saturation():
    enc = lambda v: int(nm.e4m3_encode(np.array([v]))[0])
    assert enc(2.0 ** -10) == 0x00                    # tie between 0 and 2^-9 -> even (0)
    assert enc(3 * 2.0 ** -10) == 0x02                # tie between codes 1 and 2 -> even (2)
    assert enc(1.0 + 1.0 / 16) == 0x38                # tie 1.0 / 1.125 -> even mantissa (1.0)
    assert enc(1.0 + 3.0 / 16) == 0x3A                # tie 1.125 / 1.25 -> 1.25 (m=2)
    assert enc(448.0) == 0x7E and enc(500.0) == 0x7E and enc(1e9) == 0x7E
    assert enc(-1e9) == 0xFE and enc(np.inf) == 0x7E
    assert enc(-1e-12) == 0x80                         # sign of a rounded-to-zero value kept


def test_e4m3_matches_torch_after_clamp():
    rng = np.random.default_rng(3)
    y = (rng.standard_normal(100000) * 10.0 ** rng.uniform(-4, 3, 100000)).astype(np.float32)
    y = np.clip(y, -448, 448)
    ref = torch.from_numpy(y).to(torch.float8_e4m3fn).view(torch.uint8).numpy()
    got = nm.e4m3_encode(y.astype(np.float64))
    np.testing.assert_array_equal(got, ref)
