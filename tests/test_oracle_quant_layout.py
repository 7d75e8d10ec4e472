"""Pins for oracle/quant.py and oracle/layout.py."""
import json
import os

import numpy as np

from oracle import quant as Q
from oracle import layout as L
from oracle.numerics import f16_bits, e4m3_decode

GOLD = os.path.join(os.path.dirname(__file__), "golden", "quant_pack_golden.json")
GOLD_FP8 = os.path.join(os.path.dirname(__file__), "golden", "fp8_golden.json")

import pytest


@pytest.mark.parametrize("path", [GOLD, GOLD_FP8])
def test_golden_vector(path):
    """Hand-derived vectors (int2/int4: SURVEY §8(c); fp8: reading Q3 with the
    midpoint shift and half-range/448 scale, subnormal and saturated codes)."""
    g = json.load(open(path))
    rows = np.array(g["rows"])
    groups = [tuple(x) for x in g["groups"]]
    shifts, scales, codes = [], [], []
    for gi, (s0, z, t) in enumerate(groups):
        sh, sc, cd = Q.quantize_rows(rows[:, s0:s0 + z], t)
        assert list(f16_bits(sh)) == g["shift_bits"][gi]
        assert list(f16_bits(sc)) == g["scale_bits"][gi]
        assert cd.tolist() == g["codes"][gi]
        xh = Q.dequantize_rows(sh, sc, cd, t)
        np.testing.assert_array_equal(xh, np.array(g["xhat"])[:, s0:s0 + z])
        shifts.append(sh); scales.append(sc); codes.append(cd)
    payload = L.pack(groups, shifts, scales, codes, rows.shape[0])
    assert payload.hex() == g["payload_hex"]
    sh2, sc2, cd2 = L.unpack(groups, payload, rows.shape[0])
    for a, b in zip(cd2, codes):
        np.testing.assert_array_equal(a, b)


def test_int2_exact_levels_and_constant_groups():
    sh, sc, cd = Q.quantize_rows(np.array([[0.0, 1, 2, 3]]), Q.T_INT2)
    np.testing.assert_array_equal(Q.dequantize_rows(sh, sc, cd, Q.T_INT2), [[0, 1, 2, 3]])
    for t in (Q.T_INT2, Q.T_INT4, Q.T_FP8):
        blk = np.full((3, 5), 5.0)
        xh, bits = Q.simulate_quantization(blk, t)
        np.testing.assert_array_equal(xh, blk)
        assert bits == 5 * Q.BITS[t] + 32


def test_none_type_is_zero_and_free():
    xh, bits = Q.simulate_quantization(np.random.default_rng(0).standard_normal((4, 16)), Q.T_NONE)
    assert bits == 0 and not xh.any()
    assert Q.cost_bits(1, Q.T_INT2) == 34 and Q.cost_bits(1024, Q.T_FP8) == 8224


def test_half_step_bound_intk():
    """|x - x^| <= scale/2 inside the grid [shift, shift + L*scale] (north-star bound);
    outside it (fp16 rounding of shift/scale) the error is the clamp distance."""
    rng = np.random.default_rng(1)
    for t in (Q.T_INT2, Q.T_INT4):
        Lv = (1 << Q.BITS[t]) - 1
        for size in (1, 16, 64, 256):
            x = rng.standard_normal((200, size)) * rng.uniform(0.01, 100, (200, 1)) + rng.normal(0, 5, (200, 1))
            sh, sc, cd = Q.quantize_rows(x, t)
            xh = Q.dequantize_rows(sh, sc, cd, t)
            lo = sh[:, None]
            hi = sh[:, None] + Lv * sc[:, None]
            slack = np.maximum(0, lo - x) + np.maximum(0, x - hi)
            assert np.all(np.abs(x - xh) <= sc[:, None] / 2 + slack + 1e-12 * np.abs(x))


def test_fp8_relative_error():
    rng = np.random.default_rng(2)
    x = rng.standard_normal((300, 64)) * rng.uniform(0.1, 10, (300, 1))
    sh, sc, cd = Q.quantize_rows(x, Q.T_FP8)
    y = (x - sh[:, None]) / sc[:, None]
    yh = e4m3_decode(cd)
    normal = np.abs(y) >= 2.0 ** -6
    # 3 mantissa bits: half-ulp relative error <= 2^-4 (plus fp32 pre-rounding)
    assert np.all(np.abs(y - yh)[normal] <= 2.0 ** -4 * np.abs(y)[normal] * (1 + 1e-6))
    assert np.all(np.abs(y - yh)[~normal] <= 2.0 ** -10 + 1e-12)
    assert np.all(np.abs(y) <= 448 * (1 + 2.0 ** -9))


def test_layout_roundtrip_and_sizes():
    rng = np.random.default_rng(3)
    groups = [(0, 1, Q.T_INT2), (1, 1, Q.T_FP8), (2, 1, Q.T_INT4), (3, 16, Q.T_INT4),
              (19, 64, Q.T_INT2), (83, 16, Q.T_FP8)]
    for m in (1, 5, 127, 128, 129, 300):
        sh = [rng.standard_normal(m) for _ in groups]
        sc = [np.abs(rng.standard_normal(m)) for _ in groups]
        from oracle.numerics import f16
        sh = [f16(a) for a in sh]
        sc = [f16(a) for a in sc]
        cd = [rng.integers(0, 1 << Q.BITS[t], (m, z)) for (_, z, t) in groups]
        buf = L.pack(groups, sh, sc, cd, m)
        assert len(buf) == L.payload_bytes(groups, m)
        sh2, sc2, cd2 = L.unpack(groups, buf, m)
        for a, b in zip(cd, cd2):
            np.testing.assert_array_equal(a, b)
        for a, b in zip(sh, sh2):
            np.testing.assert_array_equal(a, b)
    bits = sum(Q.cost_bits(z, t) for (_, z, t) in groups)
    assert L.tile_bytes(groups, 128) == 16 * bits
