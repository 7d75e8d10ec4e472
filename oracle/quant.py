"""Grouped scalar quantiser — oracle (test infrastructure).

Paper: "we quantize groups of *subsequent* PCA coordinates together, each group
with shared 16-bit shift and scaling factors ... restricted to {1, 16, 64, 256,
1024} components per group. The total budget equals the sum of payload bits
across all coordinates plus per-group shift and scaling factors";
types [None, int2, int4, fp8] where None "quantizes data to the array of zeros"
at 0 bits; "we adopt KIVI's uniform quantization scheme"
(P:L466); fp8 is E4M3.

Readings, applied per token row and per group (Q1):
  Q1  shift/scale are per (token, group), charged 32 bits per token per group.
  Q2  int-k, k in {2,4}: asymmetric min-max.  shift = fp16(mn),
      scale = fp16((mx - mn) / (2^k - 1)); code = clamp(rne((x - shift)/scale),
      0, 2^k - 1) using the STORED fp16 shift/scale; x^ = code*scale + shift.
  Q3  fp8: shift = fp16((mx + mn)/2), scale = fp16(((mx - mn)/2)/448);
      code = E4M3(fp32((x - shift)/scale)) (RNE, saturating); x^ =
      e4m3(code)*scale + shift.
  Q5  scale == 0 (constant group, always for size 1): code 0, x^ = shift.
All arithmetic between those rounding points is fp64.

Pins (tests/test_oracle_quant.py): the hand-computed golden vector in
tests/golden/quant_pack_golden.json; {0,1,2,3} exact in int2; constant groups
exact; |x - x^| <= scale/2 inside the grid (half a quantisation step, the
north-star bound); fp8 relative error <= 2^-4 in the normal range.
"""
from __future__ import annotations

import numpy as np

from .numerics import f16, f32, e4m3_encode, e4m3_decode

T_NONE, T_INT2, T_INT4, T_FP8 = 0, 1, 2, 3
TYPES = (T_NONE, T_INT2, T_INT4, T_FP8)           # P:L1568 order
TYPE_NAMES = {T_NONE: "None", T_INT2: "int2", T_INT4: "int4", T_FP8: "fp8"}
BITS = {T_NONE: 0, T_INT2: 2, T_INT4: 4, T_FP8: 8}
SIZES = (1, 16, 64, 256, 1024)


def cost_bits(size: int, t: int) -> int:
    """Per-token bit cost of one group: 0 for None, else size*bits + 2*16."""
    return 0 if t == T_NONE else size * BITS[t] + 32


def quantize_rows(block, t: int):
    """Quantise each row of ``block`` [n, size] as one group of type ``t``.

    Returns (shift [n], scale [n], codes [n, size] int64) — shift/scale are
    fp16 values held in fp64, codes are int-k levels or E4M3 bytes."""
    x = np.asarray(block, dtype=np.float64)
    n, size = x.shape
    if t == T_NONE:
        return np.zeros(n), np.zeros(n), np.zeros((n, size), dtype=np.int64)
    mn = x.min(axis=1)
    mx = x.max(axis=1)
    if t in (T_INT2, T_INT4):
        levels = (1 << BITS[t]) - 1
        shift = f16(mn)
        scale = f16((mx - mn) / levels)
        with np.errstate(divide="ignore", invalid="ignore"):
            y = (x - shift[:, None]) / scale[:, None]
            codes = np.clip(np.round(y), 0, levels)
        codes = np.where(scale[:, None] == 0.0, 0.0, codes).astype(np.int64)
        return shift, scale, codes
    # fp8 (E4M3)
    shift = f16((mx + mn) / 2.0)
    scale = f16(((mx - mn) / 2.0) / 448.0)
    with np.errstate(divide="ignore", invalid="ignore"):
        y = f32((x - shift[:, None]) / scale[:, None])
    y = np.where(scale[:, None] == 0.0, 0.0, y)
    codes = e4m3_encode(y).astype(np.int64)
    codes = np.where(scale[:, None] == 0.0, 0, codes)
    return shift, scale, codes


def dequantize_rows(shift, scale, codes, t: int) -> np.ndarray:
    """x^ per Q2/Q3/Q5 in fp64 (no output rounding)."""
    codes = np.asarray(codes)
    if t == T_NONE:
        return np.zeros(codes.shape, dtype=np.float64)
    shift = np.asarray(shift, dtype=np.float64)[:, None]
    scale = np.asarray(scale, dtype=np.float64)[:, None]
    if t in (T_INT2, T_INT4):
        v = codes.astype(np.float64)
    else:
        v = e4m3_decode(codes)
    return v * scale + shift


def simulate_quantization(block, t: int):
    """The pseudocode's ``simulate_quantization``: (x^, used_bits)."""
    x = np.asarray(block, dtype=np.float64)
    shift, scale, codes = quantize_rows(x, t)
    return dequantize_rows(shift, scale, codes, t), cost_bits(x.shape[1], t)


def factors_finite(shift, scale) -> bool:
    """False when a 16-bit factor overflowed (the KVTC_E_NUMERIC condition)."""
    return bool(np.all(np.isfinite(shift)) and np.all(np.isfinite(scale)))
