"""Number formats used by the KVTC rounding points — oracle (test infrastructure).

The paper fixes the *widths*: the KV cache is 16-bit (bfloat16 in
P:L411), V is "stored in 16bit precision", each quantisation group has
"shared 16-bit shift and scaling factors", one element type is fp8
 in "the E4M3 format".  The formats themselves follow the
readings in DESIGN.md §3: IEEE binary16 for shift/scale (Q4), OCP E4M3FN with
round-to-nearest-even and saturation to +-448 (Q3), bf16 = top 16 bits of
binary32 with RNE.

Everything here is written out from the format definitions with exact fp64
arithmetic: ``round_to_format`` rounds to the nearest multiple of the format's
quantum 2**(e - mantissa_bits) (ties to even via ``np.round``), where e is the
exponent of the leading bit clamped below at the format's minimum normal
exponent (which yields subnormals).  Pins (tests/test_oracle_numerics.py):
fp16 / fp32 against NumPy's own casts, bf16 against torch's fp32->bf16 cast,
E4M3 against the OCP table enumerated from the spec and against
``torch.float8_e4m3fn`` after an explicit clamp to +-448.
"""
from __future__ import annotations

import numpy as np

# (mantissa bits, minimum normal exponent, largest finite value)
FP16 = (10, -14, 65504.0)
BF16 = (7, -126, float.fromhex("0x1.fep127"))
FP32 = (23, -126, float.fromhex("0x1.fffffep127"))
E4M3 = (3, -6, 448.0)


def round_to_format(x, fmt, saturate: bool = False):
    """Round fp64 ``x`` to the nearest value of ``fmt`` (ties to even).

    Overflow: +-inf (IEEE, ``saturate=False``) or clamp to +-max finite
    (``saturate=True``, the ".satfinite" behaviour used for E4M3, Q3).
    """
    man_bits, emin, max_finite = fmt
    x = np.asarray(x, dtype=np.float64)
    out = np.array(x, dtype=np.float64, copy=True)
    nz = np.isfinite(x) & (x != 0.0)
    if np.any(nz):
        xv = x[nz]
        _, e2 = np.frexp(np.abs(xv))          # |x| = m * 2**e2, m in [0.5, 1)
        e = np.maximum(e2 - 1, emin)           # exponent of the leading bit
        q = np.ldexp(1.0, (e - man_bits).astype(np.int64))   # the format's quantum
        y = np.round(xv / q) * q               # exact scaling; np.round ties to even
        big = np.abs(y) > max_finite
        if saturate:
            y = np.where(big, np.copysign(max_finite, xv), y)
        else:
            y = np.where(big, np.copysign(np.inf, xv), y)
        out[nz] = y
    if saturate:
        inf = np.isinf(x)
        out[inf] = np.copysign(max_finite, x[inf])
    return out


def f16(x):
    """IEEE binary16 RNE of fp64 values (Q4), returned as fp64."""
    return round_to_format(x, FP16)


def bf16(x):
    """bfloat16 RNE of fp64 values, returned as fp64."""
    return round_to_format(x, BF16)


def f32(x):
    """IEEE binary32 RNE of fp64 values, returned as fp64."""
    return round_to_format(x, FP32)


def f16_bits(x) -> np.ndarray:
    """binary16 bit patterns (uint16) of values already representable in fp16."""
    return np.asarray(x, dtype=np.float64).astype(np.float16).view(np.uint16)


def bf16_bits(x) -> np.ndarray:
    """bf16 bit patterns (uint16) of values already representable in bf16."""
    v = np.asarray(x, dtype=np.float64).astype(np.float32).view(np.uint32)
    return (v >> 16).astype(np.uint16)


def bf16_from_bits(b) -> np.ndarray:
    b = np.asarray(b, dtype=np.uint16).astype(np.uint32) << 16
    return b.view(np.float32).astype(np.float64)


def f16_from_bits(b) -> np.ndarray:
    return np.asarray(b, dtype=np.uint16).view(np.float16).astype(np.float64)


# ---------------------------------------------------------------- OCP E4M3FN
def _e4m3_table() -> np.ndarray:
    """Value of each of the 256 E4M3FN codes, from the format definition:
    sign bit 7, exponent bits 6..3 (bias 7), mantissa bits 2..0; exponent 0
    encodes subnormals (m/8)*2**-6; S.1111.111 is NaN; no infinities."""
    vals = np.empty(256, dtype=np.float64)
    for c in range(256):
        s = -1.0 if c & 0x80 else 1.0
        e = (c >> 3) & 0xF
        m = c & 0x7
        if e == 0xF and m == 0x7:
            vals[c] = np.nan
        elif e == 0:
            vals[c] = s * (m / 8.0) * 2.0 ** -6
        else:
            vals[c] = s * (1.0 + m / 8.0) * 2.0 ** (e - 7)
    return vals


E4M3_VALUES = _e4m3_table()


def e4m3_decode(codes) -> np.ndarray:
    return E4M3_VALUES[np.asarray(codes, dtype=np.int64)]


def e4m3_encode(y) -> np.ndarray:
    """E4M3FN code of fp64 ``y``: RNE, saturating to +-448, never NaN (Q3).

    The sign bit follows the sign of the rounded value, including -0."""
    v = round_to_format(y, E4M3, saturate=True)
    a = np.abs(v)
    sign = np.signbit(v).astype(np.int64) << 7
    code = np.zeros(a.shape, dtype=np.int64)
    sub = a < 2.0 ** -6
    code[sub] = np.round(a[sub] / 2.0 ** -9).astype(np.int64)      # exact: a is a multiple
    nrm = ~sub
    if np.any(nrm):
        _, e2 = np.frexp(a[nrm])
        e = e2 - 1
        m = (a[nrm] / np.ldexp(1.0, e) - 1.0) * 8.0
        code[nrm] = ((e + 7) << 3) | m.astype(np.int64)
    return (sign | code).astype(np.uint8)
