"""RoPE removal / re-application — oracle (test infrastructure).

Paper: keys are compressed *before* RoPE — "positional embeddings distort the
apparent low-rank structure of keys and should be removed before compression"
(P:L219-220), calibration rows "undo positional rotations", "we apply
compression before RoPE"; the cache layout and attention are unchanged
(P:L454), so decompression re-rotates the keys.  Values are never rotated.

Readings:
  Q10  the caller supplies inv_freq[d/2] (fp32) and the pairing: half-split
       (j, j+d/2) [default, HF Llama/Mistral] or interleaved (2j, 2j+1).
       Positions are absolute: pos0 + token index.
  R1   angle theta = fp32(fp32(pos) * inv_freq[j]); c, s = fp32(cos/sin(theta))
       evaluated in fp64; un-RoPE in fp32 arithmetic (products and the sum each
       rounded to fp32), then ONE bf16 RNE:  k_pre = bf16(unrope_fp32(k_post)).
       (fp64 evaluation of a single fp32 product / sum followed by rounding to
       fp32 equals the fp32 operation: 53 >= 2*24+2, no double-rounding error.)
  R7   re-application in fp64 between rounding points using the same c, s, then
       a single bf16 RNE.

Pins (tests/test_oracle_rope.py): closed form d=2, base 1e4, pos 1, [1,0] ->
[cos 1, sin 1]; undo(apply(x)) = x and norm preservation in exact fp64;
position 0 is the identity.
"""
from __future__ import annotations

import numpy as np

from .numerics import bf16, f32


def inv_freq(head_dim: int, base: float) -> np.ndarray:
    """Standard RoPE frequencies base**(-2j/d), as fp32 values (returned fp64)."""
    j = np.arange(head_dim // 2, dtype=np.float64)
    return f32(base ** (-2.0 * j / head_dim))


def cos_sin(positions, invf) -> tuple[np.ndarray, np.ndarray]:
    """R1 tables: c, s of shape [len(positions), d/2] (fp32 values in fp64)."""
    pos = f32(np.asarray(positions, dtype=np.float64))
    theta = f32(pos[:, None] * np.asarray(invf, dtype=np.float64)[None, :])
    return f32(np.cos(theta)), f32(np.sin(theta))


def _pairs(head_dim: int, pairing: int):
    h = head_dim // 2
    if pairing == 0:
        return np.arange(h), np.arange(h) + h
    return np.arange(0, head_dim, 2), np.arange(1, head_dim, 2)


def unrope_r1(k, positions, invf, pairing: int = 0) -> np.ndarray:
    """R1: k_pre = bf16(unrope_fp32(k_post)).

    ``k``: [..., t, h, d] bf16 values (fp64 array), token axis -3; positions [t].
    Rotation by -theta:  x1' = x1*c + x2*s,  x2' = x2*c - x1*s.
    """
    k = np.asarray(k, dtype=np.float64)
    d = k.shape[-1]
    i1, i2 = _pairs(d, pairing)
    c, s = cos_sin(positions, invf)
    c = c[:, None, :]
    s = s[:, None, :]
    x1 = k[..., i1]
    x2 = k[..., i2]
    out = np.empty_like(k)
    out[..., i1] = f32(f32(x1 * c) + f32(x2 * s))
    out[..., i2] = f32(f32(x2 * c) - f32(x1 * s))
    return bf16(out)


def rope_apply_r7(x, positions, invf, pairing: int = 0) -> np.ndarray:
    """R7: rotation by +theta in fp64 using the R1 tables, then bf16 RNE.

    x1' = x1*c - x2*s,  x2' = x2*c + x1*s.
    """
    return bf16(rope_rotate_f64(x, positions, invf, pairing, +1))


def rope_rotate_f64(x, positions, invf, pairing: int = 0, direction: int = +1) -> np.ndarray:
    """Plain fp64 rotation (no output rounding) by direction*theta."""
    x = np.asarray(x, dtype=np.float64)
    d = x.shape[-1]
    i1, i2 = _pairs(d, pairing)
    c, s = cos_sin(positions, invf)
    c = c[:, None, :]
    s = s[:, None, :] * direction
    x1 = x[..., i1]
    x2 = x[..., i2]
    out = np.empty_like(x)
    out[..., i1] = x1 * c - x2 * s
    out[..., i2] = x2 * c + x1 * s
    return out
