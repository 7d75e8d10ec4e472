"""Pins for oracle/rope.py: closed forms and invariants of a rotation."""
import math

import numpy as np
import torch

from oracle import rope
from kvtc_inputs import make_spec, generate


def test_closed_form_d2():
    # d_head = 2, base 1e4 -> theta_0 = 1; position 1 rotates [1, 0] to [cos 1, sin 1]
    invf = rope.inv_freq(2, 10000.0)
    assert invf[0] == 1.0
    y = rope.rope_rotate_f64(np.array([[[1.0, 0.0]]]), [1], invf, 0, +1)
    np.testing.assert_allclose(y[0, 0], [math.cos(1.0), math.sin(1.0)], atol=1e-7)


def test_position_zero_is_identity():
    rng = np.random.default_rng(0)
    x = rng.standard_normal((3, 4, 64))
    invf = rope.inv_freq(64, 500000.0)
    np.testing.assert_array_equal(rope.rope_rotate_f64(x, np.zeros(3), invf, 0, +1), x)
    np.testing.assert_array_equal(rope.rope_rotate_f64(x, np.zeros(3), invf, 1, -1), x)


def test_undo_apply_and_norm():
    rng = np.random.default_rng(1)
    x = rng.standard_normal((50, 2, 128))
    pos = rng.integers(0, 131072, 50)
    invf = rope.inv_freq(128, 500000.0)
    for pairing in (0, 1):
        y = rope.rope_rotate_f64(x, pos, invf, pairing, +1)
        z = rope.rope_rotate_f64(y, pos, invf, pairing, -1)
        # c, s are fp32-rounded, so c^2 + s^2 = 1 only to ~2^-23
        np.testing.assert_allclose(z, x, atol=4e-7 * np.abs(x).max())
        np.testing.assert_allclose(np.linalg.norm(y, axis=-1), np.linalg.norm(x, axis=-1), rtol=3e-7)


def test_r1_within_one_bf16_rounding_of_exact_rotation():
    rng = np.random.default_rng(2)
    from oracle.numerics import bf16
    x = bf16(rng.standard_normal((40, 3, 64)) * 3)
    pos = rng.integers(0, 40000, 40)
    invf = rope.inv_freq(64, 10000.0)
    r1 = rope.unrope_r1(x, pos, invf, 0)
    exact = rope.rope_rotate_f64(x, pos, invf, 0, -1)
    # one bf16 rounding (2^-9 relative) plus fp32 arithmetic slack
    np.testing.assert_array_less(np.abs(r1 - exact), 2.0 ** -8 * np.abs(exact) + 1e-6)


def test_unrope_restores_low_rank_structure():
    """RoPE distorts the low-rank structure of keys; undoing it with
    the model's convention (half-split, HF) restores it.  The synthetic model
    has K = 32 latent directions + 1 % isotropic noise in p = 128 features."""
    spec = make_spec("toy")
    t = 512
    k = generate(spec, 0, t, pos0=0).double().numpy()               # [l, t, h, d] post-RoPE
    invf = spec.inv_freq().double().numpy()
    pos = np.arange(t)

    def top_frac(kv):
        X = np.transpose(kv, (1, 0, 2, 3)).reshape(t, -1)[spec.sinks:]
        X = X - X.mean(axis=0)
        w = np.linalg.eigvalsh(X.T @ X)[::-1]
        return w[:spec.latent].sum() / w.sum()

    good = top_frac(rope.unrope_r1(k, pos, invf, 0))
    wrong_pairing = top_frac(rope.unrope_r1(k, pos, invf, 1))
    rotated = top_frac(k)
    assert good > 0.98
    assert rotated < good - 0.05 and wrong_pairing < good - 0.05
