"""End-to-end KVTC compress / decompress — oracle (test infrastructure).

Paper: "Keys and values are compressed independently using the
(V, mu) parameters and bit allocation obtained during calibration"; "Decompression
reverses the compression steps"; the inverse projection "can be performed
layer-by-layer using sub-matrices of V^T".  Sinks and window: "We avoid
compressing both the w most recent tokens and s oldest tokens" with w=128, s=4
(P:L123-128).  CR: "we calculate CR only on the compressed tokens, not counting
the sliding window tokens"; Table 8 "count[s] the omitted sinks"
 — both are reported (Q16).

Per stream the oracle computes, in this order (rounding points R1-R7):
  X   = middle tokens flattened to rows (features (layer, head, dim));
        keys: R1 un-RoPE at absolute positions pos0 + s + tau.
  D   = X V_c - mu V_c                                          (fp64, R2)
  per (token, non-None group): shift, scale, codes            (oracle.quant, Q1-Q5)
  payload = oracle.layout.pack(...);  chunks = zlib raw DEFLATE  (Q15)
Decompress:
  payload = inflate; unpack; x^ per group; D^ = fp16(x^) (R5); uncovered PCs 0
  X^  = D^ V_d^T + mu (fp64, R6);  keys: RoPE at absolute positions (R7);
  bf16 RNE; sinks / window restored byte-identical.

End-to-end fidelity vs the paper is *parity unpinned* (the paper's errors are on
real caches); pinned here: sinks/window byte identity, lossless entropy stage,
monotone error in CR, DP <= pure-PCA truncation (tests/test_oracle_codec.py).
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import entropy, layout
from .numerics import bf16, f16
from .pca import Basis, flatten_rows, project
from .quant import quantize_rows, dequantize_rows, factors_finite
from .rope import unrope_r1, rope_apply_r7


def kv_cache_bytes(layers: int, heads: int, head_dim: int, tokens: int) -> int:
    """16-bit KV cache size 4*l*h*d_head*t bytes."""
    return 4 * layers * heads * head_dim * tokens


@dataclass
class StreamOut:
    payload: bytes
    chunks: list
    shifts: list
    scales: list
    codes: list
    D: np.ndarray


@dataclass
class Compressed:
    shape: tuple                  # (l, t, h, d)
    s: int
    w: int
    pos0: int
    m: int
    raw_k: np.ndarray             # sinks + window (bf16 values), [l, s+w, h, d]
    raw_v: np.ndarray
    k: StreamOut = None
    v: StreamOut = None
    stats: dict = field(default_factory=dict)


def stream_rows(cache, s: int, w: int, pos0: int, is_keys: bool, invf=None, pairing: int = 0):
    l, t, h, d = cache.shape
    mid = np.asarray(cache, dtype=np.float64)[:, s:t - w]
    if is_keys:
        pos = pos0 + s + np.arange(t - s - w)
        mid = unrope_r1(mid, pos, invf, pairing)
    return flatten_rows(mid)


def compress_stream(X, basis: Basis, plan, chunk: int = entropy.CHUNK_BYTES) -> StreamOut:
    groups = plan.groups
    m = X.shape[0]
    cols = np.concatenate([np.arange(s0, s0 + z) for (s0, z, _) in groups]) if groups else np.zeros(0, int)
    D = project(basis, X, cols)
    shifts, scales, codes = [], [], []
    off = 0
    for (_, z, t) in groups:
        sh, sc, cd = quantize_rows(D[:, off:off + z], t)
        if not factors_finite(sh, sc):
            raise FloatingPointError("16-bit shift/scale overflow (KVTC_E_NUMERIC)")
        shifts.append(sh)
        scales.append(sc)
        codes.append(cd)
        off += z
    payload = layout.pack(groups, shifts, scales, codes, m)
    return StreamOut(payload, entropy.deflate_chunks(payload, chunk), shifts, scales, codes, D)


def reconstruct_stream(payload: bytes, basis: Basis, plan, m: int) -> np.ndarray:
    groups = plan.groups
    shifts, scales, codes = layout.unpack(groups, payload, m)
    Dh = np.zeros((m, basis.r))
    for g, (s0, z, t) in enumerate(groups):
        Dh[:, s0:s0 + z] = f16(dequantize_rows(shifts[g], scales[g], codes[g], t))
    return Dh @ basis.Vd.T + basis.mu[None, :]


def compress(k_cache, v_cache, pos0: int, kb: Basis, kp, vb: Basis, vp, invf,
             pairing: int = 0, s: int = 4, w: int = 128, chunk: int = entropy.CHUNK_BYTES) -> Compressed:
    l, t, h, d = k_cache.shape
    raw_idx = np.r_[0:min(s, t), max(s, t - w):t] if t > s + w else np.arange(t)
    out = Compressed(shape=(l, t, h, d), s=s, w=w, pos0=pos0, m=max(0, t - s - w),
                     raw_k=np.asarray(k_cache)[:, raw_idx], raw_v=np.asarray(v_cache)[:, raw_idx])
    if t <= s + w:                                     # Q17: nothing to compress
        out.stats = {"nothing_to_compress": True}
        return out
    Xk = stream_rows(k_cache, s, w, pos0, True, invf, pairing)
    Xv = stream_rows(v_cache, s, w, pos0, False)
    out.k = compress_stream(Xk, kb, kp, chunk)
    out.v = compress_stream(Xv, vb, vp, chunk)
    p = l * h * d
    mid16 = 2 * 2 * p * out.m                                          # K+V, 16-bit
    pre = len(out.k.payload) + len(out.v.payload)
    post = sum(map(len, out.k.chunks)) + sum(map(len, out.v.chunks))
    table = 8 * (len(out.k.chunks) + len(out.v.chunks))              # u32 comp + u32 raw
    div = lambda a, b: a / b if b else float("inf")
    out.stats = {
        "cr_pre_deflate": div(mid16, pre),
        "cr": div(mid16, post + table),
        "cr_with_sinks": (mid16 + 2 * 2 * p * s) / (post + table + 2 * 2 * p * s),
        "deflate_gain": div(pre, post + table),
    }
    return out


def decompress(c: Compressed, kb: Basis, kp, vb: Basis, vp, invf, pairing: int = 0):
    l, t, h, d = c.shape
    s, w, m = c.s, c.w, c.m
    K = np.zeros((l, t, h, d))
    V = np.zeros((l, t, h, d))
    if t <= s + w:
        K[:], V[:] = c.raw_k, c.raw_v
        return K, V
    K[:, :s] = c.raw_k[:, :s]
    K[:, t - w:] = c.raw_k[:, s:]
    V[:, :s] = c.raw_v[:, :s]
    V[:, t - w:] = c.raw_v[:, s:]
    for so, basis, plan, dst, is_keys in ((c.k, kb, kp, K, True), (c.v, vb, vp, V, False)):
        payload = entropy.inflate_chunks(so.chunks)
        Xh = reconstruct_stream(payload, basis, plan, m).reshape(m, l, h, d).transpose(1, 0, 2, 3)
        if is_keys:
            Xh = rope_apply_r7(Xh, c.pos0 + s + np.arange(m), invf, pairing)
        else:
            Xh = bf16(Xh)
        dst[:, s:t - w] = Xh
    return K, V
