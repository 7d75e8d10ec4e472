"""Payload byte layout — oracle (test infrastructure).

Paper: "the quantized values are packed into a single byte array and further
compressed using the DEFLATE algorithm".  The byte order inside that
array is not given; this module writes out the layout chosen in DESIGN.md §4
(shared by the oracle and the GPU, each implementing it independently):

  * the m middle tokens are split into tiles of T = 128 tokens (last partial);
  * tile = params section, then codes section;
  * params: for each non-None group g (PC order), for each token: shift as
    binary16 bits (u16 LE), then scale (u16 LE);
  * codes: for each g, one block of ceil(ntok * size_g * bits_g / 8) bytes;
    token tau's code j sits at bits [(tau*size_g + j)*bits_g, +bits_g) of the
    block, LSB-first within bytes (DEFLATE's own bit order, RFC 1951 §3.1.1);
    fp8 codes are raw E4M3 bytes;
  * tiles are concatenated.  A full tile has exactly 128 * B_plan / 8 bytes.

Pins (tests/test_oracle_layout.py): unpack(pack(x)) == x; the 20-byte golden
vector of tests/golden/quant_pack_golden.json derived by hand from the rules
above; full-tile size == 16 * bits_per_token.
"""
from __future__ import annotations

import numpy as np

from .numerics import f16_bits, f16_from_bits
from .quant import BITS

TILE_TOKENS = 128


def tile_bytes(groups, ntok: int) -> int:
    G = len(groups)
    return 4 * G * ntok + sum((ntok * z * BITS[t] + 7) // 8 for (_, z, t) in groups)


def payload_bytes(groups, m: int) -> int:
    full, rem = divmod(m, TILE_TOKENS)
    return full * tile_bytes(groups, TILE_TOKENS) + (tile_bytes(groups, rem) if rem else 0)


def _pack_codes(codes, bits: int) -> bytes:
    codes = np.asarray(codes, dtype=np.uint64).reshape(-1)
    bitmat = ((codes[:, None] >> np.arange(bits, dtype=np.uint64)[None, :]) & 1).astype(np.uint8)
    return np.packbits(bitmat.reshape(-1), bitorder="little").tobytes()


def _unpack_codes(buf, count: int, bits: int) -> np.ndarray:
    raw = np.frombuffer(buf, dtype=np.uint8)
    b = np.unpackbits(raw, bitorder="little")[: count * bits].reshape(count, bits).astype(np.int64)
    return (b << np.arange(bits, dtype=np.int64)[None, :]).sum(axis=1)


def pack(groups, shifts, scales, codes, m: int) -> bytes:
    """groups: [(start, size, type)] non-None; shifts/scales: [G][m] fp16
    values; codes: list of [m, size_g] int arrays."""
    out = bytearray()
    for t0 in range(0, m, TILE_TOKENS):
        t1 = min(m, t0 + TILE_TOKENS)
        for g in range(len(groups)):
            pr = np.empty((t1 - t0, 2), dtype=np.uint16)
            pr[:, 0] = f16_bits(shifts[g][t0:t1])
            pr[:, 1] = f16_bits(scales[g][t0:t1])
            out += pr.astype("<u2").tobytes()
        for g, (_, z, t) in enumerate(groups):
            out += _pack_codes(np.asarray(codes[g])[t0:t1], BITS[t])
    return bytes(out)


def unpack(groups, payload: bytes, m: int):
    """Inverse of ``pack``: (shifts, scales, codes) with the same shapes."""
    G = len(groups)
    shifts = [np.zeros(m) for _ in range(G)]
    scales = [np.zeros(m) for _ in range(G)]
    codes = [np.zeros((m, z), dtype=np.int64) for (_, z, _) in groups]
    pos = 0
    for t0 in range(0, m, TILE_TOKENS):
        t1 = min(m, t0 + TILE_TOKENS)
        nt = t1 - t0
        for g in range(G):
            pr = np.frombuffer(payload, dtype="<u2", count=2 * nt, offset=pos).reshape(nt, 2)
            shifts[g][t0:t1] = f16_from_bits(pr[:, 0])
            scales[g][t0:t1] = f16_from_bits(pr[:, 1])
            pos += 4 * nt
        for g, (_, z, t) in enumerate(groups):
            nb = (nt * z * BITS[t] + 7) // 8
            codes[g][t0:t1] = _unpack_codes(payload[pos:pos + nb], nt * z, BITS[t]).reshape(nt, z)
            pos += nb
    if pos != len(payload):
        raise ValueError("payload length mismatch")
    return shifts, scales, codes
