"""Static-model interleaved rANS back-end -- oracle (test infrastructure).

Paper: the lossless stage can use other coders; the ablation lists ANS
(Duda 2014) beside DEFLATE, GDeflate, zstd, ... (Table at
P:L1320-1337).  The paper gives no format; reading Q24
 fixes the one the library implements, written out here step by
step:

  * model: order-0 byte frequencies per CLASS, class = (offset of the byte
    inside its 128-token payload tile) >> span_log2, one table per class
    estimated on the whole payload (the payload is tile-periodic: params, then
    each group's code block), so the tables cost ~nothing;
  * quantised to M = 2^12 by `normalize` (floor, forced 1s, the remainder to the
    most frequent symbol, excess taken from the largest counts);
  * chunks of chunk_bytes encoded independently; inside a chunk byte j goes to
    lane j % 32 of 32 interleaved rANS states (32-bit state, L = 2^16, 16-bit
    renormalisation: x >= f << 20 -> emit x & 0xFFFF, x >>= 16; then
    x = (x // f) * M + (x % f) + c), bytes processed from the last step to the
    first; the words a step emits are laid out in lane order, steps in reverse
    emission order, so a warp decoding steps forward reads them in order;
  * chunk stream = the 32 final states (u32 LE) then the words (u16 LE); a
    chunk whose stream would not be smaller than the raw bytes is stored raw.

Pins (tests/test_oracle_rans.py): lossless round trip; `normalize` on hand
examples and its invariants (sum M, f > 0 iff count > 0); the stream length
against the closed-form cost sum_i -log2(f_i / M) of the coded bytes (rANS is
within 32 x 16 bits of it per chunk); a one-lane worked example computed by
hand.
"""
from __future__ import annotations

import struct

import numpy as np

SCALE_BITS = 12
M = 1 << SCALE_BITS
L = 1 << 16
LANES = 32
MAGIC = 0x4154564B        # "KVTA"
VERSION = 1


def normalize(counts) -> np.ndarray:
    """Quantise byte counts to frequencies summing to M (Q24)."""
    h = np.asarray(counts, dtype=np.int64)
    n = int(h.sum())
    f = np.zeros(256, dtype=np.int64)
    if n == 0:
        return f
    for s in range(256):
        if h[s] > 0:
            f[s] = max(1, (int(h[s]) * M) // n)
    d = M - int(f.sum())
    if d > 0:
        f[int(np.argmax(h))] += d                  # argmax: first maximum (smallest symbol)
    while d < 0:
        s = int(np.argmax(f))
        take = min(-d, int(f[s]) - 1)
        f[s] -= take
        d += take
    return f


def span_log2(period: int) -> int:
    """Class span: a power of two >= 4096 giving <= 64 classes per period."""
    target = max(4096, -(-period // 64))
    b = 12
    while (1 << b) < target:
        b += 1
    return b


def classes_of(n: int, period: int, sl: int) -> np.ndarray:
    idx = np.arange(n, dtype=np.int64)
    return (idx % period) >> sl


def encode_chunk(data: np.ndarray, cls: np.ndarray, freqs: np.ndarray) -> bytes:
    """One chunk (uint8 array) -> its rANS stream (states + words)."""
    nc = len(data)
    steps = -(-nc // LANES)
    cum = np.zeros_like(freqs)
    cum[:, 1:] = np.cumsum(freqs, axis=1)[:, :-1]
    x = [L] * LANES
    out_words = []                                   # emitted words, in emission order (reversed at the end)
    for k in range(steps - 1, -1, -1):
        emitted = []
        for lane in range(LANES):
            j = k * LANES + lane
            if j >= nc:
                continue
            s = int(data[j])
            c = int(cls[j])
            f = int(freqs[c, s])
            start = int(cum[c, s])
            if x[lane] >= (f << 20):                 # renormalise: x < f 2^20 keeps x' < 2^32
                emitted.append(x[lane] & 0xFFFF)
                x[lane] >>= 16
            x[lane] = (x[lane] // f) * M + (x[lane] % f) + start
        # this step's words in lane order; steps are stored last-encoded first
        out_words.append(emitted)
    words = [w for step in reversed(out_words) for w in step]
    return struct.pack("<%dI" % LANES, *x) + struct.pack("<%dH" % len(words), *words)


def decode_chunk(stream: bytes, nc: int, cls: np.ndarray, freqs: np.ndarray) -> np.ndarray:
    x = list(struct.unpack_from("<%dI" % LANES, stream, 0))
    nwords = (len(stream) - 4 * LANES) // 2
    words = struct.unpack_from("<%dH" % nwords, stream, 4 * LANES)
    cum = np.zeros_like(freqs)
    cum[:, 1:] = np.cumsum(freqs, axis=1)[:, :-1]
    out = np.zeros(nc, dtype=np.uint8)
    pos = 0
    steps = -(-nc // LANES)
    for k in range(steps):
        for lane in range(LANES):
            j = k * LANES + lane
            if j >= nc:
                continue
            c = int(cls[j])
            slot = x[lane] & (M - 1)
            s = int(np.searchsorted(cum[c], slot, side="right") - 1)
            while freqs[c, s] == 0:                  # searchsorted lands on the last symbol of equal cum
                s -= 1
            f, start = int(freqs[c, s]), int(cum[c, s])
            out[j] = s
            x[lane] = f * (x[lane] >> SCALE_BITS) + slot - start
            if x[lane] < L:
                x[lane] = (x[lane] << 16) | words[pos]
                pos += 1
    if pos != nwords or any(v != L for v in x):
        raise ValueError("corrupt rANS chunk")
    return out


def encode(payload: bytes, chunk: int, period: int):
    """payload -> (freq tables [nclasses, 256], span_log2, [(kind, stream)] per chunk).
    period = the payload tile bytes (the whole payload when it has no tiles)."""
    a = np.frombuffer(payload, dtype=np.uint8)
    n = len(a)
    period = max(1, min(period, n)) if period > 0 else max(1, n)
    sl = span_log2(period)
    ncls = ((period - 1) >> sl) + 1
    cls = classes_of(n, period, sl)
    counts = np.zeros((ncls, 256), dtype=np.int64)
    np.add.at(counts, (cls, a.astype(np.int64)), 1)
    freqs = np.stack([normalize(counts[c]) for c in range(ncls)])
    chunks = []
    for b0 in range(0, n, chunk):
        d = a[b0:b0 + chunk]
        st = encode_chunk(d, cls[b0:b0 + chunk], freqs)
        if len(st) >= len(d):
            chunks.append((1, d.tobytes()))
        else:
            chunks.append((0, st))
    return freqs, sl, chunks


def decode(freqs, sl: int, chunks, n: int, chunk: int, period: int) -> bytes:
    period = max(1, min(period, n)) if period > 0 else max(1, n)
    cls = classes_of(n, period, sl)
    out = []
    for i, (kind, st) in enumerate(chunks):
        b0 = i * chunk
        nc = min(chunk, n - b0)
        out.append(st[:nc] if kind == 1 else decode_chunk(st, nc, cls[b0:b0 + nc], freqs).tobytes())
    return b"".join(out)


def cost_bits(payload: bytes, freqs, sl: int, period: int, b0: int = 0, b1: int | None = None) -> float:
    """The closed-form cost sum_i -log2(f(c_i, s_i) / M) of coding bytes [b0, b1)
    of the payload with the tables (what rANS achieves up to its flush)."""
    a = np.frombuffer(payload, dtype=np.uint8)
    n = len(a)
    b1 = n if b1 is None else b1
    period = max(1, min(period, n)) if period > 0 else max(1, n)
    cls = classes_of(n, period, sl)[b0:b1]
    f = np.asarray(freqs)[cls, a[b0:b1].astype(np.int64)].astype(np.float64)
    return float(-np.log2(f / M).sum())
