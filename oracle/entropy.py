"""Chunked DEFLATE — oracle (test infrastructure).

Paper: the packed byte array is "further compressed using the DEFLATE algorithm
... we leverage nvCOMP, which enables parallel operation directly on a GPU.
This step is lossless".  Reading Q15: 64 KiB chunks, each one raw
RFC-1951 stream (zlib ``wbits=-15``), zlib level 6 for the oracle.  GPU streams
need not be byte-equal to zlib's; the pin is the library routine itself:
zlib.decompress(zlib.compress(x)) == x (tests/test_oracle_codec.py).
"""
from __future__ import annotations

import zlib

CHUNK_BYTES = 65536


def deflate_chunks(payload: bytes, chunk: int = CHUNK_BYTES, level: int = 6):
    out = []
    for i in range(0, len(payload), chunk):
        c = zlib.compressobj(level=level, wbits=-15)
        out.append(c.compress(payload[i:i + chunk]) + c.flush())
    return out


def inflate_chunks(chunks) -> bytes:
    return b"".join(zlib.decompress(c, wbits=-15) for c in chunks)


def inflate_one(stream: bytes) -> bytes:
    return zlib.decompress(stream, wbits=-15)
