"""Readers of the library's byte formats for tests: entropy
sections and containers.  Parsing only — no codec arithmetic."""
from __future__ import annotations

import struct

import numpy as np

SECTION_HDR = struct.Struct("<IIQIIIIQQ16x")
CONTAINER_HDR = struct.Struct("<II6iqqqQQ2Q2Q2Q2QQ2Q")


def parse_section(buf: bytes):
    magic, ver, raw, chunk, nch, seg, nseg, data_off, total = SECTION_HDR.unpack_from(buf, 0)
    assert magic == 0x4454564B and ver == 1
    tab = np.frombuffer(buf, dtype=np.dtype([("off", "<u8"), ("bytes", "<u4"), ("kind", "<u4")]), count=nch,
                        offset=64)
    idx = np.frombuffer(buf, dtype="<u4", count=nch * nseg, offset=64 + 16 * nch).reshape(nch, nseg)
    streams = [buf[data_off + int(e["off"]): data_off + int(e["off"]) + int(e["bytes"])] for e in tab]
    return dict(raw=raw, chunk=chunk, nchunks=nch, seg=seg, nseg=nseg, data_off=data_off, total=total,
                table=tab, index=idx, streams=streams)


def parse_container(buf: bytes):
    f = CONTAINER_HDR.unpack_from(buf, 0)
    names = ["magic", "version", "layers", "kv_heads", "head_dim", "sinks", "window", "chunk_bytes", "tokens", "pos0",
             "m", "total_bytes", "raw_bytes", "pay_k", "pay_v", "ent_k", "ent_v", "bfp_k", "bfp_v", "pfp_k", "pfp_v",
             "raw_off", "sec_k", "sec_v"]
    h = dict(zip(names, f))
    assert h["magic"] == 0x4354564B
    return h
