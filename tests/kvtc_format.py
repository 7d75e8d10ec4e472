"""Readers of the library's byte formats for tests: entropy
sections and containers.  Parsing only — no codec arithmetic."""
from __future__ import annotations

import struct

import numpy as np

SECTION_HDR = struct.Struct("<IIQIIIIQQ16x")
CONTAINER_HDR = struct.Struct("<II6iqqqQQ2Q2Q2Q2QQ2QII2QQ56xQ")


def parse_section(buf: bytes):
    magic, ver, raw, chunk, nch, seg, nseg, data_off, total = SECTION_HDR.unpack_from(buf, 0)
    assert magic == 0x4454564B and ver == 3
    tab = np.frombuffer(buf, dtype=np.dtype([("off", "<u8"), ("bytes", "<u4"), ("kind", "<u4")]), count=nch,
                        offset=64)
    idx = np.frombuffer(buf, dtype="<u2", count=nch * nseg, offset=64 + 16 * nch).reshape(nch, nseg)
    assert data_off == 64 + 16 * nch + ((2 * nch * nseg + 15) & ~15)
    assert all(int(e["off"]) % 16 == 0 for e in tab)
    streams = [buf[data_off + int(e["off"]): data_off + int(e["off"]) + int(e["bytes"])] for e in tab]
    return dict(raw=raw, chunk=chunk, nchunks=nch, seg=seg, nseg=nseg, data_off=data_off, total=total,
                table=tab, index=idx, streams=streams)


def parse_container(buf: bytes):
    f = CONTAINER_HDR.unpack_from(buf, 0)
    names = ["magic", "version", "layers", "kv_heads", "head_dim", "sinks", "window", "chunk_bytes", "tokens", "pos0",
             "m", "total_bytes", "raw_bytes", "pay_k", "pay_v", "ent_k", "ent_v", "bfp_k", "bfp_v", "pfp_k", "pfp_v",
             "raw_off", "sec_k", "sec_v", "flags", "reserved", "hash_k", "hash_v", "raw_hash", "header_hash"]
    h = dict(zip(names, f))
    assert h["magic"] == 0x4354564B and h["version"] == 2 and CONTAINER_HDR.size == 256
    return h


def dynamic_header_bits(stream: bytes) -> int:
    """Bit length of the (single, final, dynamic) DEFLATE block header at the
    start of `stream` (RFC 1951 §3.2.7): the segment index counts from there."""
    bits = int.from_bytes(stream[:2048], "little")
    pos = 0

    def get(n):
        nonlocal pos
        v = (bits >> pos) & ((1 << n) - 1)
        pos += n
        return v

    return _dynamic_header(stream)[0]


def _canonical(lens):
    """(reversed code, length) per symbol, RFC 1951 §3.2.2."""
    cnt = [0] * 16
    for ln in lens:
        cnt[ln] += 1
    cnt[0] = 0
    nxt, code = [0] * 16, 0
    for b in range(1, 16):
        code = (code + cnt[b - 1]) << 1
        nxt[b] = code
    out = []
    for ln in lens:
        if ln:
            c = nxt[ln]
            nxt[ln] += 1
            out.append((int(format(c, f"0{ln}b")[::-1], 2), ln))
        else:
            out.append((0, 0))
    return out


def segment_bit_lengths(stream: bytes, nbytes: int, seg_bytes: int, nseg: int):
    """Decode one literal-only chunk stream symbol by symbol and return the bit
    length of each seg_bytes-symbol segment (the section's u16 index; the last
    segment includes the end-of-block code)."""
    hbits, lens = _dynamic_header(stream)
    codes = _canonical(lens[:257])
    table = np.full(1 << 15, -1, dtype=np.int64)
    for sym, (rc, ln) in enumerate(codes):
        if ln:
            table[rc::1 << ln] = (sym << 4) | ln
    bits = np.unpackbits(np.frombuffer(stream + b"\0" * 4, dtype=np.uint8), bitorder="little").astype(np.int64)
    win = np.zeros(len(bits) - 15, dtype=np.int64)
    for k in range(15):
        win += bits[k:len(bits) - 15 + k] << k
    pos, starts, out = hbits, [], []
    for i in range(nbytes + 1):
        if i % seg_bytes == 0 and i < nbytes:
            starts.append(pos)
        e = int(table[win[pos]])
        assert e >= 0
        sym = e >> 4
        assert (sym == 256) == (i == nbytes)
        if i < nbytes:
            out.append(sym)
        pos += e & 15
    ends = starts[1:] + [pos]
    lengths = [b - a for a, b in zip(starts, ends)] + [0] * (nseg - len(starts))
    return lengths, bytes(out), pos


def code_lengths(stream: bytes):
    """Literal/length code lengths (symbols 0..256) of a dynamic chunk stream."""
    return _dynamic_header(stream)[1][:257]


def _dynamic_header(stream: bytes):
    bits = int.from_bytes(stream[:2048], "little")
    pos = 0

    def get(n):
        nonlocal pos
        v = (bits >> pos) & ((1 << n) - 1)
        pos += n
        return v

    assert get(1) == 1 and get(2) == 2
    nlen, ndist, ncode = get(5) + 257, get(5) + 1, get(4) + 4
    order = [16, 17, 18, 0, 8, 7, 9, 6, 10, 5, 11, 4, 12, 3, 13, 2, 14, 1, 15]
    cl = [0] * 19
    for i in range(ncode):
        cl[order[i]] = get(3)
    # canonical code-length code, decoded bit by bit (MSB-first code bits)
    codes, code = {}, 0
    for ln in range(1, 8):
        for sym in range(19):
            if cl[sym] == ln:
                codes[(ln, code)] = sym
                code += 1
        code <<= 1
    lens = []
    while len(lens) < nlen + ndist:
        c, ln = 0, 0
        while (ln, c) not in codes:
            c = (c << 1) | get(1)
            ln += 1
            assert ln <= 7
        sym = codes[(ln, c)]
        if sym < 16:
            lens.append(sym)
        elif sym == 16:
            lens += [lens[-1]] * (3 + get(2))
        else:
            lens += [0] * (3 + get(3) if sym == 17 else 11 + get(7))
    return pos, lens


RANS_HDR = struct.Struct("<IIQIIQIIQQ8x")
RANS_CHUNK = np.dtype([("off", "<u8"), ("bytes", "<u4"), ("kind", "<u4")])


def _pad16(x: int) -> int:
    return (x + 15) & ~15


def parse_rans_section(buf: bytes):
    """rANS section (reading Q24): header, frequency tables, chunk table, streams."""
    magic, ver, raw, chunk, nch, period, sl, ncls, data_off, total = RANS_HDR.unpack_from(buf, 0)
    assert magic == 0x4154564B and ver == 1 and RANS_HDR.size == 64
    freqs = np.frombuffer(buf, dtype="<u2", count=ncls * 256, offset=64).reshape(ncls, 256).astype(np.int64)
    ctab_off = 64 + _pad16(ncls * 512)
    tab = np.frombuffer(buf, dtype=RANS_CHUNK, count=nch, offset=ctab_off)
    assert data_off == ctab_off + _pad16(16 * nch)
    streams = [(int(e["kind"]), buf[data_off + int(e["off"]): data_off + int(e["off"]) + int(e["bytes"])]) for e in tab]
    return dict(raw=raw, chunk=chunk, nchunks=nch, period=period, span_log2=sl, nclasses=ncls, data_off=data_off,
                total=total, freqs=freqs, table=tab, streams=streams)


def build_rans_section(freqs, sl: int, chunks, n: int, chunk: int, period: int) -> bytes:
    """The inverse of parse_rans_section (byte layout only): lets the GPU decoder
    read streams the oracle wrote."""
    freqs = np.asarray(freqs, dtype=np.int64)
    ncls = freqs.shape[0]
    ctab_off = 64 + _pad16(ncls * 512)
    data_off = ctab_off + _pad16(16 * len(chunks))
    tab, data, off = [], b"", 0
    for kind, st in chunks:
        tab.append(struct.pack("<QII", off, len(st), kind))
        data += st + b"\0" * (_pad16(len(st)) - len(st))
        off += _pad16(len(st))
    eff = max(1, min(period, n)) if period > 0 else max(1, n)          # the period the header records
    hdr = RANS_HDR.pack(0x4154564B, 1, n, chunk, len(chunks), eff, sl, ncls, data_off, data_off + off)
    body = freqs.astype("<u2").tobytes()
    out = hdr + body + b"\0" * (ctab_off - 64 - len(body))
    out += b"".join(tab) + b"\0" * (data_off - ctab_off - 16 * len(chunks))
    return out + data
