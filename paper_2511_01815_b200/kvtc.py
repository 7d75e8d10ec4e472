"""Thin Python binding over the C ABI (include/kvtc.h).

Argument marshalling only: torch tensors provide device memory and streams;
every step of the path runs in libkvtc.so's sm_100a kernels.  Names follow the
C entry points (kvtc_<name>).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib as L
from ._lib import KvtcError, check, lib  # noqa: F401  (KvtcError: the status-carrying exception)


def _stream(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def _ptr(t: torch.Tensor | None):
    return C.c_void_p(0 if t is None else t.data_ptr())


def _f32p(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_float))


def _i32p(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_int32))


def device_check() -> None:
    check(lib().kvtc_device_check())


# ------------------------------------------------------------------- views
class KVView:
    """A cache of one stream as the C ABI sees it (kvtc_kv_view).

    contiguous: tensor [layers, tokens, kv_heads, head_dim] bf16 (or a list of
    per-layer [tokens, kv_heads, head_dim] tensors);
    paged: pages [layers, num_pages, page_tokens, kv_heads, head_dim] bf16 and
    block_table int32 [ceil(tokens / page_tokens)] on the device."""

    def __init__(self, cache, pos0: int = 0, tokens: int | None = None, block_table: torch.Tensor | None = None):
        layers = list(cache) if isinstance(cache, (list, tuple)) else [cache[i] for i in range(cache.shape[0])]
        for t in layers:
            assert t.dtype == torch.bfloat16 and t.is_cuda and t.is_contiguous()
        self._keep = (cache, layers, block_table)
        paged = block_table is not None
        if paged:
            _, page_tokens, h, d = layers[0].shape
            assert tokens is not None
        else:
            t0, h, d = layers[0].shape
            tokens = t0 if tokens is None else tokens
            page_tokens = 0
        self.shape = (len(layers), h, d)
        self.tokens = tokens
        self.pos0 = pos0
        self._bases = (C.c_void_p * len(layers))(*[x.data_ptr() for x in layers])
        self.c = L.View(L.Shape(len(layers), h, d), tokens, pos0, L.LAYOUT_PAGED if paged else L.LAYOUT_CONTIGUOUS,
                        page_tokens, C.cast(self._bases, C.POINTER(C.c_void_p)),
                        C.c_void_p(block_table.data_ptr() if paged else 0), 1, 0)


def _rope(inv_freq, pairing: int):
    a = np.ascontiguousarray(np.asarray(inv_freq, dtype=np.float32))
    return L.Rope(_f32p(a), pairing), a


# ------------------------------------------------------------------- basis
class Basis:
    """kvtc_basis: mu, V (fp32 master) -> bf16 / fp16 GEMM operands (R2, R6)."""

    def __init__(self, handle, shape, which):
        self.h = C.c_void_p(handle) if not isinstance(handle, C.c_void_p) else handle
        self.shape = shape
        self.which = which

    @classmethod
    def create(cls, shape, which: int, mu, V, sigma=None, inv_freq=None, pairing: int = 0) -> "Basis":
        mu = np.ascontiguousarray(np.asarray(mu, dtype=np.float32))
        V = np.ascontiguousarray(np.asarray(V, dtype=np.float32))
        r = V.shape[1]
        sg = None if sigma is None else np.ascontiguousarray(np.asarray(sigma, dtype=np.float32))
        rope, keep = _rope(inv_freq, pairing) if inv_freq is not None else (None, None)
        out = C.c_void_p()
        check(lib().kvtc_basis_create(C.byref(L.Shape(*shape)), which, C.byref(rope) if rope else None, r,
                                      _f32p(mu), _f32p(V), _f32p(sg) if sg is not None else None, C.byref(out)))
        return cls(out, tuple(shape), which)

    def get(self):
        p, r = C.c_int32(), C.c_int32()
        check(lib().kvtc_basis_get(self.h, C.byref(p), C.byref(r), None, None, None))
        mu = np.empty(p.value, np.float32)
        V = np.empty((p.value, r.value), np.float32)
        sg = np.empty(r.value, np.float32)
        check(lib().kvtc_basis_get(self.h, None, None, _f32p(mu), _f32p(V), _f32p(sg)))
        return mu, V, sg

    def __del__(self):
        try:
            if self.h:
                lib().kvtc_basis_destroy(self.h)
        except Exception:
            pass


# -------------------------------------------------------------------- plan
@dataclass
class PlanInfo:
    r: int
    groups: list          # [(start, size, type)]
    bits_per_token: int
    r_eff: int
    expected_error: float
    budget: int


class Plan:
    def __init__(self, handle):
        self.h = handle if isinstance(handle, C.c_void_p) else C.c_void_p(handle)

    @classmethod
    def create(cls, r: int, groups) -> "Plan":
        g = np.asarray(groups, dtype=np.int32).reshape(-1, 3)
        st, sz, tp = (np.ascontiguousarray(g[:, i]) for i in range(3))
        out = C.c_void_p()
        check(lib().kvtc_plan_create(r, len(g), _i32p(st), _i32p(sz), _i32p(tp), C.byref(out)))
        return cls(out)

    def info(self) -> PlanInfo:
        r, n = C.c_int32(), C.c_int32()
        check(lib().kvtc_plan_get(self.h, C.byref(r), C.byref(n), None, None, None, None, None, None, None))
        st, sz, tp = (np.empty(max(1, n.value), np.int32) for _ in range(3))
        bits, reff, err, bud = C.c_int64(), C.c_int32(), C.c_double(), C.c_int64()
        check(lib().kvtc_plan_get(self.h, None, C.byref(n), _i32p(st), _i32p(sz), _i32p(tp), C.byref(bits),
                                  C.byref(reff), C.byref(err), C.byref(bud)))
        groups = [(int(st[i]), int(sz[i]), int(tp[i])) for i in range(n.value)]
        return PlanInfo(r.value, groups, bits.value, reff.value, err.value, bud.value)

    def payload_bytes(self, m: int) -> int:
        return int(lib().kvtc_payload_bytes(self.h, m))

    def __del__(self):
        try:
            if self.h:
                lib().kvtc_plan_destroy(self.h)
        except Exception:
            pass


# ------------------------------------------------------------ stage calls
def gather(view: KVView, tok_begin: int, ntok: int, unrope: bool, inv_freq=None, pairing: int = 0, stream=None):
    p = view.shape[0] * view.shape[1] * view.shape[2]
    X = torch.empty(ntok, p, dtype=torch.bfloat16, device="cuda")
    rope, keep = _rope(inv_freq, pairing) if unrope else (None, None)
    check(lib().kvtc_stage_gather(C.byref(view.c), tok_begin, ntok, int(unrope), C.byref(rope) if rope else None,
                                  _ptr(X), _stream(stream)))
    return X


def project(basis: Basis, plan: Plan | None, X: torch.Tensor, ncols: int, stream=None):
    D = torch.empty(X.shape[0], ncols, dtype=torch.float32, device="cuda")
    check(lib().kvtc_stage_project(basis.h, plan.h if plan else None, _ptr(X), X.shape[0], _ptr(D), _stream(stream)))
    return D


def project_partial(basis: Basis, plan: Plan, X: torch.Tensor, feat_begin: int, feat_end: int, add_bias: bool,
                    stream=None):
    """Joint cross-shard compression: this shard's partial projection (fp32 [m x ncols(plan)])."""
    ncols = sum(z for (_, z, _) in plan.info().groups)
    D = torch.zeros(X.shape[0], max(ncols, 1), dtype=torch.float32, device="cuda")
    check(lib().kvtc_stage_project_partial(basis.h, plan.h, _ptr(X), X.shape[0], feat_begin, feat_end, int(add_bias),
                                           _ptr(D), _stream(stream)))
    return D[:, :ncols]


def quantize_pack(plan: Plan, D: torch.Tensor, stream=None):
    m = D.shape[0]
    out = torch.zeros(plan.payload_bytes(m) + 16, dtype=torch.uint8, device="cuda")
    check(lib().kvtc_stage_quantize_pack(plan.h, _ptr(D), m, _ptr(out), _stream(stream)))
    return out[: plan.payload_bytes(m)]


def project_quantize(basis: Basis, plan: Plan, X: torch.Tensor, stream=None):
    m = X.shape[0]
    out = torch.zeros(plan.payload_bytes(m) + 16, dtype=torch.uint8, device="cuda")
    check(lib().kvtc_stage_project_quantize(basis.h, plan.h, _ptr(X), m, _ptr(out), _stream(stream)))
    return out[: plan.payload_bytes(m)]


def deflate(data: torch.Tensor, chunk_bytes: int = 65536, stream=None):
    n = data.numel()
    cap = int(lib().kvtc_deflate_bound(n, chunk_bytes))
    out = torch.zeros(cap + 16, dtype=torch.uint8, device="cuda")
    wsb = int(lib().kvtc_deflate_workspace_bytes(n, chunk_bytes))
    ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
    ln = C.c_size_t()
    check(lib().kvtc_stage_deflate(_ptr(data), n, chunk_bytes, _ptr(out), cap + 16, C.byref(ln), _ptr(ws), wsb,
                                   _stream(stream)))
    return out[: ln.value]


def rans_encode(data: torch.Tensor, tile_bytes: int = 0, chunk_bytes: int = 65536, stream=None):
    """rANS back-end (reading Q24): payload bytes -> section (device uint8)."""
    n = data.numel()
    cap = int(lib().kvtc_rans_bound(n, chunk_bytes, tile_bytes))
    out = torch.zeros(cap + 16, dtype=torch.uint8, device="cuda")
    wsb = int(lib().kvtc_rans_workspace_bytes(n, chunk_bytes, tile_bytes))
    ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
    ln = C.c_size_t()
    check(lib().kvtc_stage_rans_encode(_ptr(data), n, chunk_bytes, tile_bytes, _ptr(out), cap + 16, C.byref(ln),
                                       _ptr(ws), wsb, _stream(stream)))
    return out[: ln.value]


def rans_decode(section: torch.Tensor, n_out: int, stream=None):
    out = torch.zeros(max(n_out, 1), dtype=torch.uint8, device="cuda")
    check(lib().kvtc_stage_rans_decode(_ptr(section), section.numel(), _ptr(out), n_out, _stream(stream)))
    return out[:n_out]


def inflate(section: torch.Tensor, n_out: int, stream=None):
    out = torch.empty(n_out + 16, dtype=torch.uint8, device="cuda")
    sec = torch.zeros(section.numel() + 64, dtype=torch.uint8, device="cuda")
    sec[: section.numel()] = section
    check(lib().kvtc_stage_inflate(_ptr(sec), section.numel(), _ptr(out), n_out, _stream(stream)))
    return out[:n_out]


def inflate_raw(streams: list, out_lens: list, stream=None):
    """Generic inflate of independent raw DEFLATE streams (e.g. zlib wbits=-15)."""
    in_off = np.cumsum([0] + [len(s) for s in streams])[:-1].astype(np.int64)
    out_off = np.cumsum([0] + list(out_lens))[:-1].astype(np.int64)
    blob = np.frombuffer(b"".join(streams) + b"\0" * 16, dtype=np.uint8)
    dev = torch.from_numpy(blob.copy()).cuda()
    t = lambda a: torch.from_numpy(np.asarray(a, dtype=np.int64)).cuda()
    out = torch.zeros(int(sum(out_lens)) + 16, dtype=torch.uint8, device="cuda")
    status = torch.zeros(len(streams), dtype=torch.int32, device="cuda")
    ioff, ilen, ooff, olen = t(in_off), t([len(s) for s in streams]), t(out_off), t(out_lens)
    check(lib().kvtc_stage_inflate_raw(_ptr(dev), _ptr(ioff), _ptr(ilen), len(streams), _ptr(out), _ptr(ooff),
                                       _ptr(olen), _ptr(status), _stream(stream)))
    torch.cuda.synchronize()
    return out[: int(sum(out_lens))], status


def dequantize(plan: Plan, payload: torch.Tensor, m: int, ld: int | None = None, stream=None):
    ncols = sum(z for (_, z, _) in plan.info().groups)
    ld = ld or max(8, (ncols + 7) // 8 * 8)
    Dh = torch.zeros(m, ld, dtype=torch.float16, device="cuda")
    check(lib().kvtc_stage_dequantize(plan.h, _ptr(payload), m, _ptr(Dh), ld, _stream(stream)))
    return Dh


def reconstruct(basis: Basis, plan: Plan, Dh: torch.Tensor, m: int, tok_begin: int, layer_begin: int,
                layer_end: int, out: KVView, stream=None):
    check(lib().kvtc_stage_reconstruct(basis.h, plan.h, _ptr(Dh), Dh.shape[1], m, tok_begin, layer_begin, layer_end,
                                       C.byref(out.c), _stream(stream)))


def reconstruct_payload(basis: Basis, plan: Plan, payload: torch.Tensor, m: int, tok_begin: int, layer_begin: int,
                        layer_end: int, out: KVView, stream=None):
    """D2 + K5 fused: the reconstruction GEMM dequantising its A operand from the payload."""
    check(lib().kvtc_stage_reconstruct_payload(basis.h, plan.h, _ptr(payload), m, tok_begin, layer_begin, layer_end,
                                               C.byref(out.c), _stream(stream)))


# ------------------------------------------------------------------ codec
def compress(kb: Basis, kp: Plan, vb: Basis, vp: Plan, k: KVView, v: KVView, sinks: int = 4, window: int = 128,
             chunk_bytes: int = 65536, stream=None, out: torch.Tensor | None = None, workspace=None,
             sync_len: bool = True, coder: int = 0):
    """Returns (container tensor [len], status).  coder: 0 DEFLATE, 1 rANS (Q24)."""
    pol = L.Policy(sinks, window, chunk_bytes, coder)
    cap = int(lib().kvtc_compress_bound(kp.h, vp.h, C.byref(k.c), C.byref(pol)))
    wsb = int(lib().kvtc_compress_workspace_bytes(kb.h, kp.h, vb.h, vp.h, C.byref(k.c), C.byref(pol)))
    if out is None:
        out = torch.empty(cap, dtype=torch.uint8, device="cuda")
    if workspace is None:
        workspace = torch.empty(wsb, dtype=torch.uint8, device="cuda")
    ln = C.c_size_t(0)
    st = check(lib().kvtc_compress(kb.h, kp.h, vb.h, vp.h, C.byref(k.c), C.byref(v.c), C.byref(pol), _ptr(out),
                                   out.numel(), C.byref(ln) if sync_len else None, _ptr(workspace),
                                   workspace.numel(), _stream(stream)),
               allow=(L.KVTC_OK, L.KVTC_NOTHING_TO_COMPRESS))
    return (out[: ln.value] if sync_len else out), st


def compress_sizes(kb, kp, vb, vp, k: KVView, sinks=4, window=128, chunk_bytes=65536, coder: int = 0):
    pol = L.Policy(sinks, window, chunk_bytes, coder)
    cap = int(lib().kvtc_compress_bound(kp.h, vp.h, C.byref(k.c), C.byref(pol)))
    wsb = int(lib().kvtc_compress_workspace_bytes(kb.h, kp.h, vb.h, vp.h, C.byref(k.c), C.byref(pol)))
    return cap, wsb


def container_info(container: torch.Tensor) -> L.ContainerInfo:
    hdr = container[: L.HEADER_BYTES].cpu().numpy().tobytes()
    info = L.ContainerInfo()
    check(lib().kvtc_container_parse(C.c_char_p(hdr), C.byref(info)))
    return info


def decompress_workspace_bytes(kb, kp, vb, vp, header: bytes) -> int:
    return int(lib().kvtc_decompress_workspace_bytes(kb.h, kp.h, vb.h, vp.h, C.c_char_p(header)))


def decompress(kb: Basis, kp: Plan, vb: Basis, vp: Plan, container: torch.Tensor, k_out: KVView, v_out: KVView,
               layer_begin: int = 0, layer_end: int | None = None, stream=None, workspace=None):
    layer_end = k_out.shape[0] if layer_end is None else layer_end
    if workspace is None:
        hdr = container[: L.HEADER_BYTES].cpu().numpy().tobytes().ljust(L.HEADER_BYTES, b"\0")
        workspace = torch.empty(decompress_workspace_bytes(kb, kp, vb, vp, hdr), dtype=torch.uint8, device="cuda")
    check(lib().kvtc_decompress(kb.h, kp.h, vb.h, vp.h, _ptr(container), container.numel(), layer_begin, layer_end,
                                C.byref(k_out.c), C.byref(v_out.c), _ptr(workspace), workspace.numel(),
                                _stream(stream)))


def decompress_async(kb: Basis, kp: Plan, vb: Basis, vp: Plan, container: torch.Tensor, header: bytes,
                     k_out: KVView, v_out: KVView, status: torch.Tensor, layer_begin: int = 0,
                     layer_end: int | None = None, stream=None, workspace=None):
    """kvtc_decompress_async: no host synchronisation; the integrity verdict
    (0 or KVTC_E_CORRUPT) lands in status (device int32 [1]) on the stream."""
    layer_end = k_out.shape[0] if layer_end is None else layer_end
    if workspace is None:
        workspace = torch.empty(decompress_workspace_bytes(kb, kp, vb, vp, header), dtype=torch.uint8, device="cuda")
    assert status.dtype == torch.int32 and status.is_cuda
    check(lib().kvtc_decompress_async(kb.h, kp.h, vb.h, vp.h, _ptr(container), container.numel(),
                                      C.c_char_p(header), layer_begin, layer_end, C.byref(k_out.c), C.byref(v_out.c),
                                      _ptr(status), _ptr(workspace), workspace.numel(), _stream(stream)))


# ------------------------------------------------- layer-streamed decompression
class StreamedDecompress:
    """kvtc_decompress_begin once, then kvtc_decompress_layers per layer range
    (P:L210): inflate + dequantise once, each range runs only its V^T columns."""

    def __init__(self, kb: Basis, kp: Plan, vb: Basis, vp: Plan, container: torch.Tensor, stream=None):
        self.args = (kb, kp, vb, vp)
        self.container = container
        self.header = container[: L.HEADER_BYTES].cpu().numpy().tobytes()
        self.workspace = torch.empty(decompress_workspace_bytes(kb, kp, vb, vp, self.header), dtype=torch.uint8,
                                     device="cuda")
        self.begin(stream)

    def begin(self, stream=None):
        """(Re-)runs kvtc_decompress_begin: inflate + dequantise into the workspace."""
        kb, kp, vb, vp = self.args
        check(lib().kvtc_decompress_begin(kb.h, kp.h, vb.h, vp.h, _ptr(self.container), self.container.numel(),
                                          _ptr(self.workspace), self.workspace.numel(), _stream(stream)))

    def layers(self, k_out: KVView, v_out: KVView, layer_begin: int, layer_end: int, stream=None):
        kb, kp, vb, vp = self.args
        check(lib().kvtc_decompress_layers(kb.h, kp.h, vb.h, vp.h, _ptr(self.container), C.c_char_p(self.header),
                                           layer_begin, layer_end, C.byref(k_out.c), C.byref(v_out.c),
                                           _ptr(self.workspace), self.workspace.numel(), _stream(stream)))


# ------------------------------------------------------------ batched codec
def compress_batch(kb: Basis, kp: Plan, vb: Basis, vp: Plan, ks: list, vs: list, sinks: int = 4, window: int = 128,
                   chunk_bytes: int = 65536, stream=None, outs: list | None = None, workspace=None,
                   sync_len: bool = True):
    """kvtc_compress_batch: one container per (ks[i], vs[i]); returns the list of
    containers (trimmed to their lengths when sync_len)."""
    n = len(ks)
    pol = L.Policy(sinks, window, chunk_bytes, 0)
    karr, varr = _views(ks), _views(vs)
    if outs is None:
        outs = [torch.empty(int(lib().kvtc_compress_bound(kp.h, vp.h, C.byref(k.c), C.byref(pol))),
                            dtype=torch.uint8, device="cuda") for k in ks]
    if workspace is None:
        wsb = int(lib().kvtc_compress_batch_workspace_bytes(kb.h, kp.h, vb.h, vp.h, karr, n, C.byref(pol)))
        workspace = torch.empty(wsb, dtype=torch.uint8, device="cuda")
    ptrs = (C.c_void_p * n)(*[o.data_ptr() for o in outs])
    caps = (C.c_size_t * n)(*[o.numel() for o in outs])
    lens = (C.c_size_t * n)()
    check(lib().kvtc_compress_batch(kb.h, kp.h, vb.h, vp.h, karr, varr, n, C.byref(pol), ptrs, caps,
                                    lens if sync_len else None, _ptr(workspace), workspace.numel(), _stream(stream)))
    return [o[: lens[i]] for i, o in enumerate(outs)] if sync_len else outs


def compress_batch_workspace_bytes(kb, kp, vb, vp, ks: list, sinks=4, window=128, chunk_bytes=65536) -> int:
    pol = L.Policy(sinks, window, chunk_bytes, 0)
    return int(lib().kvtc_compress_batch_workspace_bytes(kb.h, kp.h, vb.h, vp.h, _views(ks), len(ks), C.byref(pol)))


def decompress_batch(kb: Basis, kp: Plan, vb: Basis, vp: Plan, containers: list, k_outs: list, v_outs: list,
                     stream=None, workspace=None, headers: list | None = None):
    """kvtc_decompress_batch: every container into its (k_outs[i], v_outs[i])."""
    n = len(containers)
    if workspace is None:
        if headers is None:
            headers = [c[: L.HEADER_BYTES].cpu().numpy().tobytes() for c in containers]
        hb = [C.create_string_buffer(h, len(h)) for h in headers]
        hp = (C.c_void_p * n)(*[C.cast(b, C.c_void_p) for b in hb])
        wsb = int(lib().kvtc_decompress_batch_workspace_bytes(kb.h, kp.h, vb.h, vp.h, hp, n))
        workspace = torch.empty(wsb, dtype=torch.uint8, device="cuda")
    ptrs = (C.c_void_p * n)(*[c.data_ptr() for c in containers])
    lens = (C.c_size_t * n)(*[c.numel() for c in containers])
    check(lib().kvtc_decompress_batch(kb.h, kp.h, vb.h, vp.h, ptrs, lens, n, _views(k_outs), _views(v_outs),
                                      _ptr(workspace), workspace.numel(), _stream(stream)))


def decompress_batch_async(kb: Basis, kp: Plan, vb: Basis, vp: Plan, containers: list, headers: list, k_outs: list,
                           v_outs: list, status: torch.Tensor, stream=None, workspace=None):
    """kvtc_decompress_batch_async: no host synchronisation; headers[i] = host
    copies of the containers' first 256 bytes; status (device int32 [n]) gets each
    item's verdict (0 or KVTC_E_CORRUPT)."""
    n = len(containers)
    hb = [C.create_string_buffer(h, len(h)) for h in headers]
    hp = (C.c_void_p * n)(*[C.cast(b, C.c_void_p) for b in hb])
    if workspace is None:
        wsb = int(lib().kvtc_decompress_batch_workspace_bytes(kb.h, kp.h, vb.h, vp.h, hp, n))
        workspace = torch.empty(wsb, dtype=torch.uint8, device="cuda")
    assert status.dtype == torch.int32 and status.is_cuda and status.numel() >= n
    ptrs = (C.c_void_p * n)(*[c.data_ptr() for c in containers])
    lens = (C.c_size_t * n)(*[c.numel() for c in containers])
    check(lib().kvtc_decompress_batch_async(kb.h, kp.h, vb.h, vp.h, ptrs, lens, hp, n, _views(k_outs), _views(v_outs),
                                            _ptr(status), _ptr(workspace), workspace.numel(), _stream(stream)))


def decompress_batch_workspace_bytes(kb, kp, vb, vp, headers: list) -> int:
    hb = [C.create_string_buffer(h, len(h)) for h in headers]
    hp = (C.c_void_p * len(headers))(*[C.cast(b, C.c_void_p) for b in hb])
    return int(lib().kvtc_decompress_batch_workspace_bytes(kb.h, kp.h, vb.h, vp.h, hp, len(headers)))


# ------------------------------------------------------------- calibration
def _samples(samples):
    s = np.ascontiguousarray(np.asarray(samples, dtype=np.int64).reshape(-1, 2))
    return s, s.ctypes.data_as(C.POINTER(C.c_int64))


def _views(views):
    arr = (L.View * len(views))(*[v.c for v in views])
    return arr


def calibrate(views: list, samples, which: int, rank_cap: int = 10000, inv_freq=None, pairing: int = 0,
              stream=None) -> Basis:
    """kvtc_calibrate: single-process accumulate + finalize."""
    s, sp = _samples(samples)
    arr = _views(views)
    rope, keep = _rope(inv_freq, pairing) if which == L.KEYS else (None, None)
    out = C.c_void_p()
    check(lib().kvtc_calibrate(arr, len(views), sp, len(s), which, C.byref(rope) if rope else None, rank_cap,
                               _stream(stream), C.byref(out)))
    return Basis(out, views[0].shape, which)


def calibrate_accumulate(views: list, samples, which: int, sum_x: torch.Tensor, xtx: torch.Tensor, inv_freq=None,
                         pairing: int = 0, stream=None, workspace: torch.Tensor | None = None):
    """Adds this process's sum_x (fp64 [p]) and X^T X (fp32 [p, p]) — the
    quantities a multi-GPU caller all-reduces before calibrate_finalize."""
    s, sp = _samples(samples)
    arr = _views(views)
    rope, keep = _rope(inv_freq, pairing) if which == L.KEYS else (None, None)
    shp = L.Shape(*views[0].shape)
    wsb = int(lib().kvtc_calibrate_workspace_bytes(C.byref(shp)))
    if workspace is None or workspace.numel() < wsb:
        workspace = torch.empty(wsb, dtype=torch.uint8, device="cuda")
    check(lib().kvtc_calibrate_accumulate(arr, len(views), sp, len(s), which, C.byref(rope) if rope else None,
                                          _ptr(sum_x), _ptr(xtx), _ptr(workspace), workspace.numel(),
                                          _stream(stream)))
    return workspace


def calibrate_finalize(shape, which: int, sum_x: torch.Tensor, xtx: torch.Tensor, n: int, rank_cap: int = 10000,
                       inv_freq=None, pairing: int = 0, stream=None) -> Basis:
    rope, keep = _rope(inv_freq, pairing) if which == L.KEYS else (None, None)
    out = C.c_void_p()
    check(lib().kvtc_calibrate_finalize(C.byref(L.Shape(*shape)), which, C.byref(rope) if rope else None,
                                        _ptr(sum_x), _ptr(xtx), n, rank_cap, _stream(stream), C.byref(out)))
    return Basis(out, tuple(shape), which)


# -------------------------------------------------------------- allocation
def dp_config(target_cr: float, sizes=(1, 16, 64, 256, 1024), type_mask: int = 0xF, dp_row_cap: int = 32768,
              feature_bits: int = 16):
    sz = np.ascontiguousarray(np.asarray(sizes, dtype=np.int32))
    cfg = L.DPConfig(float(target_cr), feature_bits, len(sz), _i32p(sz), type_mask, dp_row_cap)
    return cfg, sz


def allocate_bits_from_coeffs(P: torch.Tensor, p_original: int, target_cr: float, sizes=(1, 16, 64, 256, 1024),
                              type_mask: int = 0xF, dp_row_cap: int = 32768, stream=None) -> Plan:
    cfg, keep = dp_config(target_cr, sizes, type_mask, dp_row_cap)
    out = C.c_void_p()
    check(lib().kvtc_allocate_bits_from_coeffs(_ptr(P), P.shape[0], P.shape[1], p_original, C.byref(cfg),
                                               _stream(stream), C.byref(out)))
    return Plan(out)


def allocate_bits(basis: Basis, views: list, samples, target_cr: float, sizes=(1, 16, 64, 256, 1024),
                  type_mask: int = 0xF, dp_row_cap: int = 32768, stream=None) -> Plan:
    cfg, keep = dp_config(target_cr, sizes, type_mask, dp_row_cap)
    s, sp = _samples(samples)
    arr = _views(views)
    out = C.c_void_p()
    check(lib().kvtc_allocate_bits(basis.h, arr, len(views), sp, len(s), C.byref(cfg), _stream(stream),
                                   C.byref(out)))
    return Plan(out)


def allocate_bits_multi(basis: Basis, views: list, samples, target_crs, sizes=(1, 16, 64, 256, 1024),
                        type_mask: int = 0xF, dp_row_cap: int = 32768, stream=None) -> list:
    """kvtc_allocate_bits_multi: one plan per target CR from one DP table."""
    cfg, keep = dp_config(max(target_crs), sizes, type_mask, dp_row_cap)
    s, sp = _samples(samples)
    arr = _views(views)
    crs = (C.c_double * len(target_crs))(*target_crs)
    outs = (C.c_void_p * len(target_crs))()
    check(lib().kvtc_allocate_bits_multi(basis.h, arr, len(views), sp, len(s), C.byref(cfg), crs, len(target_crs),
                                         _stream(stream), outs))
    return [Plan(C.c_void_p(o)) for o in outs]


def allocate_bits_from_coeffs_multi(P: torch.Tensor, p_original: int, target_crs, sizes=(1, 16, 64, 256, 1024),
                                    type_mask: int = 0xF, dp_row_cap: int = 32768, stream=None) -> list:
    cfg, keep = dp_config(max(target_crs), sizes, type_mask, dp_row_cap)
    crs = (C.c_double * len(target_crs))(*target_crs)
    outs = (C.c_void_p * len(target_crs))()
    check(lib().kvtc_allocate_bits_from_coeffs_multi(_ptr(P), P.shape[0], P.shape[1], p_original, C.byref(cfg), crs,
                                                     len(target_crs), _stream(stream), outs))
    return [Plan(C.c_void_p(o)) for o in outs]


def dp_best_table(P: torch.Tensor, budget: int, sizes=(1, 16, 64, 256, 1024), type_mask: int = 0xF, stream=None):
    cfg, keep = dp_config(1.0, sizes, type_mask, P.shape[0])
    r = P.shape[1]
    out = torch.empty(r + 1, budget // 2 + 1, dtype=torch.float64, device="cuda")
    check(lib().kvtc_dp_best_table(_ptr(P), P.shape[0], r, budget, C.byref(cfg), _ptr(out), _stream(stream)))
    return out


# ------------------------------------------------------------ diagnostics
def profile_enable(on: bool = True):
    lib().kvtc_profile_enable(int(on))


def profile_read() -> dict:
    """{stage: (total_ms, calls)} of the stages recorded since profile_enable."""
    names = C.create_string_buffer(8192)
    ms = (C.c_double * 64)()
    calls = (C.c_int32 * 64)()
    n = lib().kvtc_profile_read(names, 8192, ms, calls, 64)
    keys = names.raw.split(b"\0")[:n]
    return {keys[i].decode(): (ms[i], calls[i]) for i in range(n)}


def launch_count() -> int:
    return int(lib().kvtc_launch_count())


def launch_count_reset():
    lib().kvtc_launch_count_reset()
