"""End-to-end GPU compress / decompress through the C ABI vs the oracle."""
import zlib

import numpy as np
import pytest
import torch

from tests import gpu_env as E
from tests.kvtc_format import parse_container, parse_section

pytestmark = pytest.mark.gpu

from oracle import codec as OC
from oracle import dp as ODP
from oracle import layout as OL
from oracle import quant as OQ


@pytest.fixture(scope="module")
def K():
    from paper_2511_01815_b200 import kvtc
    kvtc.device_check()
    return kvtc


def _setup(K, name):
    spec, invf, kb, vb, Ck, Cv = E.setup(name)
    shape = (spec.layers, spec.kv_heads, spec.head_dim)
    if name == "toy":
        kp, vp = E.toy_plans(16)
        gk, gv = kp.groups, vp.groups
    else:
        gk = gv = E.mid_plan_groups()
    KB = K.Basis.create(shape, 0, kb.mu, kb.V, kb.sigma, inv_freq=invf, pairing=0)
    VB = K.Basis.create(shape, 1, vb.mu, vb.V, vb.sigma)
    KP = K.Plan.create(kb.r, gk)
    VP = K.Plan.create(vb.r, gv)
    okp = ODP.Plan(r=kb.r, blocks=list(gk))
    ovp = ODP.Plan(r=vb.r, blocks=list(gv))
    return spec, invf, kb, vb, KB, VB, KP, VP, okp, ovp


@pytest.mark.parametrize("name,tokens,pos0", [("toy", 512, 0), ("toy", 133, 0), ("mid", 1000, 300), ("mid", 260, 0)])
def test_compress_decompress_vs_oracle(K, name, tokens, pos0):
    spec, invf, kb, vb, KB, VB, KP, VP, okp, ovp = _setup(K, name)
    Kc, Vc = E.caches(name, tokens, pos0, conversation=5)
    kd, vd = Kc.cuda(), Vc.cuda()
    cont, st = K.compress(KB, KP, VB, VP, K.KVView(kd, pos0=pos0), K.KVView(vd, pos0=pos0))
    buf = cont.cpu().numpy().tobytes()
    h = parse_container(buf)
    m = tokens - 132
    assert h["m"] == m and h["total_bytes"] == len(buf)
    # oracle on the same inputs
    oc = OC.compress(Kc.double().numpy(), Vc.double().numpy(), pos0, kb, okp, vb, ovp, invf)
    for sv, so, groups, ob, cache in ((0, oc.k, okp.groups, kb, Kc), (1, oc.v, ovp.groups, vb, Vc)):
        sec = parse_section(buf[h["sec_k" if sv == 0 else "sec_v"]:])
        payload = b"".join(zlib.decompress(s, wbits=-15) for s in sec["streams"])   # stock zlib inflates GPU chunks
        assert len(payload) == len(so.payload)
        if m > 0:
            X = OC.stream_rows(cache.double().numpy(), 4, 128, pos0, sv == 0, invf, 0)
            cols = np.concatenate([np.arange(s0, s0 + z) for (s0, z, _) in groups])
            E.assert_codes_parity(payload, groups, so.D, m, X, ob, cols, f"e2e {name} stream={sv}")
    ko = torch.zeros_like(kd)
    vo = torch.zeros_like(vd)
    K.decompress(KB, KP, VB, VP, cont, K.KVView(ko, pos0=pos0), K.KVView(vo, pos0=pos0))
    torch.cuda.synchronize()
    K2, V2 = OC.decompress(oc, kb, okp, vb, ovp, invf)
    mid = slice(4, tokens - 128)
    for sv, got, ref, orig, ob, op, so in ((0, ko, K2, Kc, kb, okp, oc.k), (1, vo, V2, Vc, vb, ovp, oc.v)):
        g = got.float().cpu().numpy().astype(np.float64)
        o = orig.double().numpy()
        # sinks and window byte-identical
        np.testing.assert_array_equal(g[:, :4], o[:, :4])
        np.testing.assert_array_equal(g[:, tokens - 128:], o[:, tokens - 128:])
        if m == 0:
            continue
        # (a) decompress-path parity: the oracle decompressing the GPU's own payload
        sec = parse_section(buf[h["sec_k" if sv == 0 else "sec_v"]:])
        payload = b"".join(zlib.decompress(s, wbits=-15) for s in sec["streams"])
        Xh = OC.reconstruct_stream(payload, ob, op, m).reshape(m, spec.layers, spec.kv_heads, spec.head_dim)
        Xh = Xh.transpose(1, 0, 2, 3)
        from oracle import rope as OR, numerics as ON
        ref_a = OR.rope_apply_r7(Xh, pos0 + 4 + np.arange(m), invf, 0) if sv == 0 else ON.bf16(Xh)
        rel_a = np.linalg.norm(g[:, mid] - ref_a) / np.linalg.norm(ref_a)
        assert rel_a < 1e-3, rel_a
        # (b) end to end vs the oracle's own pipeline: within 1e-3 plus the effect
        # of the boundary code flips, whose X-space energy equals their D-space
        # energy (orthonormal invariance)
        sh_g, sc_g, cd_g = OL.unpack(op.groups, payload, m)
        dD = 0.0
        for gi, (_, z, t) in enumerate(op.groups):
            a = ON.f16(OQ.dequantize_rows(sh_g[gi], sc_g[gi], cd_g[gi], t))
            b = ON.f16(OQ.dequantize_rows(so.shifts[gi], so.scales[gi], so.codes[gi], t))
            dD += float(np.sum((a - b) ** 2))
        nref = np.linalg.norm(ref[:, mid])
        rel_b = np.linalg.norm(g[:, mid] - ref[:, mid]) / nref
        allow = 1e-3 + 1.02 * np.sqrt(dD) / nref
        print(f"\n[recon] {name} stream={sv} decompress-path rel={rel_a:.2e} e2e rel={rel_b:.2e} "
              f"code-flip part={np.sqrt(dD) / nref:.2e}")
        assert rel_b < allow, (rel_b, allow)


def test_layer_range_decompress(K):
    name, tokens = "mid", 700
    spec, invf, kb, vb, KB, VB, KP, VP, okp, ovp = _setup(K, name)
    Kc, Vc = E.caches(name, tokens, 0, conversation=6)
    kd, vd = Kc.cuda(), Vc.cuda()
    cont, _ = K.compress(KB, KP, VB, VP, K.KVView(kd), K.KVView(vd))
    full_k, full_v = torch.zeros_like(kd), torch.zeros_like(vd)
    K.decompress(KB, KP, VB, VP, cont, K.KVView(full_k), K.KVView(full_v))
    part_k, part_v = torch.zeros_like(kd), torch.zeros_like(vd)
    K.decompress(KB, KP, VB, VP, cont, K.KVView(part_k), K.KVView(part_v), layer_begin=1, layer_end=2)
    torch.cuda.synchronize()
    assert torch.equal(part_k[1], full_k[1]) and torch.equal(part_v[1], full_v[1])
    assert not part_k[0].any() and not part_v[0].any()
    # and directly against the oracle's decompression of the same container (layer 1 only)
    rk, rv = E.oracle_restore(cont.cpu().numpy().tobytes(), kb, okp, vb, ovp, invf)
    E.assert_restored_like_oracle(part_k, part_v, rk, rv, layers=slice(1, 2))
    assert torch.equal(part_k[1, :4], kd[1, :4]) and torch.equal(part_v[1, tokens - 128:], vd[1, tokens - 128:])


@pytest.mark.parametrize("name,tokens", [("mid", 700), ("toy", 400)])
def test_layer_streamed_decompress(K, name, tokens):
    """kvtc_decompress_begin once + kvtc_decompress_layers per layer
    == kvtc_decompress, bit for bit; layers not yet requested stay untouched."""
    spec, invf, kb, vb, KB, VB, KP, VP, okp, ovp = _setup(K, name)
    Kc, Vc = E.caches(name, tokens, 17, conversation=9)
    kd, vd = Kc.cuda(), Vc.cuda()
    cont, _ = K.compress(KB, KP, VB, VP, K.KVView(kd, pos0=17), K.KVView(vd, pos0=17))
    full_k, full_v = torch.zeros_like(kd), torch.zeros_like(vd)
    K.decompress(KB, KP, VB, VP, cont, K.KVView(full_k, pos0=17), K.KVView(full_v, pos0=17))
    sk, sv = torch.zeros_like(kd), torch.zeros_like(vd)
    sd = K.StreamedDecompress(KB, KP, VB, VP, cont)
    for l in range(spec.layers):
        sd.layers(K.KVView(sk, pos0=17), K.KVView(sv, pos0=17), l, l + 1)
        torch.cuda.synchronize()
        assert torch.equal(sk[: l + 1], full_k[: l + 1]) and torch.equal(sv[: l + 1], full_v[: l + 1])
        assert not sk[l + 1:].any() and not sv[l + 1:].any()


def test_empty_plan_reconstructs_the_mean(K):
    """A plan with no groups (every PC None): nothing is coded, the
    middle tokens decompress to the mean mu (re-rotated for keys, R7), exactly as
    the oracle's decompression of the same container; sinks / window raw."""
    name, tokens, pos0 = "mid", 500, 9
    spec, invf, kb, vb, KB, VB, KP, VP, okp, ovp = _setup(K, name)
    EP = K.Plan.create(kb.r, [])
    EPV = K.Plan.create(vb.r, [])
    Kc, Vc = E.caches(name, tokens, pos0, conversation=11)
    kd, vd = Kc.cuda(), Vc.cuda()
    cont, st = K.compress(KB, EP, VB, EPV, K.KVView(kd, pos0=pos0), K.KVView(vd, pos0=pos0))
    ko, vo = torch.zeros_like(kd), torch.zeros_like(vd)
    K.decompress(KB, EP, VB, EPV, cont, K.KVView(ko, pos0=pos0), K.KVView(vo, pos0=pos0))
    torch.cuda.synchronize()
    eok, eov = ODP.Plan(r=kb.r, blocks=[]), ODP.Plan(r=vb.r, blocks=[])
    oc = OC.compress(Kc.double().numpy(), Vc.double().numpy(), pos0, kb, eok, vb, eov, invf)
    K2, V2 = OC.decompress(oc, kb, eok, vb, eov, invf)
    for got, ref, orig in ((ko, K2, Kc), (vo, V2, Vc)):
        g = got.float().cpu().numpy().astype(np.float64)
        np.testing.assert_array_equal(g[:, :4], orig.double().numpy()[:, :4])
        np.testing.assert_array_equal(g[:, tokens - 128:], orig.double().numpy()[:, tokens - 128:])
        mid = slice(4, tokens - 128)
        rel = np.linalg.norm(g[:, mid] - ref[:, mid]) / np.linalg.norm(ref[:, mid])
        assert rel < 1e-3, rel


@pytest.mark.parametrize("tokens", [1, 100, 132])
def test_passthrough_short_conversation(K, tokens):
    """t <= s + w (Q17): KVTC_NOTHING_TO_COMPRESS, the container holds the raw
    tokens, and decompression restores them bit for bit."""
    spec, invf, kb, vb, KB, VB, KP, VP, okp, ovp = _setup(K, "mid")
    Kc, Vc = E.caches("mid", tokens, 0, conversation=12)
    kd, vd = Kc.cuda(), Vc.cuda()
    cont, st = K.compress(KB, KP, VB, VP, K.KVView(kd), K.KVView(vd))
    assert st == 1                                      # KVTC_NOTHING_TO_COMPRESS
    ko, vo = torch.zeros_like(kd), torch.zeros_like(vd)
    K.decompress(KB, KP, VB, VP, cont, K.KVView(ko), K.KVView(vo))
    torch.cuda.synchronize()
    assert torch.equal(ko, kd) and torch.equal(vo, vd)


def test_paged_output(K):
    name, tokens = "mid", 600
    spec, invf, kb, vb, KB, VB, KP, VP, okp, ovp = _setup(K, name)
    Kc, Vc = E.caches(name, tokens, 0, conversation=7)
    kd, vd = Kc.cuda(), Vc.cuda()
    cont, _ = K.compress(KB, KP, VB, VP, K.KVView(kd), K.KVView(vd))
    full_k, full_v = torch.zeros_like(kd), torch.zeros_like(vd)
    K.decompress(KB, KP, VB, VP, cont, K.KVView(full_k), K.KVView(full_v))
    page = 16
    npg = (tokens + page - 1) // page
    bt = torch.randperm(npg + 3, generator=torch.Generator().manual_seed(1))[:npg].int().cuda()
    pk = torch.zeros(spec.layers, npg + 3, page, spec.kv_heads, spec.head_dim, dtype=torch.bfloat16, device="cuda")
    pv = torch.zeros_like(pk)
    K.decompress(KB, KP, VB, VP, cont, K.KVView(pk, tokens=tokens, block_table=bt),
                 K.KVView(pv, tokens=tokens, block_table=bt))
    torch.cuda.synchronize()
    tok = torch.arange(tokens, device="cuda")
    gk = pk[:, bt[tok // page].long(), tok % page]
    gv = pv[:, bt[tok // page].long(), tok % page]
    assert torch.equal(gk, full_k) and torch.equal(gv, full_v)


def test_mismatched_plan_rejected(K):
    spec, invf, kb, vb, KB, VB, KP, VP, okp, ovp = _setup(K, "toy")
    Kc, Vc = E.caches("toy", 400, 0)
    cont, _ = K.compress(KB, KP, VB, VP, K.KVView(Kc.cuda()), K.KVView(Vc.cuda()))
    other = K.Plan.create(kb.r, [(0, 16, OQ.T_INT4)])
    with pytest.raises(Exception) as e:
        K.decompress(KB, other, VB, VP, cont, K.KVView(torch.zeros_like(Kc).cuda()), K.KVView(torch.zeros_like(Vc).cuda()))
    assert "MISMATCH" in str(e.value)


def test_direct_cache_read_matches_gather(K, monkeypatch):
    """The values' GEMM reads a contiguous cache in place through a 3-D tensor
    map; the container must be byte-identical to the gathered path's, for a
    tight cache, an over-allocated one (layer stride > tokens) and per-layer
    tensors at unrelated addresses (gather fallback)."""
    name, tokens = "mid", 900
    spec, invf, kb, vb, KB, VB, KP, VP, okp, ovp = _setup(K, name)
    Kc, Vc = E.caches(name, tokens, 0, conversation=8)
    kd, vd = Kc.cuda(), Vc.cuda()

    def run(vview):
        cont, _ = K.compress(KB, KP, VB, VP, K.KVView(kd), vview)
        torch.cuda.synchronize()
        return cont.cpu().numpy().tobytes()

    direct = run(K.KVView(vd))
    monkeypatch.setenv("KVTC_DIRECT_2D", "1")          # packed layers through a 2-D map
    direct2d = run(K.KVView(vd))
    monkeypatch.delenv("KVTC_DIRECT_2D")
    big = torch.zeros(spec.layers, tokens + 77, spec.kv_heads, spec.head_dim, dtype=torch.bfloat16, device="cuda")
    big[:, :tokens] = vd
    strided = run(K.KVView(big, tokens=tokens))
    separate = run(K.KVView([vd[i].clone() for i in range(spec.layers)]))
    monkeypatch.setenv("KVTC_NO_DIRECT", "1")
    gathered = run(K.KVView(vd))
    assert direct == gathered and direct2d == gathered and strided == gathered and separate == gathered


def test_separate_key_value_compression_ratios(K):
    """Separate K / V targets ("different compression
    ratios for keys and values"): keys at DP target 8, values at 32 on the toy
    config.  Each stream meets its own target before DEFLATE, the codes and the
    reconstruction match the oracle run with the same two plans."""
    spec, invf, kb, vb, Ck, Cv = E.setup("toy")
    shape = (spec.layers, spec.kv_heads, spec.head_dim)
    from oracle import pca as OPCA
    okp = ODP.allocate(OPCA.dp_coefficients(kb, Ck), 8.0, spec.p)[0]
    ovp = ODP.allocate(OPCA.dp_coefficients(vb, Cv), 32.0, spec.p)[0]
    assert okp.bits_per_token > 2 * ovp.bits_per_token
    KB = K.Basis.create(shape, 0, kb.mu, kb.V, kb.sigma, inv_freq=invf, pairing=0)
    VB = K.Basis.create(shape, 1, vb.mu, vb.V, vb.sigma)
    KP, VP = K.Plan.create(kb.r, okp.groups), K.Plan.create(vb.r, ovp.groups)
    tokens, pos0 = 512, 0
    Kc, Vc = E.caches("toy", tokens, pos0, conversation=31)
    kd, vd = Kc.cuda(), Vc.cuda()
    cont, _ = K.compress(KB, KP, VB, VP, K.KVView(kd), K.KVView(vd))
    info = K.container_info(cont)
    m = tokens - 132
    for sv, target in ((0, 8.0), (1, 32.0)):
        assert 2 * spec.p * m / info.payload_bytes[sv] >= target
    print(f"\n[per-stream CR] keys {2 * spec.p * m / info.entropy_bytes[0]:.1f}x, "
          f"values {2 * spec.p * m / info.entropy_bytes[1]:.1f}x after DEFLATE")
    buf = cont.cpu().numpy().tobytes()
    h = parse_container(buf)
    oc = OC.compress(Kc.double().numpy(), Vc.double().numpy(), pos0, kb, okp, vb, ovp, invf)
    for sv, so, groups, ob, cache in ((0, oc.k, okp.groups, kb, Kc), (1, oc.v, ovp.groups, vb, Vc)):
        sec = parse_section(buf[h["sec_k" if sv == 0 else "sec_v"]:])
        payload = b"".join(zlib.decompress(s, wbits=-15) for s in sec["streams"])
        X = OC.stream_rows(cache.double().numpy(), 4, 128, pos0, sv == 0, invf, 0)
        cols = np.concatenate([np.arange(s0, s0 + z) for (s0, z, _) in groups])
        E.assert_codes_parity(payload, groups, so.D, m, X, ob, cols, f"per-stream CR stream={sv}")
    ko, vo = torch.zeros_like(kd), torch.zeros_like(vd)
    K.decompress(KB, KP, VB, VP, cont, K.KVView(ko), K.KVView(vo))
    rk, rv = E.oracle_restore(buf, kb, okp, vb, ovp, invf)
    E.assert_restored_like_oracle(ko, vo, rk, rv)


@pytest.mark.parametrize("name,tokens", [("mid", 1000), ("toy", 400)])
def test_fused_dequant_decompress_matches(K, monkeypatch, name, tokens):
    """KVTC_DQ_FUSED=1 (the reconstruction GEMM's producer warps dequantise the
    payload straight into shared memory, D^ never in HBM; D2 fused into K5,
    P:L209) gives bit-identical caches to the default D^-through-TMA path, for the
    whole decompression, a layer range and the layer-streamed calls."""
    spec, invf, kb, vb, KB, VB, KP, VP, okp, ovp = _setup(K, name)
    Kc, Vc = E.caches(name, tokens, 5, conversation=11)
    kd, vd = Kc.cuda(), Vc.cuda()
    cont, _ = K.compress(KB, KP, VB, VP, K.KVView(kd, pos0=5), K.KVView(vd, pos0=5))

    def run(lb=0, le=None, streamed=False):
        ok, ov = torch.zeros_like(kd), torch.zeros_like(vd)
        le = spec.layers if le is None else le
        if streamed:
            sd = K.StreamedDecompress(KB, KP, VB, VP, cont)
            sd.layers(K.KVView(ok, pos0=5), K.KVView(ov, pos0=5), lb, le)
        else:
            K.decompress(KB, KP, VB, VP, cont, K.KVView(ok, pos0=5), K.KVView(ov, pos0=5), layer_begin=lb,
                         layer_end=le)
        torch.cuda.synchronize()
        return ok, ov

    ref = [run(), run(spec.layers - 1), run(0, 1, True)]
    monkeypatch.setenv("KVTC_DQ_FUSED", "1")
    got = [run(), run(spec.layers - 1), run(0, 1, True)]
    for (a, b), (c, d) in zip(ref, got):
        assert torch.equal(a, c) and torch.equal(b, d)


@pytest.mark.parametrize("name,tokens", [("mid", 1000), ("toy", 400), ("mid", 132)])
def test_rans_container_roundtrip(K, name, tokens):
    """coder = rANS (reading Q24): the same payloads behind another
    lossless back-end, so decompression is bit-identical to the DEFLATE
    container's; the payload checksums still verify every decoded byte."""
    spec, invf, kb, vb, KB, VB, KP, VP, okp, ovp = _setup(K, name)
    Kc, Vc = E.caches(name, tokens, 3, conversation=12)
    kd, vd = Kc.cuda(), Vc.cuda()
    cd, _ = K.compress(KB, KP, VB, VP, K.KVView(kd, pos0=3), K.KVView(vd, pos0=3))
    cr, _ = K.compress(KB, KP, VB, VP, K.KVView(kd, pos0=3), K.KVView(vd, pos0=3), coder=1)
    outs = []
    for c in (cd, cr):
        ok, ov = torch.zeros_like(kd), torch.zeros_like(vd)
        K.decompress(KB, KP, VB, VP, c, K.KVView(ok, pos0=3), K.KVView(ov, pos0=3))
        torch.cuda.synchronize()
        outs.append((ok, ov))
    assert torch.equal(outs[0][0], outs[1][0]) and torch.equal(outs[0][1], outs[1][1])
    ii, ir = K.container_info(cd), K.container_info(cr)
    assert ii.payload_bytes[0] == ir.payload_bytes[0] and ii.payload_bytes[1] == ir.payload_bytes[1]
    print(f"\n[rans] {name} t={tokens}: sections deflate={ii.entropy_bytes[0] + ii.entropy_bytes[1]} "
          f"rans={ir.entropy_bytes[0] + ir.entropy_bytes[1]} payload={ii.payload_bytes[0] + ii.payload_bytes[1]}")
    # a damaged rANS section is reported
    if tokens > 132:
        from tests.kvtc_format import parse_container
        hc = parse_container(cr.cpu().numpy().tobytes())
        assert hc["flags"] & 2                                    # the rANS flag
        bad = cr.clone()
        bad[int(hc["sec_k"]) + int(hc["ent_k"]) // 2] ^= 0x41
        ok, ov = torch.zeros_like(kd), torch.zeros_like(vd)
        from paper_2511_01815_b200 import _lib as L
        with pytest.raises(L.KvtcError) as e:
            K.decompress(KB, KP, VB, VP, bad, K.KVView(ok, pos0=3), K.KVView(ov, pos0=3))
        assert e.value.status == -3


@pytest.mark.parametrize("name,tokens", [("toy", 512), ("toy", 389), ("mid", 1000)])
def test_inflate_dequant_front_end_equals_split_path(K, name, tokens, monkeypatch):
    """KVTC_D_INFLATE_DQ=1 inflates and dequantises both streams in one launch
    (inflate_dequant_kernel, the measured alternative); the default runs the
    inflater and the dequantiser separately.  Both restore the cache bit for bit,
    also through the layer-streamed calls (kvtc_decompress_begin / _layers)."""
    spec, invf, kb, vb, KB, VB, KP, VP, okp, ovp = _setup(K, name)
    Kc, Vc = E.caches(name, tokens, 0, conversation=9)
    kd, vd = Kc.cuda(), Vc.cuda()
    cont, _ = K.compress(KB, KP, VB, VP, K.KVView(kd), K.KVView(vd))
    outs = {}
    for flag in ("1", "0"):
        monkeypatch.setenv("KVTC_D_INFLATE_DQ", flag)
        ko, vo = torch.zeros_like(kd), torch.zeros_like(vd)
        K.decompress(KB, KP, VB, VP, cont, K.KVView(ko), K.KVView(vo))
        lo, lv = torch.zeros_like(kd), torch.zeros_like(vd)
        ls = K.StreamedDecompress(KB, KP, VB, VP, cont)      # runs kvtc_decompress_begin
        ls.layers(K.KVView(lo), K.KVView(lv), 0, spec.layers)
        torch.cuda.synchronize()
        outs[flag] = (ko, vo, lo, lv)
    for a, b in zip(outs["1"], outs["0"]):
        assert torch.equal(a.view(torch.int16), b.view(torch.int16))
    assert torch.equal(outs["1"][0].view(torch.int16), outs["1"][2].view(torch.int16))


@pytest.mark.parametrize("name,tokens", [("toy", 512), ("mid", 1000)])
def test_overlapped_schedule_equals_serial(K, name, tokens, monkeypatch):
    """The integer codec kernels run on the library's side stream beside the GEMMs
    by default (KVTC_OVERLAP=1); KVTC_OVERLAP=0 runs everything on the caller's
    stream.  Same container bytes, same restored cache, either way."""
    spec, invf, kb, vb, KB, VB, KP, VP, okp, ovp = _setup(K, name)
    Kc, Vc = E.caches(name, tokens, 0, conversation=11)
    kd, vd = Kc.cuda(), Vc.cuda()
    res = {}
    for flag in ("0", "1"):
        monkeypatch.setenv("KVTC_OVERLAP", flag)
        cont, _ = K.compress(KB, KP, VB, VP, K.KVView(kd), K.KVView(vd))
        ko, vo = torch.zeros_like(kd), torch.zeros_like(vd)
        K.decompress(KB, KP, VB, VP, cont, K.KVView(ko), K.KVView(vo))
        torch.cuda.synchronize()
        res[flag] = (cont.cpu(), ko, vo)
    assert torch.equal(res["0"][0], res["1"][0])
    assert torch.equal(res["0"][1].view(torch.int16), res["1"][1].view(torch.int16))
    assert torch.equal(res["0"][2].view(torch.int16), res["1"][2].view(torch.int16))
