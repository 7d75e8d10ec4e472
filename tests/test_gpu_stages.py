"""GPU parity of each kernel against the oracle on identical seeded inputs."""
import os
import subprocess
import sys
import zlib

import numpy as np
import pytest
import torch

from tests import gpu_env as E
from tests.kvtc_format import code_lengths, parse_section, segment_bit_lengths

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

pytestmark = pytest.mark.gpu

from oracle import layout as OL
from oracle import pca as OPCA
from oracle import quant as OQ
from oracle import rope as OR
from oracle import numerics as ON


@pytest.fixture(scope="module")
def K():
    from paper_2511_01815_b200 import kvtc
    kvtc.device_check()
    return kvtc


def _basis(K, b, shape, which, invf):
    return K.Basis.create(shape, which, b.mu, b.V, b.sigma, inv_freq=invf if which == 0 else None)


def _bf16_np(t):
    return t.float().cpu().numpy().astype(np.float64)


@pytest.mark.parametrize("name,tokens,pos0", [("toy", 512, 0), ("mid", 700, 1000)])
def test_gather_unrope_bitexact(K, name, tokens, pos0):
    spec, invf = E.setup(name)[:2]
    Kc, Vc = E.caches(name, tokens, pos0)
    view_k = K.KVView(Kc.cuda(), pos0=pos0)
    view_v = K.KVView(Vc.cuda(), pos0=pos0)
    s, m = 4, tokens - 132
    Xk = K.gather(view_k, s, m, True, invf.astype(np.float32), 0)
    Xv = K.gather(view_v, s, m, False)
    ref_k = OPCA.flatten_rows(OR.unrope_r1(Kc.double().numpy()[:, s:s + m], pos0 + s + np.arange(m), invf, 0))
    ref_v = OPCA.flatten_rows(Vc.double().numpy()[:, s:s + m])
    np.testing.assert_array_equal(_bf16_np(Xk), ref_k)
    np.testing.assert_array_equal(_bf16_np(Xv), ref_v)


def test_gather_paged_layout(K):
    name, tokens, pos0 = "mid", 700, 7
    spec, invf = E.setup(name)[:2]
    Kc, _ = E.caches(name, tokens, pos0)
    page = 16
    npages = (tokens + page - 1) // page
    perm = torch.randperm(npages + 5, generator=torch.Generator().manual_seed(0))[:npages].int()
    pages = torch.zeros(spec.layers, npages + 5, page, spec.kv_heads, spec.head_dim, dtype=torch.bfloat16)
    for t in range(tokens):
        pages[:, perm[t // page], t % page] = Kc[:, t]
    view = K.KVView(pages.cuda(), pos0=pos0, tokens=tokens, block_table=perm.cuda())
    X = K.gather(view, 4, tokens - 132, True, invf.astype(np.float32), 0)
    ref = K.gather(K.KVView(Kc.cuda(), pos0=pos0), 4, tokens - 132, True, invf.astype(np.float32), 0)
    assert torch.equal(X, ref)


def _plan_for(name):
    if name == "toy":
        kp, vp = E.toy_plans(16)
        return kp.groups, vp.groups
    if name == "mid-runs":
        g = E.runs_plan_groups()
        return g, g
    if name == "mid-typed-runs":
        g = E.same_type_runs_plan_groups()
        return g, g
    g = E.mid_plan_groups()
    return g, g


@pytest.mark.parametrize("name,tokens", [("toy", 512), ("mid", 1000)])
def test_project_fp32(K, name, tokens):
    spec, invf, kb, vb, Ck, Cv = E.setup(name)
    Kc, Vc = E.caches(name, tokens, 0)
    m = tokens - 132
    B = _basis(K, vb, (spec.layers, spec.kv_heads, spec.head_dim), 1, invf)
    X = K.gather(K.KVView(Vc.cuda()), 4, m, False)
    D = K.project(B, None, X, vb.r).cpu().numpy().astype(np.float64)
    ref = OPCA.project(vb, _bf16_np(X))
    scale = np.abs(ref).max()
    err = np.abs(D - ref).max() / scale
    assert err < 2e-5, err


@pytest.mark.parametrize("name,tokens", [("toy", 512), ("mid", 1000), ("mid", 132 + 128 * 3), ("mid-runs", 777)])
def test_quantize_pack_and_fused(K, name, tokens):
    gk, gv = _plan_for(name)
    name = "mid" if name == "mid-runs" else name
    spec, invf, kb, vb, Ck, Cv = E.setup(name)
    Kc, Vc = E.caches(name, tokens, 0)
    m = tokens - 132
    shape = (spec.layers, spec.kv_heads, spec.head_dim)
    for which, ob, groups, cache in ((0, kb, gk, Kc), (1, vb, gv, Vc)):
        B = _basis(K, ob, shape, which, invf)
        Pl = K.Plan.create(ob.r, groups)
        X = K.gather(K.KVView(cache.cuda()), 4, m, which == 0, invf.astype(np.float32), 0)
        ncols = sum(z for (_, z, _) in groups)
        D = K.project(B, Pl, X, ncols)
        simt = K.quantize_pack(Pl, D)
        fused = K.project_quantize(B, Pl, X)
        assert simt.numel() == OL.payload_bytes(groups, m)
        # fused tcgen05 epilogue == SIMT reference on the same fp32 accumulator
        assert torch.equal(simt, fused)
        pb = fused.cpu().numpy().tobytes()
        # layout parity: oracle unpack -> repack reproduces the GPU bytes exactly
        sh, sc, cd = OL.unpack(groups, pb, m)
        assert OL.pack(groups, sh, sc, cd, m) == pb
        # code parity against the oracle's fp64 projection
        cols = np.concatenate([np.arange(s0, s0 + z) for (s0, z, _) in groups])
        D_ref = OPCA.project(ob, _bf16_np(X), cols)
        E.assert_codes_parity(pb, groups, D_ref, m, _bf16_np(X), ob, cols, f"{name} stream={which}")


def test_deflate_roundtrip_zlib(K):
    rng = np.random.default_rng(0)
    cases = [
        rng.integers(0, 4, 200000, dtype=np.uint8),                     # low entropy
        rng.integers(0, 256, 70000, dtype=np.uint8),                    # incompressible -> stored
        np.zeros(65536 * 2 + 17, dtype=np.uint8),                       # single symbol
        (rng.geometric(0.05, 300001) % 256).astype(np.uint8),           # skewed: long codes
        np.array([7], dtype=np.uint8),
    ]
    for ci, data in enumerate(cases):
        t = torch.from_numpy(data).cuda()
        sec = K.deflate(t)
        info = parse_section(sec.cpu().numpy().tobytes())
        if ci == 3:   # skewed: codes past the inflater's 11-bit first level (its subtable path)
            assert max(max(code_lengths(s)) for s, e in zip(info["streams"], info["table"]) if e["kind"] == 0) > 11
        assert info["raw"] == len(data)
        # every chunk is an independent raw DEFLATE stream stock zlib inflates
        got = b"".join(zlib.decompress(s, wbits=-15) for s in info["streams"])
        assert got == data.tobytes()
        # the side index: bit length of each 1/64 of a chunk, checked by decoding
        # the first chunks symbol by symbol (Q19)
        assert info["nseg"] == 64 and info["seg"] * 64 == info["chunk"]
        for c in range(min(2, info["nchunks"])):
            if info["table"][c]["kind"] != 0:
                assert not info["index"][c].any()
                continue
            assert max(code_lengths(info["streams"][c])) <= 15          # RFC 1951 limit
            nb = min(info["chunk"], len(data) - c * info["chunk"])
            lens, dec, end = segment_bit_lengths(info["streams"][c], nb, info["seg"], 64)
            assert dec == data.tobytes()[c * info["chunk"]: c * info["chunk"] + nb]
            assert list(info["index"][c]) == lens
            assert (end + 7) // 8 == info["table"][c]["bytes"]
        # and the GPU inflates its own section
        back = K.inflate(sec, len(data))
        assert torch.equal(back.cpu(), t.cpu())


_RFC_LIMIT_SCRIPT = r"""
import sys, zlib, numpy as np, torch
sys.path.insert(0, sys.argv[1])
sys.path.insert(0, sys.argv[1] + "/tests")
from paper_2511_01815_b200 import kvtc as K
from kvtc_format import parse_section, code_lengths
rng = np.random.default_rng(3)
data = (rng.geometric(0.05, 300001) % 256).astype(np.uint8)
t = torch.from_numpy(data).cuda()
sec = K.deflate(t)
info = parse_section(sec.cpu().numpy().tobytes())
assert b"".join(zlib.decompress(s, wbits=-15) for s in info["streams"]) == data.tobytes()
longest = max(max(code_lengths(s)) for s, e in zip(info["streams"], info["table"]) if e["kind"] == 0)
assert longest == 11, longest
assert torch.equal(K.inflate(sec, len(data)).cpu(), t.cpu())
print("ok", longest)
"""


def test_deflate_limit11_fast_inflate():
    """KVTC_DEFLATE_MAXBITS=11: skewed chunks (codes up to 15 bits under the
    default RFC limit, test above) get length-limited codes that zlib still
    inflates, and the inflater takes its subtable-free path."""
    env = dict(os.environ, KVTC_DEFLATE_MAXBITS="11")
    r = subprocess.run([sys.executable, "-c", _RFC_LIMIT_SCRIPT, ROOT], env=env, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0 and r.stdout.startswith("ok"), r.stdout + r.stderr


def test_gpu_inflates_zlib_streams(K):
    rng = np.random.default_rng(1)
    raw = [rng.integers(0, 5, 60000, dtype=np.uint8).tobytes(),
           (b"kv cache transform coding " * 3000)[:65536],                 # LZ77 back-references
           rng.integers(0, 256, 5000, dtype=np.uint8).tobytes(),
           b"", b"a"]
    streams, lens = [], []
    for lvl in (0, 1, 6, 9):
        for r in raw:
            c = zlib.compressobj(level=lvl, wbits=-15)
            streams.append(c.compress(r) + c.flush())
            lens.append(len(r))
    out, status = K.inflate_raw(streams, lens)
    assert int(status.abs().sum()) == 0, status
    assert out.cpu().numpy().tobytes() == b"".join(raw * 4)


@pytest.mark.parametrize("name,tokens", [("toy", 512), ("mid", 1000), ("mid-runs", 777), ("mid-typed-runs", 643)])
def test_dequant_and_reconstruct(K, name, tokens):
    gk, gv = _plan_for(name)
    name = "mid" if name.startswith("mid") else name
    spec, invf, kb, vb, Ck, Cv = E.setup(name)
    Kc, Vc = E.caches(name, tokens, 50)
    m = tokens - 132
    shape = (spec.layers, spec.kv_heads, spec.head_dim)
    for which, ob, groups, cache in ((0, kb, gk, Kc), (1, vb, gv, Vc)):
        B = _basis(K, ob, shape, which, invf)
        Pl = K.Plan.create(ob.r, groups)
        X = K.gather(K.KVView(cache.cuda(), pos0=50), 4, m, which == 0, invf.astype(np.float32), 0)
        payload = K.project_quantize(B, Pl, X)
        Dh = K.dequantize(Pl, payload, m)
        sh, sc, cd = OL.unpack(groups, payload.cpu().numpy().tobytes(), m)
        off = 0
        Dh_np = Dh.float().cpu().numpy().astype(np.float64)
        for g, (_, z, t) in enumerate(groups):
            ref = ON.f16(OQ.dequantize_rows(sh[g], sc[g], cd[g], t))
            got = Dh_np[:, off:off + z]
            # R5: D^ = fp16(x^) rounded once from the exact x^ (one fp16 fma on the GPU,
            # fp64 then fp16 in the oracle): bit-exact
            np.testing.assert_array_equal(got, ref, err_msg=f"group {g}")
            off += z
        out = torch.zeros_like(cache).cuda()
        view = K.KVView(out, pos0=50)
        K.reconstruct(B, Pl, Dh, m, 4, 0, spec.layers, view)
        # D2 fused into K5 (the product path): the GEMM dequantises its A operand from
        # the payload in shared memory; same D^, same MMA sequence -> bitwise equal
        out_f = torch.zeros_like(cache).cuda()
        K.reconstruct_payload(B, Pl, payload, m, 4, 0, spec.layers, K.KVView(out_f, pos0=50))
        torch.cuda.synchronize()
        assert torch.equal(out_f[:, 4:4 + m], out[:, 4:4 + m])
        assert int((out_f[:, :4] != 0).sum()) == 0 and int((out_f[:, 4 + m:] != 0).sum()) == 0
        # oracle from the same D^ (GPU dequant output)
        full = np.zeros((m, ob.r))
        off = 0
        for (s0, z, t) in groups:
            full[:, s0:s0 + z] = Dh_np[:, off:off + z]
            off += z
        Xh = (full @ ob.Vd.T + ob.mu[None, :]).reshape(m, spec.layers, spec.kv_heads, spec.head_dim)
        Xh = Xh.transpose(1, 0, 2, 3)
        ref = OR.rope_apply_r7(Xh, 50 + 4 + np.arange(m), invf, 0) if which == 0 else ON.bf16(Xh)
        got = _bf16_np(out[:, 4:4 + m])
        rel = np.linalg.norm(got - ref) / np.linalg.norm(ref)
        assert rel < 1e-3, rel
        assert (got != ref).mean() < 0.02
