"""Batched codec (kvtc_compress_batch / kvtc_decompress_batch): several
conversations in one call must give byte-identical containers and bitwise
identical reconstructions to the single-conversation calls (rows are
independent under Q1, and the batched GEMMs run the same k-loop per tile), for
ragged lengths, a passthrough item (t <= s + w), paged outputs, and the
incremental compression of 16-token ranges that leave the window."""
import numpy as np
import pytest
import torch

from tests import gpu_env as E

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def K():
    from paper_2511_01815_b200 import kvtc
    kvtc.device_check()
    return kvtc


@pytest.fixture(scope="module")
def art(K):
    spec, invf, kb, vb, Ck, Cv = E.setup("mid")
    shape = (spec.layers, spec.kv_heads, spec.head_dim)
    g = E.mid_plan_groups()
    KB = K.Basis.create(shape, 0, kb.mu, kb.V, kb.sigma, inv_freq=invf, pairing=0)
    VB = K.Basis.create(shape, 1, vb.mu, vb.V, vb.sigma)
    return spec, KB, VB, K.Plan.create(kb.r, g), K.Plan.create(vb.r, g)


@pytest.fixture(scope="module")
def oracle_art():
    from oracle import dp as ODP
    spec, invf, kb, vb, Ck, Cv = E.setup("mid")
    g = E.mid_plan_groups()
    return invf, kb, vb, ODP.Plan(r=kb.r, blocks=list(g)), ODP.Plan(r=vb.r, blocks=list(g))


def _caches(lengths, pos0s):
    out = []
    for i, (t, p0) in enumerate(zip(lengths, pos0s)):
        Kc, Vc = E.caches("mid", t, p0, conversation=20 + i)
        out.append((Kc.cuda(), Vc.cuda()))
    return out


def test_compress_batch_matches_single(K, art):
    spec, KB, VB, KP, VP = art
    lengths, pos0s = [700, 133, 1000, 260, 100], [0, 40, 300, 0, 7]      # ragged tails, one passthrough
    cc = _caches(lengths, pos0s)
    ks = [K.KVView(k, pos0=p) for (k, _), p in zip(cc, pos0s)]
    vs = [K.KVView(v, pos0=p) for (_, v), p in zip(cc, pos0s)]
    batch = K.compress_batch(KB, KP, VB, VP, ks, vs)
    for i in range(len(cc)):
        single, _ = K.compress(KB, KP, VB, VP, ks[i], vs[i])
        assert torch.equal(batch[i], single), i


def test_decompress_batch_matches_single(K, art):
    spec, KB, VB, KP, VP = art
    lengths, pos0s = [650, 400, 133, 999], [0, 11, 5, 2048]
    cc = _caches(lengths, pos0s)
    conts = [K.compress(KB, KP, VB, VP, K.KVView(k, pos0=p), K.KVView(v, pos0=p))[0] for (k, v), p in zip(cc, pos0s)]
    refs = []
    for c, (k, v), p in zip(conts, cc, pos0s):
        rk, rv = torch.zeros_like(k), torch.zeros_like(v)
        K.decompress(KB, KP, VB, VP, c, K.KVView(rk, pos0=p), K.KVView(rv, pos0=p))
        refs.append((rk, rv))
    # item 1 is restored into a paged cache
    page, t1 = 16, lengths[1]
    npg = (t1 + page - 1) // page
    bt = torch.randperm(npg + 2, generator=torch.Generator().manual_seed(3))[:npg].int().cuda()
    pk = torch.zeros(spec.layers, npg + 2, page, spec.kv_heads, spec.head_dim, dtype=torch.bfloat16, device="cuda")
    pv = torch.zeros_like(pk)
    outs = [(torch.zeros_like(k), torch.zeros_like(v)) for (k, v) in cc]
    kov = [K.KVView(o[0], pos0=p) for o, p in zip(outs, pos0s)]
    vov = [K.KVView(o[1], pos0=p) for o, p in zip(outs, pos0s)]
    kov[1] = K.KVView(pk, pos0=pos0s[1], tokens=t1, block_table=bt)
    vov[1] = K.KVView(pv, pos0=pos0s[1], tokens=t1, block_table=bt)
    K.decompress_batch(KB, KP, VB, VP, conts, kov, vov)
    torch.cuda.synchronize()
    for i, (rk, rv) in enumerate(refs):
        if i == 1:
            tok = torch.arange(t1, device="cuda")
            gk, gv = pk[:, bt[tok // page].long(), tok % page], pv[:, bt[tok // page].long(), tok % page]
        else:
            gk, gv = outs[i]
        assert torch.equal(gk, rk) and torch.equal(gv, rv), i


def test_incremental_ranges(K, art, oracle_art):
    """Turn-by-turn compression: every 16 tokens that leave the window
    are compressed as their own range (sinks = window = 0 inside the range),
    for several conversations at once; each range decompresses to exactly what
    a single call on the same range gives."""
    spec, KB, VB, KP, VP = art
    t = 1200
    cc = _caches([t, t, t], [0, 0, 0])
    ranges = [(4 + 16 * j, 4 + 16 * (j + 1)) for j in range(5)]          # 5 turns of c = 16 tokens
    ks, vs, meta = [], [], []
    for ci, (k, v) in enumerate(cc):
        for a, b in ranges:
            ks.append(K.KVView([k[l, a:b] for l in range(k.shape[0])], pos0=a))
            vs.append(K.KVView([v[l, a:b] for l in range(v.shape[0])], pos0=a))
            meta.append((ci, a, b))
    conts = K.compress_batch(KB, KP, VB, VP, ks, vs, sinks=0, window=0)
    for i, c in enumerate(conts[:4]):
        single, _ = K.compress(KB, KP, VB, VP, ks[i], vs[i], sinks=0, window=0)
        assert torch.equal(c, single), i
    outs = [(torch.zeros(spec.layers, b - a, spec.kv_heads, spec.head_dim, dtype=torch.bfloat16, device="cuda"),
             torch.zeros(spec.layers, b - a, spec.kv_heads, spec.head_dim, dtype=torch.bfloat16, device="cuda"))
            for (_, a, b) in meta]
    K.decompress_batch(KB, KP, VB, VP, conts, [K.KVView(o[0], pos0=m[1]) for o, m in zip(outs, meta)],
                       [K.KVView(o[1], pos0=m[1]) for o, m in zip(outs, meta)])
    for i in (0, 7, 14):
        rk, rv = torch.zeros_like(outs[i][0]), torch.zeros_like(outs[i][1])
        K.decompress(KB, KP, VB, VP, conts[i], K.KVView(rk, pos0=meta[i][1]), K.KVView(rv, pos0=meta[i][1]))
        torch.cuda.synchronize()
        assert torch.equal(outs[i][0], rk) and torch.equal(outs[i][1], rv), i
        # and directly against the oracle: its decompression of the range's container
        # (s = w = 0: every token coded) and its own compression of the same 16 tokens
        invf, kb, vb, okp, ovp = oracle_art
        ci, a, b = meta[i]
        buf = conts[i].cpu().numpy().tobytes()
        rk_o, rv_o = E.oracle_restore(buf, kb, okp, vb, ovp, invf)
        E.assert_restored_like_oracle(outs[i][0], outs[i][1], rk_o, rv_o)
        from oracle import codec as OC
        from tests.kvtc_format import parse_container, parse_section
        import zlib
        Kr = cc[ci][0][:, a:b].double().cpu().numpy()
        Vr = cc[ci][1][:, a:b].double().cpu().numpy()
        oc = OC.compress(Kr, Vr, a, kb, okp, vb, ovp, invf, s=0, w=0)
        h = parse_container(buf)
        for sv, so, ob, X in ((0, oc.k, kb, OC.stream_rows(Kr, 0, 0, a, True, invf, 0)),
                              (1, oc.v, vb, OC.stream_rows(Vr, 0, 0, a, False))):
            sec = parse_section(buf[h["sec_k" if sv == 0 else "sec_v"]:])
            payload = b"".join(zlib.decompress(x, wbits=-15) for x in sec["streams"])
            cols = np.concatenate([np.arange(s0, s0 + z) for (s0, z, _) in okp.groups])
            E.assert_codes_parity(payload, okp.groups, so.D, b - a, X, ob, cols, f"range {i} stream={sv}")
