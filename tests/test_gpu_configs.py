"""BASELINE.json's other configs as GPU parity cases: the
Mistral-NeMo-12B shape (p = 40960, 64K tokens) at the CR sweep 10x / 20x / 40x
(DP targets 8 / 16 / 32), and one 8-GPU layer shard of the
Llama-3.3-70B shape (10 layers, p = 10240, 128K tokens, its own basis and plan,
P:L443).  Each: GPU calibration + DP, compress + decompress through the C ABI,
then sampled tokens checked against the oracle (codes, reconstruction), stock
zlib inflating every chunk, and the plan's budget.  Expected values come from
oracle/ only."""
import argparse
import zlib

import numpy as np
import pytest
import torch

from tests import gpu_env as E
from tests.kvtc_format import parse_container, parse_section

pytestmark = pytest.mark.gpu

from oracle import layout as OL
from oracle import numerics as ON
from oracle import pca as OPCA
from oracle import quant as OQ
from oracle import rope as OR


@pytest.fixture(scope="module")
def K():
    from paper_2511_01815_b200 import kvtc
    kvtc.device_check()
    return kvtc


def _bases(K, spec):
    """GPU calibration on two 32K-token calibration conversations (as bench.py)."""
    from kvtc_inputs import generate, sample_positions
    from paper_2511_01815_b200.distributed import calibrate_distributed
    invf = spec.inv_freq().numpy().astype(np.float32)
    lens = [32768, 32768]
    samples = sample_positions(lens, 65000, sinks=4, seed=7)
    out = []
    for stream in (0, 1):
        caches = [generate(spec, stream, L, pos0=0, conversation=1000 + i, device="cuda") for i, L in enumerate(lens)]
        views = [K.KVView(c) for c in caches]
        B = calibrate_distributed(K, views, samples, stream, 10000, inv_freq=invf)
        out.append((B, views, caches))
    return out, samples


def _check(K, spec, KB, VB, KP, VP, t, pos0, label):
    from kvtc_inputs import generate
    Kc = generate(spec, 0, t, pos0=pos0, conversation=3, device="cuda")
    Vc = generate(spec, 1, t, pos0=pos0, conversation=3, device="cuda")
    cont, _ = K.compress(KB, KP, VB, VP, K.KVView(Kc, pos0=pos0), K.KVView(Vc, pos0=pos0))
    ko, vo = torch.zeros_like(Kc), torch.zeros_like(Vc)
    K.decompress(KB, KP, VB, VP, cont, K.KVView(ko, pos0=pos0), K.KVView(vo, pos0=pos0))
    torch.cuda.synchronize()
    buf = cont.cpu().numpy().tobytes()
    h = parse_container(buf)
    m = t - 132
    assert h["m"] == m
    rng = np.random.default_rng(1)
    taus = np.unique(np.concatenate([[0, 127, 128, m - 1], rng.integers(0, m, 24)]))
    invf = spec.inv_freq().double().numpy()
    p = spec.layers * spec.kv_heads * spec.head_dim
    comp = 0
    for sv, B, P, cache, out in ((0, KB, KP, Kc, ko), (1, VB, VP, Vc, vo)):
        pi = P.info()
        groups = [tuple(g) for g in pi.groups]
        mu, V, sg = B.get()
        ob = OPCA.Basis(mu=mu.astype(np.float64), V=V[:, :pi.r_eff].astype(np.float64), sigma=sg[:pi.r_eff], n=0)
        sec = parse_section(buf[h["sec_k" if sv == 0 else "sec_v"]:])
        payload = b"".join(zlib.decompress(s, wbits=-15) for s in sec["streams"])   # stock zlib, every chunk
        assert len(payload) == OL.payload_bytes(groups, m)
        comp += sec["total"]
        full = OL.tile_bytes(groups, 128)
        rows = cache[:, 4 + taus].float().cpu().numpy().astype(np.float64)
        if sv == 0:
            rows = OR.unrope_r1(rows, pos0 + 4 + taus, invf, 0)
        X = OPCA.flatten_rows(rows)
        cols = np.concatenate([np.arange(s0, s0 + z) for (s0, z, _) in groups])
        D = OPCA.project(ob, X, cols)
        shs, scs, cds = [[] for _ in groups], [[] for _ in groups], [[] for _ in groups]
        for tau in taus:
            k = tau // 128
            ntok = min(128, m - k * 128)
            sh, sc, cd = OL.unpack(groups, payload[k * full: k * full + OL.tile_bytes(groups, ntok)], ntok)
            for g in range(len(groups)):
                shs[g].append(sh[g][tau - k * 128])
                scs[g].append(sc[g][tau - k * 128])
                cds[g].append(cd[g][tau - k * 128])
        gpu_payload = OL.pack(groups, [np.array(a) for a in shs], [np.array(a) for a in scs],
                              [np.array(a) for a in cds], len(taus))
        E.assert_codes_parity(gpu_payload, groups, D, len(taus), X, ob, cols, f"{label} stream={sv}")
        Dh = np.zeros((len(taus), ob.r))
        for g, (s0, z, ty) in enumerate(groups):
            Dh[:, s0:s0 + z] = ON.f16(OQ.dequantize_rows(np.array(shs[g]), np.array(scs[g]), np.array(cds[g]), ty))
        Xh = (Dh @ ob.Vd.T + ob.mu[None, :]).reshape(len(taus), spec.layers, spec.kv_heads, spec.head_dim)
        Xh = Xh.transpose(1, 0, 2, 3)
        ref = OR.rope_apply_r7(Xh, pos0 + 4 + taus, invf, 0) if sv == 0 else ON.bf16(Xh)
        got = out[:, 4 + taus].float().cpu().numpy().astype(np.float64)
        rel = np.linalg.norm(got - ref) / np.linalg.norm(ref)
        assert rel < 1e-3, (label, sv, rel)
        assert torch.equal(out[:, :4], cache[:, :4]) and torch.equal(out[:, t - 128:], cache[:, t - 128:])
        # the plan spends at most B = floor(16 p / CR) bits per token (Q6)
        assert pi.bits_per_token <= pi.budget
    return 2 * 2 * p * m / comp


SWEEP = [8.0, 16.0, 32.0]


@pytest.fixture(scope="module")
def nemo(K):
    """One calibration, and ONE DP table per stream for the whole CR sweep
    (kvtc_allocate_bits_multi), checked against a separate DP run at CR 16."""
    from kvtc_inputs import make_spec
    spec = make_spec("nemo12b")
    (kb, vb), samples = _bases(K, spec)
    (KB, kviews, _), (VB, vviews, _) = kb, vb
    kplans = K.allocate_bits_multi(KB, kviews, samples, SWEEP)
    vplans = K.allocate_bits_multi(VB, vviews, samples, SWEEP)
    single = K.allocate_bits(KB, kviews, samples, 16.0)
    assert single.info().groups == kplans[1].info().groups
    assert single.info().expected_error == kplans[1].info().expected_error
    return spec, kb, vb, samples, dict(zip(SWEEP, zip(kplans, vplans)))


@pytest.mark.parametrize("cr_target", SWEEP)
def test_nemo12b_cr_sweep(K, nemo, cr_target):
    spec, (KB, kviews, _), (VB, vviews, _), samples, plans = nemo
    KP, VP = plans[cr_target]
    p = spec.layers * spec.kv_heads * spec.head_dim
    assert KP.info().budget == int(16 * p // cr_target)
    cr = _check(K, spec, KB, VB, KP, VP, 65536, 0, f"nemo12b cr{cr_target:g}")
    print(f"\n[nemo12b] DP target {cr_target:g}x -> CR after DEFLATE {cr:.2f}x")
    assert cr >= cr_target                      # DEFLATE only adds compression on top of the plan


def test_llama70b_layer_shard(K):
    from kvtc_inputs import make_spec
    spec = make_spec("llama70b_shard")
    assert spec.layers * spec.kv_heads * spec.head_dim == 10240
    (kb, vb), samples = _bases(K, spec)
    KB, kviews, _ = kb
    VB, vviews, _ = vb
    KP = K.allocate_bits(KB, kviews, samples, 16.0)
    VP = K.allocate_bits(VB, vviews, samples, 16.0)
    cr = _check(K, spec, KB, VB, KP, VP, 131072, 4096, "llama70b shard")
    print(f"\n[llama70b shard] CR after DEFLATE {cr:.2f}x")
    assert cr >= 16.0
