"""Parity at BASELINE.json's full size (Llama-3.1-8B shape, 32K tokens, CR 16) in
the launch configuration bench.py times, on sampled outputs the oracle computes
one by one, plus properties that hold at any size."""
import argparse
import zlib

import numpy as np
import pytest
import torch

from tests import gpu_env as E
from tests.kvtc_format import parse_container, parse_section

pytestmark = pytest.mark.gpu

from oracle import dp as ODP
from oracle import layout as OL
from oracle import numerics as ON
from oracle import pca as OPCA
from oracle import quant as OQ
from oracle import rope as OR


@pytest.fixture(scope="module")
def run():
    import bench
    from paper_2511_01815_b200 import kvtc as K
    from kvtc_inputs import make_spec, generate
    K.device_check()
    spec = make_spec("llama8b")
    ns = argparse.Namespace(cal_tokens=32768, cal_seqs=2, ncal=65000, rank_cap=10000, cr=16.0)
    (KB, VB), (KP, VP), info = bench.build_artifacts(K, spec, ns, 0, 1, None)
    t = 32768
    Kc = generate(spec, 0, t, conversation=0, device="cuda")
    Vc = generate(spec, 1, t, conversation=0, device="cuda")
    cont, _ = K.compress(KB, KP, VB, VP, K.KVView(Kc), K.KVView(Vc))
    ko, vo = torch.zeros_like(Kc), torch.zeros_like(Vc)
    K.decompress(KB, KP, VB, VP, cont, K.KVView(ko), K.KVView(vo))
    torch.cuda.synchronize()
    return dict(K=K, spec=spec, KB=KB, VB=VB, KP=KP, VP=VP, Kc=Kc, Vc=Vc, ko=ko, vo=vo,
                buf=cont.cpu().numpy().tobytes(), t=t)


def _oracle_basis(B, plan_info):
    mu, V, sg = B.get()
    r_use = plan_info.r_eff
    return OPCA.Basis(mu=mu.astype(np.float64), V=V[:, :r_use].astype(np.float64), sigma=sg[:r_use], n=0)


def test_fullscale_sampled_codes_and_reconstruction(run):
    spec, t, buf = run["spec"], run["t"], run["buf"]
    h = parse_container(buf)
    m = t - 132
    assert h["m"] == m
    rng = np.random.default_rng(0)
    # sampled middle tokens: first tile, last (partial) tile, random ones
    taus = np.unique(np.concatenate([[0, 1, 127, 128, m - 1, m - 2], rng.integers(0, m, 40)]))
    invf = spec.inv_freq().double().numpy()
    for sv, B, P, cache, out in ((0, run["KB"], run["KP"], run["Kc"], run["ko"]),
                                 (1, run["VB"], run["VP"], run["Vc"], run["vo"])):
        pi = P.info()
        groups = [tuple(g) for g in pi.groups]
        ob = _oracle_basis(B, pi)
        sec = parse_section(buf[h["sec_k" if sv == 0 else "sec_v"]:])
        payload = b"".join(zlib.decompress(s, wbits=-15) for s in sec["streams"])   # stock zlib, every chunk
        assert len(payload) == OL.payload_bytes(groups, m)
        full = OL.tile_bytes(groups, 128)
        rows = cache[:, 4 + taus].float().cpu().numpy().astype(np.float64)         # [l, n, h, d]
        if sv == 0:
            rows = OR.unrope_r1(rows, 4 + taus, invf, 0)
        X = OPCA.flatten_rows(rows)
        cols = np.concatenate([np.arange(s0, s0 + z) for (s0, z, _) in groups])
        D = OPCA.project(ob, X, cols)
        # the GPU codes of those tokens, read tile by tile from the payload
        shs, scs, cds = [[] for _ in groups], [[] for _ in groups], [[] for _ in groups]
        for tau in taus:
            k = tau // 128
            ntok = min(128, m - k * 128)
            sub = payload[k * full: k * full + OL.tile_bytes(groups, ntok)]
            sh, sc, cd = OL.unpack(groups, sub, ntok)
            for g in range(len(groups)):
                shs[g].append(sh[g][tau - k * 128])
                scs[g].append(sc[g][tau - k * 128])
                cds[g].append(cd[g][tau - k * 128])
        gpu_payload = OL.pack(groups, [np.array(a) for a in shs], [np.array(a) for a in scs],
                              [np.array(a) for a in cds], len(taus))
        E.assert_codes_parity(gpu_payload, groups, D, len(taus), X, ob, cols, f"fullscale stream={sv}")
        # reconstruction of the same tokens from the GPU payload by the oracle
        Dh = np.zeros((len(taus), ob.r))
        for g, (s0, z, ty) in enumerate(groups):
            Dh[:, s0:s0 + z] = ON.f16(OQ.dequantize_rows(np.array(shs[g]), np.array(scs[g]), np.array(cds[g]), ty))
        Xh = (Dh @ ob.Vd.T + ob.mu[None, :]).reshape(len(taus), spec.layers, spec.kv_heads, spec.head_dim)
        Xh = Xh.transpose(1, 0, 2, 3)
        ref = OR.rope_apply_r7(Xh, 4 + taus, invf, 0) if sv == 0 else ON.bf16(Xh)
        got = out[:, 4 + taus].float().cpu().numpy().astype(np.float64)
        rel = np.linalg.norm(got - ref) / np.linalg.norm(ref)
        print(f"\n[fullscale] stream={sv} r_eff={pi.r_eff} groups={len(groups)} recon rel={rel:.2e}")
        assert rel < 1e-3, rel
        # sinks and window byte-identical
        assert torch.equal(out[:, :4], cache[:, :4]) and torch.equal(out[:, t - 128:], cache[:, t - 128:])


def test_fullscale_plan_properties(run):
    """Any-size properties of the GPU DP output (the literal loop is pinned
    bit-exactly at small sizes): cost within the budget, r_eff within the rank."""
    for P in (run["KP"], run["VP"]):
        pi = P.info()
        assert pi.budget == 32768
        assert pi.bits_per_token <= pi.budget
        assert 0 < pi.r_eff <= pi.r
        starts = [s for (s, _, _) in pi.groups]
        assert starts == sorted(starts)
        assert all(z in (1, 16, 64, 256, 1024) for (_, z, _) in pi.groups)
        assert np.isfinite(pi.expected_error) and pi.expected_error > 0
