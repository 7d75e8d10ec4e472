"""__graft_entry__.smoke(): one small invocation of the whole path on cuda:0,
checked against the oracle (toy config, BASELINE.json configs[0]).

  oracle PCA basis (fp64)  ->  GPU DP plan (bit-exact vs the literal loop)
  -> kvtc_compress / kvtc_decompress on cuda:0 through the C ABI
  -> codes vs the oracle's fp64 projection, stock zlib inflates every chunk,
     sinks/window byte-identical, reconstruction within 1e-3 of the oracle's.
"""
from __future__ import annotations

import zlib

import numpy as np
import torch


def run_smoke() -> None:
    from paper_2511_01815_b200 import kvtc as K
    from kvtc_inputs import make_spec, generate, sample_positions
    from oracle import codec as OC, dp as ODP, layout as OL, pca as OPCA
    from tests.kvtc_format import parse_container, parse_section
    from tests import gpu_env as E

    K.device_check()
    spec = make_spec("toy")
    invf = spec.inv_freq().double().numpy()
    cal = [generate(spec, st, 2048, conversation=100).double().numpy() for st in (0, 1)]
    samples = sample_positions([2048], 2000, sinks=4, seed=0)
    Ck = OPCA.gather([(cal[0], 0)], samples, True, invf)
    Cv = OPCA.gather([(cal[1], 0)], samples, False)
    kb, vb = OPCA.fit(Ck, 10000), OPCA.fit(Cv, 10000)
    shape = (spec.layers, spec.kv_heads, spec.head_dim)
    KB = K.Basis.create(shape, 0, kb.mu, kb.V, kb.sigma, inv_freq=invf.astype(np.float32))
    VB = K.Basis.create(shape, 1, vb.mu, vb.V, vb.sigma)
    plans = []
    for ob, C in ((kb, Ck), (vb, Cv)):
        P = OPCA.dp_coefficients(ob, C).astype(np.float32)
        oplan, res, B = ODP.allocate(P.astype(np.float64), 16, spec.p)
        gp = K.allocate_bits_from_coeffs(torch.from_numpy(P).cuda(), spec.p, 16.0)
        info = gp.info()
        assert info.groups == [tuple(g) for g in oplan.groups], "GPU DP plan differs from the literal loop"
        assert info.expected_error == res.best[-1, B], "GPU DP table value differs"
        plans.append((gp, oplan))
    (KP, okp), (VP, ovp) = plans
    t = 512
    Kc = generate(spec, 0, t, conversation=0)
    Vc = generate(spec, 1, t, conversation=0)
    kd, vd = Kc.cuda(), Vc.cuda()
    cont, _ = K.compress(KB, KP, VB, VP, K.KVView(kd), K.KVView(vd))
    ko, vo = torch.zeros_like(kd), torch.zeros_like(vd)
    K.decompress(KB, KP, VB, VP, cont, K.KVView(ko), K.KVView(vo))
    torch.cuda.synchronize()
    buf = cont.cpu().numpy().tobytes()
    h = parse_container(buf)
    m = t - 132
    oc = OC.compress(Kc.double().numpy(), Vc.double().numpy(), 0, kb, okp, vb, ovp, invf)
    K2, V2 = OC.decompress(oc, kb, okp, vb, ovp, invf)
    for sv, so, op, ob, cache, got, ref in ((0, oc.k, okp, kb, Kc, ko, K2), (1, oc.v, ovp, vb, Vc, vo, V2)):
        sec = parse_section(buf[h["sec_k" if sv == 0 else "sec_v"]:])
        payload = b"".join(zlib.decompress(s, wbits=-15) for s in sec["streams"])
        assert len(payload) == len(so.payload)
        X = OC.stream_rows(cache.double().numpy(), 4, 128, 0, sv == 0, invf, 0)
        cols = np.concatenate([np.arange(s0, s0 + z) for (s0, z, _) in op.groups])
        E.assert_codes_parity(payload, op.groups, so.D, m, X, ob, cols, f"smoke stream={sv}")
        g = got.float().cpu().numpy().astype(np.float64)
        o = cache.double().numpy()
        assert np.array_equal(g[:, :4], o[:, :4]) and np.array_equal(g[:, t - 128:], o[:, t - 128:])
        rel = np.linalg.norm(g[:, 4:t - 128] - ref[:, 4:t - 128]) / np.linalg.norm(ref[:, 4:t - 128])
        assert rel < 1e-3, rel
    print(f"smoke ok: toy compress+decompress on {torch.cuda.get_device_name(0)}, container {len(buf)} B, "
          f"launches {K.launch_count()}")
