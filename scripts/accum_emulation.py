#!/usr/bin/env python
"""How far is the >= 99.99 % code-agreement target from an fp32-accumulated
projection?  (writes profiles/r02_accum_emulation.json.)

On the Llama-8B bench workload (GPU calibration + DP as bench.py), for a sample
of middle tokens: the oracle's fp64 D = X V_c - mu V_c (R2) and the codes it
implies; the GPU's actual codes (from its container); and host EMULATIONS of
fp32 accumulation orders over the K = p = 32768 terms, each K = 16 MMA block's
dot product taken exactly and added into an fp32 accumulator with RNE:
  acc1 — one accumulator, blocks in order (what the tensor core does);
  acc2 / acc4 — 2 / 4 accumulators, blocks interleaved, summed at the end
  (a split-K over TMEM accumulators); tree — pairwise tree over the blocks.
If acc1 reproduces the GPU's measured mismatch rate, the others predict what a
split-K kernel would reach.  Emulation only: numbers from the oracle side
(quantize_rows on each emulated D); nothing here feeds a parity test.
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def f32(a):
    return np.asarray(a, dtype=np.float64).astype(np.float32).astype(np.float64)


def codes_of(D, groups):
    from oracle import quant as OQ
    out, off = [], 0
    for (_, z, t) in groups:
        out.append((t, OQ.quantize_rows(D[:, off:off + z], t)[2]))
        off += z
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tokens", type=int, default=128)
    args = ap.parse_args()
    import bench
    import zlib
    from kvtc_inputs import generate, make_spec
    from oracle import layout as OL
    from oracle import pca as OPCA
    from oracle import rope as OR
    from paper_2511_01815_b200 import kvtc as K
    from tests.kvtc_format import parse_container, parse_section
    spec = make_spec("llama8b")
    ns = argparse.Namespace(cal_tokens=32768, cal_seqs=2, ncal=65000, rank_cap=10000, cr=16.0)
    (KB, VB), (KP, VP), _ = bench.build_artifacts(K, spec, ns, 0, 1, None)
    t = 32768
    Kc = generate(spec, 0, t, conversation=0, device="cuda")
    Vc = generate(spec, 1, t, conversation=0, device="cuda")
    cont, _ = K.compress(KB, KP, VB, VP, K.KVView(Kc), K.KVView(Vc))
    buf = cont.cpu().numpy().tobytes()
    h = parse_container(buf)
    m = t - 132
    rng = np.random.default_rng(5)
    taus = np.sort(rng.choice(m, args.tokens, replace=False))
    invf = spec.inv_freq().double().numpy()
    res = {}
    for sv, B, P, cache in ((0, KB, KP, Kc), (1, VB, VP, Vc)):
        pi = P.info()
        groups = [tuple(g) for g in pi.groups]
        mu, V, sg = B.get()
        ob = OPCA.Basis(mu=mu.astype(np.float64), V=V[:, :pi.r_eff].astype(np.float64), sigma=sg[:pi.r_eff], n=0)
        rows = cache[:, 4 + taus].float().cpu().numpy().astype(np.float64)
        if sv == 0:
            rows = OR.unrope_r1(rows, 4 + taus, invf, 0)
        X = OPCA.flatten_rows(rows)
        cols = np.concatenate([np.arange(s0, s0 + z) for (s0, z, _) in groups])
        Vcc = ob.Vc[:, cols]
        bias = f32(ob.mu @ Vcc)
        D_ref = X @ Vcc - (ob.mu @ Vcc)[None, :]
        # GPU codes of the sampled tokens
        sec = parse_section(buf[h["sec_k" if sv == 0 else "sec_v"]:])
        payload = b"".join(zlib.decompress(x, wbits=-15) for x in sec["streams"])
        full = OL.tile_bytes(groups, 128)
        gpu = [[] for _ in groups]
        for tau in taus:
            k = tau // 128
            ntok = min(128, m - k * 128)
            _, _, cd = OL.unpack(groups, payload[k * full: k * full + OL.tile_bytes(groups, ntok)], ntok)
            for g in range(len(groups)):
                gpu[g].append(cd[g][tau - k * 128])
        # emulated accumulation orders (16-term exact blocks, fp32 RNE adds)
        nb = X.shape[1] // 16
        parts = np.stack([X[:, 16 * b:16 * b + 16] @ Vcc[16 * b:16 * b + 16] for b in range(nb)])   # [nb, T, C]
        emu = {}
        for name, nacc in (("acc1", 1), ("acc2", 2), ("acc4", 4)):
            accs = [np.zeros(parts.shape[1:]) for _ in range(nacc)]
            for b in range(nb):
                accs[b % nacc] = f32(accs[b % nacc] + f32(parts[b]))
            tot = accs[0]
            for a in accs[1:]:
                tot = f32(tot + a)
            emu[name] = f32(tot - bias[None, :])
        w = [f32(p) for p in parts]
        while len(w) > 1:
            w = [f32(w[i] + w[i + 1]) if i + 1 < len(w) else w[i] for i in range(0, len(w), 2)]
        emu["tree"] = f32(w[0] - bias[None, :])
        # measured on the GPU: the K = p projection as 1 / 2 / 4 tcgen05 GEMMs over
        # feature ranges (kvtc_stage_project_partial), the partials added in fp32 (RNE),
        # quantised by the library's SIMT quantiser: does a shorter tensor-core
        # accumulation chain reduce the boundary flips?
        import torch
        Xg = torch.from_numpy(X).to(torch.bfloat16).cuda()
        p_ = X.shape[1]
        gpu_split = {}
        for nsp in (1, 2, 4):
            step = p_ // nsp
            Dg = None
            for q in range(nsp):
                Pq = K.project_partial(B, P, Xg[:, q * step:(q + 1) * step].contiguous(), q * step, (q + 1) * step, q == 0)
                Dg = Pq if Dg is None else Dg + Pq
            pay = K.quantize_pack(P, Dg.contiguous()).cpu().numpy().tobytes()
            _, _, cdq = OL.unpack(groups, pay, len(taus))
            gpu_split["gpu_split%d" % nsp] = [(t, np.array(cdq[g])) for g, (_, _, t) in enumerate(groups)]
        ref = codes_of(D_ref, groups)
        out = {}
        for name, D in [("gpu", None)] + list(gpu_split.items()) + list(emu.items()):
            per = {}
            if isinstance(D, list):
                cds = D
            else:
                cds = codes_of(D, groups) if D is not None else [(t, np.array(gpu[g])) for g, (_, _, t) in enumerate(groups)]
            for (t, a), (_, b) in zip(ref, cds):
                x, y = per.get(t, (0, 0))
                per[t] = (x + int((a != b).sum()), y + a.size)
            out[name] = {["", "int2", "int4", "fp8"][t]: {"mismatch": x, "codes": y, "rate": x / y}
                         for t, (x, y) in sorted(per.items())}
        res["kv"[sv]] = out
        print("kv"[sv], json.dumps(out), flush=True)
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "r02_accum_emulation.json"), "w") as f:
        json.dump({"tokens": int(args.tokens), "what": __doc__.strip().splitlines()[0], "streams": res}, f, indent=1)


if __name__ == "__main__":
    main()
