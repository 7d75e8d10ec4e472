#!/usr/bin/env python
"""Times the reconstruction GEMM alone on the Llama-8B bench shape (plan of the
bench, random orthonormal-ish basis, random rows): unfused (dequantise + TMA-fed
GEMM) vs fused (dequantising producer warps), under env variants.  Measurement
only.  usage: python scripts/fused_probe.py 'KVTC_DQ_DEBUG=1' ..."""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2511_01815_b200 import kvtc as K  # noqa: E402


def main():
    plans = json.load(open(os.path.join(ROOT, "profiles", "plans_llama8b_cr16.json")))
    groups = [tuple(g) for g in plans["k"] if g[2] != 0]
    r = max(s + z for s, z, _ in groups)
    L, H, D = 32, 8, 128
    p = L * H * D
    m = 32636
    rng = np.random.default_rng(0)
    V = (rng.standard_normal((p, r), dtype=np.float32) / np.sqrt(p)).astype(np.float32)
    mu = np.zeros(p, np.float32)
    B = K.Basis.create((L, H, D), 1, mu, V)
    del V
    Pl = K.Plan.create(r, groups)
    X = (torch.randn(m, p, device="cuda") * 0.3).bfloat16()
    payload = K.project_quantize(B, Pl, X)
    del X
    out = torch.zeros(L, m + 132, H, D, dtype=torch.bfloat16, device="cuda")
    view = K.KVView(out)
    base = dict(os.environ)
    for var in ["baseline"] + sys.argv[1:] + ["baseline"]:
        os.environ.clear()
        os.environ.update(base)
        if var != "baseline":
            for kv in var.split(","):
                k, v = kv.split("=")
                os.environ[k] = v
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        for it in range(4):
            if it == 1:
                e0.record()
            K.reconstruct_payload(B, Pl, payload, m, 4, 0, L, view)
        e1.record()
        torch.cuda.synchronize()
        fused = e0.elapsed_time(e1) / 3
        Dh = K.dequantize(Pl, payload, m)
        for it in range(4):
            if it == 1:
                e0.record()
            K.reconstruct(B, Pl, Dh, m, 4, 0, L, view)
        e1.record()
        torch.cuda.synchronize()
        unf = e0.elapsed_time(e1) / 3
        print(f"[probe] {var:36s} fused={fused:.2f} ms  tma-fed={unf:.2f} ms", flush=True)


if __name__ == "__main__":
    main()
