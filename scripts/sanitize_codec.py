"""Toy compress + decompress through every decompression front end (split path,
one-launch inflate + dequantise, layer-streamed) and the stage kernels, for
compute-sanitizer (memcheck / racecheck / synccheck) runs."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from tests import gpu_env as E  # noqa: E402
from paper_2511_01815_b200 import kvtc as K  # noqa: E402


def main():
    spec, invf, kb, vb, Ck, Cv = E.setup("toy")
    shape = (spec.layers, spec.kv_heads, spec.head_dim)
    kp, vp = E.toy_plans(16)
    KB = K.Basis.create(shape, 0, kb.mu, kb.V, kb.sigma, inv_freq=invf, pairing=0)
    VB = K.Basis.create(shape, 1, vb.mu, vb.V, vb.sigma)
    KP, VP = K.Plan.create(kb.r, kp.groups), K.Plan.create(vb.r, vp.groups)
    Kc, Vc = E.caches("toy", 389, 0, conversation=3)
    kd, vd = Kc.cuda(), Vc.cuda()
    cont, _ = K.compress(KB, KP, VB, VP, K.KVView(kd), K.KVView(vd))
    outs = []
    for flag in ("0", "1"):
        os.environ["KVTC_D_INFLATE_DQ"] = flag
        ko, vo = torch.zeros_like(kd), torch.zeros_like(vd)
        K.decompress(KB, KP, VB, VP, cont, K.KVView(ko), K.KVView(vo))
        ls = K.StreamedDecompress(KB, KP, VB, VP, cont)
        lo, lv = torch.zeros_like(kd), torch.zeros_like(vd)
        ls.layers(K.KVView(lo), K.KVView(lv), 0, spec.layers)
        torch.cuda.synchronize()
        outs.append((ko, vo, lo, lv))
    for a, b in zip(outs[0], outs[1]):
        assert torch.equal(a.view(torch.int16), b.view(torch.int16))
    rng = np.random.default_rng(0)
    data = torch.from_numpy((rng.geometric(0.05, 150001) % 256).astype(np.uint8)).cuda()
    sec = K.deflate(data)
    assert torch.equal(K.inflate(sec, data.numel()), data)
    print("sanitize_codec ok")


if __name__ == "__main__":
    main()
