#!/usr/bin/env python
"""Lossless-stage ablation on the bench payload.

The paper compresses the packed byte array with DEFLATE (Huffman + LZ77)
and ablates other lossless coders (GDeflate within 0.1 CR, zstd,
ANS, ...).  This script measures, on the Llama-8B bench payload (GPU calibration +
DP exactly as bench.py, then the fused projection + quantise + pack of one
32K-token conversation), what each coder reaches per 64 KiB chunk:
  * the library's literal-only DEFLATE sections (what kvtc_compress ships),
  * zlib raw streams at levels 1 / 6 / 9 (LZ77 + Huffman), Z_HUFFMAN_ONLY, Z_RLE,
  * the order-0 entropy bound of each chunk (a static per-chunk model: what an
    ideal ANS / arithmetic coder with a free table would reach),
  * one zlib level-9 stream over the whole payload (no chunking).
Host-side measurement only (stock zlib on the box's cores); nothing here feeds a
parity test.  Writes a JSON summary (default gpurun_out/entropy_ablation.json).
"""
import argparse
import json
import os
import sys
import time
import zlib
from multiprocessing import Pool

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
from kvtc_inputs import make_spec, generate  # noqa: E402
from paper_2511_01815_b200 import kvtc as K  # noqa: E402

CHUNK = 65536


def zsize(args):
    data, level, strategy = args
    c = zlib.compressobj(level, zlib.DEFLATED, -15, 9, strategy)
    return len(c.compress(data) + c.flush())


def h0_bytes(data: bytes) -> float:
    a = np.frombuffer(data, dtype=np.uint8)
    cnt = np.bincount(a, minlength=256).astype(np.float64)
    p = cnt[cnt > 0] / a.size
    return float(-(cnt[cnt > 0] * np.log2(p)).sum() / 8.0)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="llama8b")
    ap.add_argument("--tokens", type=int, default=32768)
    ap.add_argument("--cr", type=float, default=16.0)
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "entropy_ablation.json"))
    args = ap.parse_args()
    ns = argparse.Namespace(cal_tokens=32768, cal_seqs=2, ncal=65000, rank_cap=10000, cr=args.cr)
    spec = make_spec(args.config)
    torch.cuda.set_device(0)
    (kb, vb), (kp, vp), _ = bench.build_artifacts(K, spec, ns, 0, 1, None)
    invf = spec.inv_freq().numpy().astype(np.float32)
    m = args.tokens - 132
    res = {"config": args.config, "tokens": args.tokens, "cr_target": args.cr, "chunk_bytes": CHUNK,
           "host_cores": os.cpu_count(), "streams": {}}
    pool = Pool(os.cpu_count())
    for sv, (b, pl) in enumerate(((kb, kp), (vb, vp))):
        cache = generate(spec, sv, args.tokens, conversation=0, device="cuda")
        X = K.gather(K.KVView(cache), 4, m, sv == 0, invf if sv == 0 else None, 0)
        payload = K.project_quantize(b, pl, X)
        sec = K.deflate(payload)
        torch.cuda.synchronize()
        pb = payload.cpu().numpy().tobytes()
        chunks = [pb[i:i + CHUNK] for i in range(0, len(pb), CHUNK)]
        row = {"payload_bytes": len(pb), "chunks": len(chunks), "library_deflate_section": int(sec.numel())}
        for name, level, strat in (("zlib_l1", 1, zlib.Z_DEFAULT_STRATEGY), ("zlib_l6", 6, zlib.Z_DEFAULT_STRATEGY),
                                   ("zlib_l9", 9, zlib.Z_DEFAULT_STRATEGY),
                                   ("zlib_huffman_only", 6, zlib.Z_HUFFMAN_ONLY), ("zlib_rle", 6, zlib.Z_RLE)):
            t0 = time.time()
            row[name] = int(sum(pool.map(zsize, [(c, level, strat) for c in chunks])))
            row[name + "_s"] = round(time.time() - t0, 2)
        row["order0_entropy_bound"] = float(sum(pool.map(h0_bytes, chunks)))
        t0 = time.time()
        row["zlib_l9_unchunked"] = zsize((pb, 9, zlib.Z_DEFAULT_STRATEGY))
        row["zlib_l9_unchunked_s"] = round(time.time() - t0, 2)
        for k in list(row):
            if k not in ("payload_bytes", "chunks") and not k.endswith("_s"):
                row["gain_" + k] = row["payload_bytes"] / row[k]
        res["streams"][("keys", "values")[sv]] = row
        print(json.dumps({("keys", "values")[sv]: {k: (round(v, 4) if isinstance(v, float) else v)
                                                   for k, v in row.items() if k.startswith("gain_")}}), flush=True)
        del cache, X, payload, sec
        torch.cuda.empty_cache()
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    with open(args.out, "w") as f:
        json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
