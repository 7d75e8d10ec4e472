#!/usr/bin/env python
"""rANS back-end kernels alone on a bench-shaped payload (measurement): encode /
decode times, for ncu."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2511_01815_b200 import kvtc as K  # noqa: E402


def main():
    # tile-periodic bytes with the bench payload's size (133 MB) and tile (512 KiB)
    n, tile = 133_700_000, 524288
    rng = np.random.default_rng(0)
    idx = np.arange(tile)
    base = ((rng.geometric(0.08, tile) + (idx * 7) // tile * 37) % 256).astype(np.uint8)
    data = np.resize(base, n) ^ rng.integers(0, 4, n, dtype=np.uint8)
    t = torch.from_numpy(data).cuda()
    chunk = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
    for it in range(3):
        e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        e0.record()
        sec = K.rans_encode(t, tile, chunk)
        e1.record()
        out = K.rans_decode(sec, n)
        e2.record()
        torch.cuda.synchronize()
        print(f"[rans] chunk {chunk} encode {e0.elapsed_time(e1):.2f} ms decode {e1.elapsed_time(e2):.2f} ms "
              f"gain {n / sec.numel():.4f} ok {bool(torch.equal(out, t))}", flush=True)


if __name__ == "__main__":
    main()
