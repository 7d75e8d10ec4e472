"""One compress + decompress of the bench workload inside cudaProfilerStart/Stop,
for ncu (--profile-from-start off).  Setup (calibration + DP) is identical to
bench.py and runs outside the profiled range."""
import argparse
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
from kvtc_inputs import make_spec, generate  # noqa: E402
from paper_2511_01815_b200 import kvtc as K  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="llama8b")
    ap.add_argument("--tokens", type=int, default=32768)
    ap.add_argument("--cr", type=float, default=16.0)
    ap.add_argument("--iters", type=int, default=1)
    args = ap.parse_args()
    ns = argparse.Namespace(cal_tokens=32768, cal_seqs=2, ncal=65000, rank_cap=10000, cr=args.cr)
    spec = make_spec(args.config)
    torch.cuda.set_device(0)
    (kb, vb), (kp, vp), _ = bench.build_artifacts(K, spec, ns, 0, 1, None)
    Kc = generate(spec, 0, args.tokens, conversation=0, device="cuda")
    Vc = generate(spec, 1, args.tokens, conversation=0, device="cuda")
    kv, vv = K.KVView(Kc), K.KVView(Vc)
    Ko, Vo = torch.zeros_like(Kc), torch.zeros_like(Vc)
    cap, wsb = K.compress_sizes(kb, kp, vb, vp, kv)
    cont = torch.empty(cap, dtype=torch.uint8, device="cuda")
    cws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
    K.compress(kb, kp, vb, vp, kv, vv, out=cont, workspace=cws)
    dws = torch.empty(K.decompress_workspace_bytes(kb, kp, vb, vp, cont[:256].cpu().numpy().tobytes()),
                      dtype=torch.uint8, device="cuda")
    K.decompress(kb, kp, vb, vp, cont, K.KVView(Ko), K.KVView(Vo), workspace=dws)
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    for _ in range(args.iters):
        K.compress(kb, kp, vb, vp, kv, vv, out=cont, workspace=cws, sync_len=False)
        K.decompress(kb, kp, vb, vp, cont, K.KVView(Ko), K.KVView(Vo), workspace=dws)
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()


if __name__ == "__main__":
    main()
