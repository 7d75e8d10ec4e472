"""Stage times of the bench workload under environment-variable variants
(tuning experiments; one process, setup once).  Usage:
  python scripts/sweep_env.py 'KVTC_GROUP_M_QUANT=4' 'KVTC_GROUP_M_QUANT=16' ..."""
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
    ap.add_argument("variants", nargs="*")
    ap.add_argument("--iters", type=int, default=5)
    args = ap.parse_args()
    ns = argparse.Namespace(cal_tokens=32768, cal_seqs=2, ncal=65000, rank_cap=10000, cr=16.0)
    spec = make_spec("llama8b")
    torch.cuda.set_device(0)
    (kb, vb), (kp, vp), _ = bench.build_artifacts(K, spec, ns, 0, 1, None)
    Kc = generate(spec, 0, 32768, conversation=0, device="cuda")
    Vc = generate(spec, 1, 32768, conversation=0, device="cuda")
    kv, vv = K.KVView(Kc), K.KVView(Vc)
    Ko, Vo = torch.zeros_like(Kc), torch.zeros_like(Vc)
    cap, wsb = K.compress_sizes(kb, kp, vb, vp, kv)
    cont = torch.empty(cap, dtype=torch.uint8, device="cuda")
    cws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
    K.compress(kb, kp, vb, vp, kv, vv, out=cont, workspace=cws)
    dws = torch.empty(K.decompress_workspace_bytes(kb, kp, vb, vp, cont[:256].cpu().numpy().tobytes()),
                      dtype=torch.uint8, device="cuda")
    base = dict(os.environ)
    order = ["baseline"] + [x for v in args.variants for x in (v, "baseline")]
    for var in order:
        os.environ.clear()
        os.environ.update(base)
        if var != "baseline":
            for kvp in var.split(","):
                k, v = kvp.split("=")
                os.environ[k] = v
        # the decompression workspace depends on the variant (KVTC_DQ_FUSED=0 adds D^)
        dws = torch.empty(K.decompress_workspace_bytes(kb, kp, vb, vp, cont[:256].cpu().numpy().tobytes()),
                          dtype=torch.uint8, device="cuda")
        for _ in range(2):
            K.compress(kb, kp, vb, vp, kv, vv, out=cont, workspace=cws, sync_len=False)
            K.decompress(kb, kp, vb, vp, cont, K.KVView(Ko), K.KVView(Vo), workspace=dws)
        torch.cuda.synchronize()
        K.profile_enable(True)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.iters):
            K.compress(kb, kp, vb, vp, kv, vv, out=cont, workspace=cws, sync_len=False)
            K.decompress(kb, kp, vb, vp, cont, K.KVView(Ko), K.KVView(Vo), workspace=dws)
        e1.record()
        torch.cuda.synchronize()
        st = K.profile_read()
        K.profile_enable(False)
        step = e0.elapsed_time(e1) / args.iters
        parts = " ".join(f"{k}={v[0] / args.iters:.2f}" for k, v in st.items())
        print(f"[sweep] {var:40s} step={step:.2f} ms {parts}", flush=True)


if __name__ == "__main__":
    main()
