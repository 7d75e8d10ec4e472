"""cuBLAS (torch.matmul) bf16 on the bench's GEMM shapes, back to back for ~2 s each,
as a reference for what a library GEMM reaches on these shapes under the power cap."""
import time
import torch

def run(M, N, K, label, secs=2.0):
    a = torch.randn(M, K, device="cuda", dtype=torch.bfloat16)
    b = torch.randn(K, N, device="cuda", dtype=torch.bfloat16)
    for _ in range(3):
        c = a @ b
    torch.cuda.synchronize()
    n, t0 = 0, time.time()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    while time.time() - t0 < secs:
        for _ in range(5):
            c = a @ b
        n += 5
        torch.cuda.synchronize()
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / n
    print(f"[cublas] {label}: M={M} N={N} K={K} {ms:.3f} ms {2*M*N*K/ms/1e9:.1f} TFLOP/s", flush=True)

run(32636, 4352, 32768, "compress-shape X.Vc")
run(32636, 32768, 4352, "decompress-shape D.Vd^T")
run(8192, 8192, 8192, "8192^3")
