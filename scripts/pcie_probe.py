import torch, time
n = 2 * 1024**3
h1 = torch.empty(n, dtype=torch.uint8).pin_memory(); h2 = torch.empty(n, dtype=torch.uint8).pin_memory()
d1 = torch.empty(n, dtype=torch.uint8, device="cuda"); d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def t(f, reps=5):
    torch.cuda.synchronize(); a = time.perf_counter()
    for _ in range(reps): f()
    torch.cuda.synchronize(); return (time.perf_counter() - a) / reps
h2d = t(lambda: d1.copy_(h1, non_blocking=True)); print("H2D GB/s", n / h2d / 1e9)
d2h = t(lambda: h2.copy_(d2, non_blocking=True)); print("D2H GB/s", n / d2h / 1e9)
def both():
    with torch.cuda.stream(s1): d1.copy_(h1, non_blocking=True)
    with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
bt = t(both); print("concurrent: each direction GB/s", n / bt / 1e9)
