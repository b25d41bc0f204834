"""PCIe copy bandwidth: H2D alone, D2H alone, both concurrently (pinned host buffers)."""
import time, torch
n = 4 << 30
h1 = torch.empty(n, dtype=torch.uint8).pin_memory(); h2 = torch.empty(n, dtype=torch.uint8).pin_memory()
d1 = torch.empty(n, dtype=torch.uint8, device="cuda"); d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def run(h2d, d2h):
    torch.cuda.synchronize(); t = time.perf_counter()
    if h2d:
        with torch.cuda.stream(s1): d1.copy_(h1, non_blocking=True)
    if d2h:
        with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
    torch.cuda.synchronize(); return time.perf_counter() - t
for _ in range(2): run(1, 1)
a, b, c = run(1, 0), run(0, 1), run(1, 1)
print(f"H2D {n/a/1e9:.1f} GB/s, D2H {n/b/1e9:.1f} GB/s, both: {c*1e3:.0f} ms vs sum {1e3*(a+b):.0f} ms / max {1e3*max(a,b):.0f} ms")
