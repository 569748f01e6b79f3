"""PCIe copy bandwidth: H2D, D2H alone and concurrently (pinned, 2 streams)."""
import torch
n = 64 << 20  # floats (256 MB)
h1 = torch.empty(n).pin_memory(); h2 = torch.empty(n).pin_memory()
d1 = torch.empty(n, device="cuda"); d2 = torch.empty(n, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def t(fn):
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(); fn(); torch.cuda.synchronize(); e1.record(); e1.synchronize()
    return e0.elapsed_time(e1)
for _ in range(2):
    a = t(lambda: d1.copy_(h1, non_blocking=True))
    b = t(lambda: h2.copy_(d2, non_blocking=True))
    def both():
        with torch.cuda.stream(s1): d1.copy_(h1, non_blocking=True)
        with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
    c = t(both)
    gb = n * 4 / 1e9
    print(f"H2D {gb / a * 1e3:.1f} GB/s, D2H {gb / b * 1e3:.1f} GB/s, both concurrently {2 * gb / c * 1e3:.1f} GB/s total ({c:.2f} ms vs {a + b:.2f} serial)")
