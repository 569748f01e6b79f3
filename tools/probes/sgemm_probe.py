"""cuBLAS strict-FP32 SGEMM throughput on this B200 (context for KM-SIMT's FMA roofline)."""
import torch
torch.backends.cuda.matmul.allow_tf32 = False
dev = torch.device("cuda")
for (m, n, k) in [(8192, 8192, 8192), (4096, 144, 4608), (4096, 256, 4608), (256, 676, 2304), (512, 25, 4608)]:
    a = torch.randn(m, k, device=dev); b = torch.randn(k, n, device=dev)
    for _ in range(3): torch.mm(a, b)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 20 if m * n * k > 1e10 else 200
    e0.record()
    for _ in range(reps): torch.mm(a, b)
    e1.record(); torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / reps
    tf = 2 * m * n * k / us / 1e6
    print(f"sgemm {m}x{n}x{k}: {us:8.2f} us  {tf:6.2f} TFLOP/s  ({tf / 74.45 * 100:.1f}% of 74.45)")
