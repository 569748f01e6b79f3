import torch
torch.backends.cuda.matmul.allow_tf32 = True
for dt in (torch.float32, torch.bfloat16):
    A = torch.randn(4096, 4608, device="cuda", dtype=dt)
    As = [A.clone() for _ in range(4)]
    B = torch.randn(4608, 144, device="cuda", dtype=dt)
    for a in As: torch.matmul(a, B)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for i in range(12): torch.matmul(As[i % 4], B)
    g.replay(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / 12
    by = A.numel() * A.element_size() + B.numel() * B.element_size() + 4096 * 144 * A.element_size()
    print(dt, f"{us:.2f} us", f"{by / us / 1e3:.0f} GB/s")
