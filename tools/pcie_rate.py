import torch, time
for n in (6553600, 13107200):
    h = torch.empty(n, dtype=torch.uint8, pin_memory=True); d = torch.empty(n, dtype=torch.uint8, device="cuda")
    for _ in range(3): d.copy_(h, non_blocking=True); h.copy_(d, non_blocking=True)
    torch.cuda.synchronize()
    e0, e1, e2 = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    e0.record(); d.copy_(h, non_blocking=True); e1.record(); h.copy_(d, non_blocking=True); e2.record(); torch.cuda.synchronize()
    print(n, "H2D GB/s", n / e0.elapsed_time(e1) / 1e6, "D2H GB/s", n / e1.elapsed_time(e2) / 1e6)
