import torch, time
for mb in (26, 59, 105, 1024):
    n = mb << 20
    h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    h.fill_(1)
    d = torch.empty(n, dtype=torch.uint8, device="cuda")
    s = torch.cuda.Stream()
    for _ in range(3):
        with torch.cuda.stream(s):
            d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(s):
        e0.record(); 
        for _ in range(5): d.copy_(h, non_blocking=True)
        e1.record()
    torch.cuda.synchronize()
    print(mb, "MB H2D", 5 * n / (e0.elapsed_time(e1) / 1e3) / 1e9, "GB/s")
    with torch.cuda.stream(s):
        e0.record(); 
        for _ in range(5): h.copy_(d, non_blocking=True)
        e1.record()
    torch.cuda.synchronize()
    print(mb, "MB D2H", 5 * n / (e0.elapsed_time(e1) / 1e3) / 1e9, "GB/s")
