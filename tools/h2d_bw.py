import torch, time
for mb in (4, 8, 16, 32, 64, 256):
    n = mb * 1024 * 1024 // 2
    h = torch.empty(n, dtype=torch.bfloat16).pin_memory()
    d = torch.empty(n, dtype=torch.bfloat16, device="cuda")
    for _ in range(2): d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(); 
    for _ in range(5): d.copy_(h, non_blocking=True)
    e.record(); torch.cuda.synchronize()
    ms = s.elapsed_time(e) / 5
    s.record(); 
    for _ in range(5): h.copy_(d, non_blocking=True)
    e.record(); torch.cuda.synchronize()
    ms2 = s.elapsed_time(e) / 5
    print(f"{mb} MB: H2D {mb/1024/ms*1e3:.1f} GB/s  D2H {mb/1024/ms2*1e3:.1f} GB/s")
