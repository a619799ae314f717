import torch, time
for mb in (32, 256):
    n = mb * 1024 * 1024 // 2
    h = torch.empty(n, dtype=torch.bfloat16).pin_memory()
    d = torch.empty(n, dtype=torch.bfloat16, device="cuda")
    s = torch.cuda.Stream()
    for chunks in (1, 4):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(s):
            e0.record(s)
            for _ in range(10):
                for c in range(chunks):
                    sl = slice(c * n // chunks, (c + 1) * n // chunks)
                    d[sl].copy_(h[sl], non_blocking=True)
            e1.record(s)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 10
        print(f"{mb} MB chunks={chunks}: {ms:.3f} ms  {mb*1.048576/ms:.1f} GB/s")
