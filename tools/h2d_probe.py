import torch, time
n = 1 << 30
h = torch.empty(n, dtype=torch.float16, pin_memory=True)
d = torch.empty(n, dtype=torch.float16, device="cuda")
for chunks in (1, 8, 32):
    s = torch.cuda.Stream()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(3):
        c = n // chunks
        with torch.cuda.stream(s):
            for i in range(chunks):
                d[i*c:(i+1)*c].copy_(h[i*c:(i+1)*c], non_blocking=True)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / 3
    print(f"H2D 2 GiB in {chunks} chunks: {dt*1e3:.1f} ms = {2*n/dt/1e9:.1f} GB/s")
