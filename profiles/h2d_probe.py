import torch, time
n = 1 << 28  # 1 GiB fp32
h = torch.empty(n * 8, dtype=torch.float32, pin_memory=True)
d = torch.empty(n * 8, dtype=torch.float32, device="cuda")
for streams in (1, 2, 4):
    ss = [torch.cuda.Stream() for _ in range(streams)]
    torch.cuda.synchronize()
    for rep in range(2):
        t0 = time.perf_counter()
        chunk = (n * 8) // 32
        for c in range(32):
            s = ss[c % streams]
            with torch.cuda.stream(s):
                d[c * chunk:(c + 1) * chunk].copy_(h[c * chunk:(c + 1) * chunk], non_blocking=True)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
    print(f"streams={streams}: {h.numel() * 4 / dt / 1e9:.1f} GB/s", flush=True)
