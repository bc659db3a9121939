import torch, time
nb = 64 << 20
h = torch.empty(nb + 4096, dtype=torch.uint8).pin_memory()
d = torch.empty(nb + 4096, dtype=torch.uint8, device="cuda")
for (so, do) in ((0, 0), (28, 0), (0, 28), (28, 28), (28, 1000), (28, 28 + 4096)):
    for name in ("d2h", "h2d"):
        def f():
            if name == "d2h": h[do:do + nb].copy_(d[so:so + nb], non_blocking=True)
            else: d[do:do + nb].copy_(h[so:so + nb], non_blocking=True)
        f(); torch.cuda.synchronize()
        t = time.perf_counter()
        for _ in range(5): f()
        torch.cuda.synchronize()
        print(f"{name} src+{so} dst+{do}: {5 * nb / (time.perf_counter() - t) / 1e9:.1f} GB/s")
