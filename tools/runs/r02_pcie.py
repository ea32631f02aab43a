# Raw PCIe bandwidth on the box: pinned 280 MB H2D alone, and H2D with a 33 MB D2H alongside
import torch, time
n = 280_000_000
h = torch.empty(n, dtype=torch.uint8).pin_memory()
d = torch.empty(n, dtype=torch.uint8, device="cuda")
o = torch.empty(33_177_600, dtype=torch.uint8, device="cuda")
oh = torch.empty(33_177_600, dtype=torch.uint8).pin_memory()
s2 = torch.cuda.Stream()
for mode in ("h2d", "h2d+d2h", "h2d 4 chunks"):
    ts = []
    for it in range(8):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        if mode == "h2d 4 chunks":
            c = n // 4
            for k in range(4):
                d[k * c:(k + 1) * c].copy_(h[k * c:(k + 1) * c], non_blocking=True)
        else:
            d.copy_(h, non_blocking=True)
        if mode == "h2d+d2h":
            with torch.cuda.stream(s2):
                oh.copy_(o, non_blocking=True)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    print(mode, f"median {ts[4]:.3f} ms -> {n / ts[4] / 1e6:.1f} GB/s")
