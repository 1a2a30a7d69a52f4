"""Pinned-memory H2D / D2H bandwidth on this box (what the e2e leg's exposed
first upload and last download cost).  usage: python tools/pcie_probe.py"""
import torch
for mb in (80, 1280):
    n = mb * 1000 * 1000 // 8
    h = torch.empty(n, dtype=torch.float64).pin_memory()
    d = torch.empty(n, dtype=torch.float64, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    def t(fn, reps=5):
        fn(); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps): fn()
        e1.record(); torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps
    up = t(lambda: d.copy_(h, non_blocking=True))
    dn = t(lambda: h.copy_(d, non_blocking=True))
    h2 = torch.empty(n, dtype=torch.float64).pin_memory(); d2 = torch.empty_like(d)
    def both():
        with torch.cuda.stream(s1): d.copy_(h, non_blocking=True)
        with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
        torch.cuda.current_stream().wait_stream(s1); torch.cuda.current_stream().wait_stream(s2)
    bi = t(both)
    print(f"{mb} MB: H2D {up:.3f} ms ({mb/up:.1f} GB/s)  D2H {dn:.3f} ms ({mb/dn:.1f} GB/s)  both at once {bi:.3f} ms")

# one 80 MB upload as k concurrent pieces on k streams
n = 80 * 1000 * 1000 // 8
h = torch.empty(n, dtype=torch.float64).pin_memory(); d = torch.empty(n, dtype=torch.float64, device="cuda")
for k in (1, 2, 4):
    ss = [torch.cuda.Stream() for _ in range(k)]
    def split():
        m = n // k
        for i, s in enumerate(ss):
            with torch.cuda.stream(s): d[i * m:(i + 1) * m].copy_(h[i * m:(i + 1) * m], non_blocking=True)
        for s in ss: torch.cuda.current_stream().wait_stream(s)
    for _ in range(3): split()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10): split()
    e1.record(); torch.cuda.synchronize()
    print(f"80 MB H2D in {k} piece(s): {e0.elapsed_time(e1)/10:.3f} ms")
