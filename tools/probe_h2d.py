import time, torch
n = 100_000
hx = torch.randn(n, dtype=torch.float64).pin_memory()
dx = torch.empty(n, dtype=torch.float64, device="cuda")
main = torch.cuda.Stream()
for parts in (1, 2, 4, 8):
    streams = [torch.cuda.Stream() for _ in range(parts)]
    ch = (n + parts - 1) // parts
    def go():
        ev = torch.cuda.Event()
        ev.record(main)
        done = []
        for p, st in enumerate(streams):
            st.wait_event(ev)
            with torch.cuda.stream(st):
                dx[p * ch:(p + 1) * ch].copy_(hx[p * ch:(p + 1) * ch], non_blocking=True)
            e = torch.cuda.Event(); e.record(st); done.append(e)
        for e in done:
            main.wait_event(e)
    for _ in range(20): go()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(main)
    for _ in range(300): go()
    b.record(main); torch.cuda.synchronize()
    us = a.elapsed_time(b) / 300 * 1000
    print(f"H2D 800 KB in {parts} part(s): {us:.1f} us  ({8 * n / us / 1e3:.1f} GB/s)")
big = torch.randn(64 * n, dtype=torch.float64).pin_memory(); dbig = torch.empty(64 * n, dtype=torch.float64, device="cuda")
for _ in range(3): dbig.copy_(big, non_blocking=True)
torch.cuda.synchronize(); t = time.perf_counter()
for _ in range(10): dbig.copy_(big, non_blocking=True)
torch.cuda.synchronize(); print(f"H2D 51 MB: {51.2e6 * 10 / (time.perf_counter() - t) / 1e9:.1f} GB/s")
