import ctypes as C, time
import numpy as np, torch
import paper_1808_04580_b200 as fgs
info = fgs.workload_info(2)
X = fgs.workload_nodes(2, 2024); n = X.shape[0]
op = fgs.AdjacencyOperator(X, fgs.KernelSpec.gaussian(info["sigma"]), fgs.FastsumParams(info["N"], info["m"], info["p"], 0.0))
s = torch.cuda.Stream(); torch.cuda.set_stream(s); op.set_stream(s.cuda_stream)
hx = torch.randn(n, dtype=torch.float64).pin_memory(); hy = torch.empty_like(hx).pin_memory()
dx = torch.empty(n, dtype=torch.float64, device="cuda"); dy = torch.empty_like(dx)
L = fgs.lib(); xp = C.cast(hx.data_ptr(), C.POINTER(C.c_double)); yp = C.cast(hy.data_ptr(), C.POINTER(C.c_double))
def timeit(fn, reps=300):
    for _ in range(20): fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter(); a.record(s)
    for _ in range(reps): fn()
    b.record(s); torch.cuda.synchronize(); t1 = time.perf_counter()
    return a.elapsed_time(b) / reps * 1000, (t1 - t0) / reps * 1e6
print("h2d only        us(dev, wall)", timeit(lambda: dx.copy_(hx, non_blocking=True)))
print("d2h only                     ", timeit(lambda: hy.copy_(dx, non_blocking=True)))
print("h2d+d2h+sync                 ", timeit(lambda: (dx.copy_(hx, non_blocking=True), hy.copy_(dx, non_blocking=True), s.synchronize())))
print("device apply (caller order)  ", timeit(lambda: op.apply_device(fgs.OP_SYM_LAPLACIAN, dx.data_ptr(), dy.data_ptr(), nvec=1, ld=n, internal_order=False)))
print("device apply + sync          ", timeit(lambda: (op.apply_device(fgs.OP_SYM_LAPLACIAN, dx.data_ptr(), dy.data_ptr(), nvec=1, ld=n, internal_order=False), s.synchronize())))
print("C ABI host call              ", timeit(lambda: L.fgs_adjacency_apply(op.handle, fgs.OP_SYM_LAPLACIAN, xp, yp, 1, C.c_int64(n))))
