import time, numpy as np
import paper_1808_04580_b200 as fgs
info = fgs.workload_info(4)
X = fgs.workload_nodes(4, 2024)
t = time.perf_counter()
op = fgs.AdjacencyOperator(X, fgs.KernelSpec.gaussian(info["sigma"]), fgs.FastsumParams(info["N"], info["m"], info["p"], 0.0))
print("setup s", round(time.perf_counter() - t, 4))
for rep in range(2):
    for wv in (True, False):
        li = fgs.LanczosInfo()
        t = time.perf_counter()
        pairs = fgs.lanczos_largest(op, 20, fgs.LanczosOptions(tol=1e-8, seed=1), li, want_vectors=wv)
        print("vectors" if wv else "values ", "solve s", round(time.perf_counter() - t, 4), li.iterations, op.lanczos_stats())
