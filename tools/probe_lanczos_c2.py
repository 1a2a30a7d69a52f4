import time
import paper_1808_04580_b200 as fgs
for cfg in (2, 1):
    info = fgs.workload_info(cfg)
    X = fgs.workload_nodes(cfg, 2024)
    op = fgs.AdjacencyOperator(X, fgs.KernelSpec.gaussian(info["sigma"]), fgs.FastsumParams(info["N"], info["m"], info["p"], 0.0))
    for rep in range(3):
        li = fgs.LanczosInfo()
        t = time.perf_counter()
        pairs = fgs.lanczos_largest(op, info["k"], fgs.LanczosOptions(tol=1e-8, seed=1), li)
        print(f"config {cfg} solve {1e3*(time.perf_counter()-t):.2f} ms it={li.iterations}", op.lanczos_stats())
