"""Host-side phase breakdown of warm Lanczos solves (FGS_LANCZOS_TRACE=1:
prologue / loop / Ritz / vectors copy-out lines on stderr) for the given
configs.  usage: FGS_LANCZOS_TRACE=1 python tools/lz_trace.py 2 4"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1808_04580_b200 as fgs

for cfg in [int(a) for a in sys.argv[1:]] or [2, 4]:
    info = fgs.workload_info(cfg)
    X = fgs.workload_nodes(cfg, 2024)
    op = fgs.AdjacencyOperator(X, fgs.KernelSpec.gaussian(info["sigma"]),
                               fgs.FastsumParams(info["N"], info["m"], info["p"], 0.0))
    for rep in range(3):
        li = fgs.LanczosInfo()
        print(f"--- config {cfg} solve {rep}", file=sys.stderr, flush=True)
        t0 = time.perf_counter()
        fgs.lanczos_largest(op, info["k"], fgs.LanczosOptions(tol=1e-8, seed=1), li)
        print(f"config {cfg} solve {rep}: {1e3 * (time.perf_counter() - t0):.2f} ms, {li.iterations} iterations",
              file=sys.stderr, flush=True)
