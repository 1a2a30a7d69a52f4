"""Times device Lanczos on a BASELINE config with the per-phase trace on."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["FGS_LANCZOS_TRACE"] = "1"
import paper_1808_04580_b200 as fgs  # noqa: E402

c = int(sys.argv[1]) if len(sys.argv) > 1 else 4
info = fgs.workload_info(c)
X = fgs.workload_nodes(c, 2024)
t0 = time.perf_counter()
op = fgs.AdjacencyOperator(X, fgs.KernelSpec.gaussian(info["sigma"]), fgs.FastsumParams(info["N"], info["m"], info["p"]))
t1 = time.perf_counter()
li = fgs.LanczosInfo()
p = fgs.lanczos_largest(op, info["k"], fgs.LanczosOptions(tol=1e-8), li)
t2 = time.perf_counter()
print(f"config {c}: setup {t1 - t0:.3f} s  solve {t2 - t1:.3f} s  iters {li.iterations} conv {li.converged}")
print("stats", op.lanczos_stats())
