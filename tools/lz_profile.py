"""One C4 Lanczos solve (k = 20) for an ncu launch list of the step kernels."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1808_04580_b200 as fgs
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
info = fgs.workload_info(cfg)
X = fgs.workload_nodes(cfg, 2024)
op = fgs.AdjacencyOperator(X, fgs.KernelSpec.gaussian(info["sigma"]), fgs.FastsumParams(info["N"], info["m"], info["p"], 0.0))
li = fgs.LanczosInfo()
fgs.lanczos_largest(op, info["k"], fgs.LanczosOptions(tol=1e-8, seed=1), li)
print(li.iterations)
