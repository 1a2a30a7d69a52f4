import paper_1808_04580_b200 as fgs
info = fgs.workload_info(2)
X = fgs.workload_nodes(2, 2024)
op = fgs.AdjacencyOperator(X, fgs.KernelSpec.gaussian(info["sigma"]), fgs.FastsumParams(info["N"], info["m"], info["p"], 0.0))
li = fgs.LanczosInfo()
pairs = fgs.lanczos_largest(op, info["k"], fgs.LanczosOptions(tol=1e-8, seed=1), li)
print(li.iterations)
