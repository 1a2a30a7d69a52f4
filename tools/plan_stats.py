import sys; sys.path.insert(0,'.')
import paper_1808_04580_b200 as fgs
from oracle import oracle as orc
for c in (4,):
    info = orc.workload_info(c); X = orc.workload_nodes(c, 2024)
    op = fgs.AdjacencyOperator(X, fgs.KernelSpec.gaussian(info["sigma"]), fgs.FastsumParams(info["N"], info["m"], info["p"], 0.0))
    print(c, op.plan_stats())
