"""Print plan statistics (FGS_PLAN_STATS) for the BASELINE configs."""
import os
import sys

os.environ["FGS_PLAN_STATS"] = "1"
import paper_1808_04580_b200 as fgs  # noqa: E402

for c in [int(a) for a in sys.argv[1:]] or [1, 2, 3, 4]:
    info = fgs.workload_info(c)
    X = fgs.workload_nodes(c, seed=2024)
    print(f"config {c}", flush=True)
    op = fgs.AdjacencyOperator(X, fgs.KernelSpec.gaussian(info["sigma"]),
                               fgs.FastsumParams(info["N"], info["m"], info["p"], 0.0))
    op.apply_sym_laplacian(fgs.workload_vectors(X.shape[0], 1, 1))
    del op
