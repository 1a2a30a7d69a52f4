"""Compare one C4 L_s apply against a saved reference vector (A/B builds)."""
import sys
import numpy as np
import paper_1808_04580_b200 as fgs
info = fgs.workload_info(4)
X = fgs.workload_nodes(4, 2024)
op = fgs.AdjacencyOperator(X, fgs.KernelSpec.gaussian(info["sigma"]), fgs.FastsumParams(info["N"], info["m"], info["p"], 0.0))
y = op.apply_sym_laplacian(fgs.workload_vectors(X.shape[0], 1, 99))
if sys.argv[1] == "save":
    np.save("gpurun_out/c4_ref.npy", y)
else:
    r = np.load("gpurun_out/c4_ref.npy")
    print(sys.argv[2], "rel diff vs A", np.linalg.norm(y - r) / np.linalg.norm(r), flush=True)
