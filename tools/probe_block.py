import numpy as np, os
import paper_1808_04580_b200 as fgs
rng = np.random.default_rng(1)
X = rng.uniform(-1, 1, (2000, 3))
for backend in ("direct", "fastsum"):
    op = fgs.AdjacencyOperator(X, fgs.KernelSpec.gaussian(0.8), fgs.FastsumParams.preset(2), backend=backend)
    V = rng.standard_normal((2000, 6))
    errs = []
    for rep in range(3):
        B = op.apply_normalized(V)
        S = np.stack([op.apply_normalized(V[:, j]) for j in range(6)], 1)
        errs.append(np.max(np.abs(B - S), axis=0))
    print(backend, os.environ.get("FGS_PDL"), os.environ.get("FGS_GRAPHS"), np.array(errs).max(0))
