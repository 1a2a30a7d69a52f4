import numpy as np, os
import paper_1808_04580_b200 as fgs
rng = np.random.default_rng(2)
n = 1_000_000
X = rng.uniform(-0.25, 0.25, (n, 3))
op = fgs.AdjacencyOperator(X, fgs.KernelSpec.gaussian(0.3), fgs.FastsumParams(32, 4, 4, 0.0))
V = rng.standard_normal((n, 4))
ref = np.stack([op.apply_normalized(V[:, j]) for j in range(4)], 1)
bad = 0
for rep in range(6):
    W = V.copy()  # fresh pageable buffer
    B = op.apply_normalized(W)
    e = np.max(np.abs(B - ref))
    bad += e > 0
    print(os.environ.get("FGS_PDL"), rep, e)
print("BAD" if bad else "ok")
