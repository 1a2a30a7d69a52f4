import numpy as np, sys
import paper_1808_04580_b200 as fgs
X = np.loadtxt("/tmp/s.csv", delimiter=",", skiprows=1)[:, :3]
op = fgs.AdjacencyOperator(X, fgs.KernelSpec.gaussian(3.5), fgs.FastsumParams.preset(2))
pairs = fgs.lanczos_largest(op, 6, fgs.LanczosOptions(tol=1e-12, seed=1))
AV = op.apply_normalized(pairs.vectors)
rf = np.linalg.norm(AV - pairs.vectors * pairs.values, axis=0).max()
ex = fgs.AdjacencyOperator(X, fgs.KernelSpec.gaussian(3.5), backend="direct")
AVx = ex.apply_normalized(pairs.vectors)
rx = np.linalg.norm(AVx - pairs.vectors * pairs.values, axis=0)
print("BAD" if rf > 1e-10 or rx.max() > 1e-6 else "ok", f"{rf:.2e}", np.array2string(rx, precision=2))
