import numpy as np
import paper_1808_04580_b200 as fgs
X = np.loadtxt("/tmp/s.csv", delimiter=",", skiprows=1)[:, :3]
k = fgs.KernelSpec.gaussian(3.5)
op = fgs.AdjacencyOperator(X, k, fgs.FastsumParams.preset(2))
print("degrees finite", np.isfinite(op.degrees()).all())
x = np.random.default_rng(0).standard_normal(2000)
print("single apply finite", np.isfinite(op.apply_normalized(x)).all())
pairs = fgs.lanczos_largest(op, 6, fgs.LanczosOptions(tol=1e-12, seed=1))
print("vals", pairs.values, "vec finite", np.isfinite(pairs.vectors).all())
AV = op.apply_normalized(pairs.vectors)
print("fast block finite per col", np.isfinite(AV).all(0), np.linalg.norm(AV - pairs.vectors * pairs.values, axis=0))
ex = fgs.AdjacencyOperator(X, k, backend="direct")
print("direct degrees finite", np.isfinite(ex.degrees()).all())
AVx = ex.apply_normalized(pairs.vectors)
print("direct block finite per col", np.isfinite(AVx).all(0), np.linalg.norm(AVx - pairs.vectors * pairs.values, axis=0))
for nv in (1, 2, 3, 4, 5, 7):
    B = ex.apply_normalized(pairs.vectors[:, :min(nv, 6)] if nv <= 6 else np.concatenate([pairs.vectors, pairs.vectors[:, :1]], 1))
    print("direct nvec", nv, np.isfinite(B).all(0))
