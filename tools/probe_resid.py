import numpy as np, subprocess, json, sys
import paper_1808_04580_b200 as fgs
from paper_1808_04580_b200 import build
build.build()
exe = "paper_1808_04580_b200/fgs-b200"
subprocess.run([exe, "gen", "--spiral", "--per-class", "400", "--out", "/tmp/s.csv", "--seed", "4"], check=True)
X = np.loadtxt("/tmp/s.csv", delimiter=",", skiprows=1)[:, :3]
op = fgs.AdjacencyOperator(X, fgs.KernelSpec.gaussian(3.5), fgs.FastsumParams.preset(2))
pairs = fgs.lanczos_largest(op, 6, fgs.LanczosOptions(tol=1e-12, seed=1))
AV = op.apply_normalized(pairs.vectors)
print("python resid", np.linalg.norm(AV - pairs.vectors * pairs.values, axis=0))
AV1 = np.stack([op.apply_normalized(pairs.vectors[:, j]) for j in range(6)], 1)
print("python resid single", np.linalg.norm(AV1 - pairs.vectors * pairs.values, axis=0))
print("vals", pairs.values)
subprocess.run([exe, "eigs", "--in", "/tmp/s.csv", "--out", "/tmp/e.json", "--sigma", "3.5", "--k", "6"], check=True)
rep = json.load(open("/tmp/e.json"))
print("cli ok")
subprocess.run([exe, "eigs", "--in", "/tmp/s.csv", "--out", "/tmp/e2.json", "--sigma", "3.5", "--k", "6", "--with-reference"], check=True)
rep = json.load(open("/tmp/e2.json"))
print("cli+ref", rep["eigenvalues"], json.dumps(rep["metrics"]))
ex = fgs.AdjacencyOperator(X, fgs.KernelSpec.gaussian(3.5), backend="direct")
AVx = ex.apply_normalized(pairs.vectors)
print("exact resid", np.linalg.norm(AVx - pairs.vectors * pairs.values, axis=0))
pe = fgs.lanczos_largest(ex, 6, fgs.LanczosOptions(tol=1e-13, seed=12345))
print("exact vals", pe.values)
