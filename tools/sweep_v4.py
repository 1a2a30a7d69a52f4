"""Per-kernel timing of d = 3 tensor-core kernel variants (point streams P,
chunk QS) on one plan: FGS_V4_SPREAD / FGS_V4_INTERP are read per launch, so
one operator serves every variant (profile mode = direct launches)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["FGS_GRAPHS"] = "0"
import paper_1808_04580_b200 as fgs  # noqa: E402
import torch  # noqa: E402

cfg = int(sys.argv[1])
variants = sys.argv[2].split(";") if len(sys.argv) > 2 else ["0,32", "1,32", "2,32", "0,64", "1,64", "2,64", "4,32"]
info = fgs.workload_info(cfg)
X = fgs.workload_nodes(cfg, 2024)
if cfg == 5:
    X = X[:2_500_000]  # quarter of config 5 (same density profile scaled): keeps the sweep short
op = fgs.AdjacencyOperator(X, fgs.KernelSpec.gaussian(info["sigma"]), fgs.FastsumParams(info["N"], info["m"], info["p"]))
n = X.shape[0]
x = torch.from_numpy(np.random.default_rng(1).standard_normal(n)).cuda()
y = torch.empty_like(x)
reps = 5
for v in variants:
    os.environ["FGS_V4_SPREAD"] = v
    os.environ["FGS_V4_INTERP"] = v
    try:
        op.apply_device(fgs.OP_SYM_LAPLACIAN, x.data_ptr(), y.data_ptr())
        torch.cuda.synchronize()
        op.profile(True)
        for _ in range(reps):
            op.apply_device(fgs.OP_SYM_LAPLACIAN, x.data_ptr(), y.data_ptr())
        torch.cuda.synchronize()
        op.profile(False)
        ms, napp = op.profile_read()
        print(f"config {cfg} n={n} variant P,QS={v}: spread {1e3 * ms[0] / napp:8.1f} us  interp {1e3 * ms[5] / napp:8.1f} us")
    except Exception as e:  # noqa: BLE001
        print(f"variant {v}: {e}")
        op.profile(False)
