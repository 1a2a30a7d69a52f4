"""Per-shard stage times of an emulated N-rank apply: python tools/group_stages.py config world [n_max]"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1808_04580_b200 as fgs
cfg, world = int(sys.argv[1]), int(sys.argv[2])
info = fgs.workload_info(cfg)
X = fgs.workload_nodes(cfg, 2024)
n = X.shape[0]
nvec = 16 if cfg == 5 else 1
g = fgs.ShardGroup(X, fgs.KernelSpec.gaussian(info["sigma"]), fgs.FastsumParams(info["N"], info["m"], info["p"], 0.0), world=world)
x = torch.from_numpy(np.ascontiguousarray(fgs.workload_vectors(n, nvec, 5).T)).cuda()
y = torch.empty_like(x)
g.profile(fgs.OP_SYM_LAPLACIAN, x.data_ptr(), y.data_ptr(), nvec=nvec, reps=2)
ms, ex = g.profile(fgs.OP_SYM_LAPLACIAN, x.data_ptr(), y.data_ptr(), nvec=nvec, reps=5)
st = g.stage_profile(fgs.OP_SYM_LAPLACIAN, x.data_ptr(), y.data_ptr(), nvec=nvec, reps=5)
print("config", cfg, "world", world, "shard ms (phases, graph-free)", np.round(ms, 4), "exchange", round(ex, 4))
print("stages [spread, assemble, planes_fwd, lines(+between), planes_inv, interp] ms:")
for r in range(world):
    print(r, np.round(st[r], 4), g.stats(r))
