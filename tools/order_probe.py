"""Config-5 block apply on device vectors: internal order vs caller order
(the permutation the C-ABI host path applies inside the handle)."""
import sys, json
sys.path.insert(0, ".")
import numpy as np, torch
import paper_1808_04580_b200 as fgs
from oracle import oracle as orc
info = orc.workload_info(5); X = orc.workload_nodes(5, 2024)
op = fgs.AdjacencyOperator(X, fgs.KernelSpec.gaussian(info["sigma"]), fgs.FastsumParams(info["N"], info["m"], info["p"], 0.0))
s = torch.cuda.Stream(); torch.cuda.set_stream(s); op.set_stream(s.cuda_stream)
n = X.shape[0]
for nvec in (16, 1):
    x = torch.randn(nvec, n, dtype=torch.float64, device="cuda"); y = torch.empty_like(x)
    for internal in (True, False):
        def step():
            op.apply_device(fgs.OP_SYM_LAPLACIAN, x.data_ptr(), y.data_ptr(), nvec=nvec, ld=n, internal_order=internal)
        for _ in range(2): step()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        K = 4 if nvec == 16 else 16
        e0.record(s)
        for _ in range(K): step()
        e1.record(s); torch.cuda.synchronize()
        print(f"nvec {nvec} internal_order={internal}: {e0.elapsed_time(e1)/K:.3f} ms per block, {e0.elapsed_time(e1)/K/nvec:.3f} per vector")
