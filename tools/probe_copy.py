"""Time Lanczos with Ritz vectors (C2, C4) and a C5-sized block apply from
pageable host memory: the host_copy bounce path (FGS_* unchanged)."""
import sys
import time

import numpy as np

import paper_1808_04580_b200 as fgs

for cfg in [int(a) for a in sys.argv[1:]] or [2, 4]:
    info = fgs.workload_info(cfg)
    X = fgs.workload_nodes(cfg, 2024)
    op = fgs.AdjacencyOperator(X, fgs.KernelSpec.gaussian(info["sigma"]),
                               fgs.FastsumParams(info["N"], info["m"], info["p"], 0.0))
    if cfg == 5:
        B = fgs.workload_vectors(X.shape[0], 16, 7)
        for rep in range(3):
            t = time.perf_counter()
            Y = op.apply_sym_laplacian(B)
            print(f"config 5 block apply (pageable in/out) {1e3 * (time.perf_counter() - t):.1f} ms", flush=True)
        continue
    for rep in range(3):
        li = fgs.LanczosInfo()
        t = time.perf_counter()
        pairs = fgs.lanczos_largest(op, info["k"], fgs.LanczosOptions(tol=1e-8, seed=1), li)
        print(f"config {cfg} solve+vectors {1e3 * (time.perf_counter() - t):.1f} ms it={li.iterations}", flush=True)
