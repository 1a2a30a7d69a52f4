"""Lanczos time-to-k (C2, C4) for tuning builds: python tools/lz_variant.py tag [tag ...] ('base' = product)"""
import json, os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import json, sys, time
sys.path.insert(0, __ROOT__)
import numpy as np, torch
import paper_1808_04580_b200 as fgs
if __TAG__:
    fgs.LIB_PATH = fgs.LIB_PATH.replace("libfgs_b200.so", f"libfgs_b200_{__TAG__}.so")
out = {"tag": __TAG__}
for cfg in (2, 4):
    info = fgs.workload_info(cfg)
    X = fgs.workload_nodes(cfg, 2024)
    op = fgs.AdjacencyOperator(X, fgs.KernelSpec.gaussian(info["sigma"]), fgs.FastsumParams(info["N"], info["m"], info["p"], 0.0))
    ts = []
    for _ in range(3):
        li = fgs.LanczosInfo()
        torch.cuda.synchronize(); t0 = time.perf_counter()
        fgs.lanczos_largest(op, info["k"], fgs.LanczosOptions(tol=1e-8, seed=1), li, want_vectors=False)
        torch.cuda.synchronize(); ts.append(time.perf_counter() - t0)
    out[f"c{cfg}"] = {"warm_s": min(ts[1:]), "iters": li.iterations, **op.lanczos_stats()}
print(json.dumps(out))
'''
for tag in sys.argv[1:]:
    tag = "" if tag == "base" else tag
    code = CHILD.replace("__ROOT__", repr(ROOT)).replace("__TAG__", repr(tag))
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=900)
    print(r.stdout.strip().splitlines()[-1] if r.stdout.strip() else json.dumps({"tag": tag, "error": r.stderr[-600:]}), flush=True)
