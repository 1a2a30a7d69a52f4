"""Per-stage device times of one BASELINE config for several tuning builds
(libfgs_b200_<tag>.so from FGS_BUILD_TAG=<tag> FGS_NVCC_DEFINES=...
python -m paper_1808_04580_b200.build).  Each build runs in its own process.
Usage: python tools/variant_bench.py <config> <tag> [<tag> ...]   ('' = the product .so)"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r'''
import json, sys, time
sys.path.insert(0, __ROOT__)
import numpy as np, torch
import paper_1808_04580_b200 as fgs
if __TAG__:
    fgs.LIB_PATH = fgs.LIB_PATH.replace("libfgs_b200.so", f"libfgs_b200_{__TAG__}.so")
from oracle import oracle as orc
info = orc.workload_info(__CFG__)
X = orc.workload_nodes(__CFG__, 2024)
nvec = 16 if __CFG__ == 5 else 1
op = fgs.AdjacencyOperator(X, fgs.KernelSpec.gaussian(info["sigma"]), fgs.FastsumParams(info["N"], info["m"], info["p"], 0.0))
s = torch.cuda.Stream(); torch.cuda.set_stream(s); op.set_stream(s.cuda_stream)
n = X.shape[0]
x = torch.randn(nvec, n, dtype=torch.float64, device="cuda"); y = torch.empty_like(x)
flush = torch.empty(int(256e6) // 4, dtype=torch.float32, device="cuda")
def step():
    op.apply_device(fgs.OP_SYM_LAPLACIAN, x.data_ptr(), y.data_ptr(), nvec=nvec, ld=n, internal_order=True)
for _ in range(3): step()
K = 3 if __CFG__ == 5 else 20
ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
torch.cuda.synchronize()
for a, b in ev:
    flush.zero_(); a.record(s); step(); b.record(s)
torch.cuda.synchronize()
ms = sum(a.elapsed_time(b) for a, b in ev) / K
op.profile(True)
for _ in range(K):
    flush.zero_(); step()
torch.cuda.synchronize(); op.profile(False)
st, napp = op.profile_read()
print(json.dumps({"tag": __TAG__, "config": __CFG__, "ms_per_step": ms, "matvecs_s": nvec / ms * 1e3,
                  "stages": dict(zip(fgs.STAGES, [round(v / napp, 4) for v in st]))}))
'''

if __name__ == "__main__":
    cfg = int(sys.argv[1])
    for tag in sys.argv[2:]:
        tag = "" if tag in ("''", "-", "base") else tag
        code = CHILD.replace("__ROOT__", repr(ROOT)).replace("__TAG__", repr(tag)).replace("__CFG__", str(cfg))
        r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=900)
        line = r.stdout.strip().splitlines()[-1] if r.stdout.strip() else json.dumps({"tag": tag, "error": r.stderr[-800:]})
        print(line, flush=True)
