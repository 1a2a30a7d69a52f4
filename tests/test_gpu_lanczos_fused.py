"""The single-device Lanczos step runs as fused kernels (last-block
reductions, three-term + first Gram-Schmidt product, second update + norm +
step scalars); the unfused sequence (FGS_LANCZOS_FUSED=0, what sharded runs
use) performs the same floating-point operations in the same order, so the
two must agree bit for bit -- eigenvalues, Ritz vectors and iteration count
(spectral.cpp:141-256 is the algorithm both follow)."""
import hashlib
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import hashlib, sys
import numpy as np
import paper_1808_04580_b200 as fgs
cfg = int(sys.argv[1])
info = fgs.workload_info(cfg)
X = fgs.workload_nodes(cfg, 2024)
if cfg == 2:
    X = X[::4].copy()
op = fgs.AdjacencyOperator(X, fgs.KernelSpec.gaussian(info["sigma"]),
                           fgs.FastsumParams(info["N"], info["m"], info["p"], 0.0))
li = fgs.LanczosInfo()
pairs = fgs.lanczos_largest(op, info["k"], fgs.LanczosOptions(tol=1e-8, seed=3), li)
h = hashlib.sha256(np.ascontiguousarray(pairs.values).tobytes() + np.ascontiguousarray(pairs.vectors).tobytes())
print(li.iterations, int(li.converged), h.hexdigest())
"""


def _run(cfg, fused):
    env = dict(os.environ)
    env["FGS_LANCZOS_FUSED"] = "1" if fused else "0"
    env["PYTHONPATH"] = ROOT + os.pathsep + env.get("PYTHONPATH", "")
    out = subprocess.run([sys.executable, "-c", SCRIPT, str(cfg)], env=env, capture_output=True, text=True,
                         timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    return out.stdout.strip().splitlines()[-1]


@pytest.mark.parametrize("cfg", [1, 2])
def test_fused_lanczos_bitwise_equals_unfused(cfg):
    a, b = _run(cfg, True), _run(cfg, False)
    assert a == b
    assert a.split()[1] == "1"
