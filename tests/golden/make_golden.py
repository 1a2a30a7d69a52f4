"""Generates tests/golden/golden.npz: small seeded inputs + the REFERENCE'S
outputs on them.  The NFFT / graph-operator / Lanczos fixtures come from
oracle/_ref/libfgsref.so -- the reference's own nfft.cpp, kernels.cpp,
fastsum.cpp, graphop.cpp and spectral.cpp compiled unchanged against the
shim Eigen/FFTW headers (oracle/build_ref.sh); inputs come from the oracle's
seeded generators; the kernel-coefficient fixtures from the oracle (pinned
bitwise to the reference by tests/test_ref_pin.py).  The CPU suite checks
that both the oracle and the reference binary reproduce them bit for bit,
the GPU suite checks the B200 path against them at the north-star
tolerances.

    python tests/golden/make_golden.py
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import oracle as orc  # noqa: E402
from oracle import ref  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.npz")


def main():
    orc.build()
    if not ref.available():
        raise SystemExit("oracle/_ref is not built: bash oracle/build_ref.sh")
    g = {}
    # NFFT (nfft.cpp), d = 1..3, m = 4 and 8
    for d in (1, 2, 3):
        for m in (4, 8):
            n = 60 if d == 3 else 150
            nodes = orc.random_nodes(n, d, 10 * d + m)
            N = 8
            plan = ref.NfftPlan(d, N, m, nodes)
            f = orc.random_coeffs(N ** d, 3 + d)
            x = orc.random_coeffs(n, 5 + d)
            key = f"nfft_d{d}_m{m}"
            g[key + "_nodes"] = nodes
            g[key + "_fhat"] = f
            g[key + "_x"] = x
            g[key + "_forward"] = plan.forward(f)
            g[key + "_adjoint"] = plan.adjoint(x)
    # kernel coefficients (kernels.cpp:266-335), eps_b > 0 and = 0
    for fam, shape, eps, p, d, N in [(0, 0.3, 0.0, 4, 3, 8), (3, 0.6, 0.125, 3, 1, 16), (2, 1.2, 0.1, 5, 2, 8)]:
        g[f"coef_f{fam}_d{d}_N{N}"] = orc.kernel_coefficients(fam, shape, eps, p, d, N)
    # fastsum + graph operator on a config-1-like cloud (graphop.cpp:36-103)
    rng = np.random.default_rng(11)
    for d, n, sigma, N, m in [(3, 400, 0.35, 32, 4), (2, 500, 0.05, 64, 6)]:
        dirs = rng.standard_normal((n, d))
        X = 0.2 * dirs / np.linalg.norm(dirs, axis=1)[:, None] * rng.uniform(0, 1, (n, 1)) ** (1.0 / d)
        x = rng.standard_normal(n)
        op = ref.AdjacencyOperator(X, 0, sigma, N=N, m=m, p=m)
        key = f"graph_d{d}"
        g[key + "_nodes"] = X
        g[key + "_x"] = x
        g[key + "_params"] = np.array([sigma, N, m])
        g[key + "_degrees"] = op.degrees()
        g[key + "_normalized"] = op.apply_normalized(x)
        g[key + "_laplacian"] = op.apply_sym_laplacian(x)
        vals, vecs, it, conv = op.lanczos_largest(4, tol=1e-10)
        g[key + "_lanczos_values"] = vals
        g[key + "_lanczos_vectors"] = vecs
    np.savez_compressed(OUT, **g)
    print(OUT, os.path.getsize(OUT), "bytes,", len(g), "arrays")


if __name__ == "__main__":
    main()
