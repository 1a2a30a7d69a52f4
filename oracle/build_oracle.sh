#!/usr/bin/env bash
# Builds the CPU oracle (test infrastructure only) into oracle/liboracle.so.
# -ffp-contract=off mirrors the reference's default x86-64 Release build,
# which emits no fused multiply-adds (proj/CMakeLists.txt:8-10,36).
set -euo pipefail
here="$(cd "$(dirname "${BASH_SOURCE[0]}")" && pwd)"
# The seeded BASELINE workload generator (the product's workload.cpp) is
# linked in as well, so bench.py's reference arm never loads the product.
g++ -std=c++20 -O3 -ffp-contract=off -fPIC -shared -Wall -Wextra \
    -I "$here/../include" \
    -o "$here/liboracle.so" "$here/fgs_oracle.cpp" "$here/../paper_1808_04580_b200/csrc/workload.cpp"
