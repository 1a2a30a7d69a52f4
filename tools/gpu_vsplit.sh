#!/usr/bin/env bash
# config-5 stage times for several vector splits of the slot-layout kernels
# (FGS_VSPLIT CTAs per item), then the dense-cell and full-size parity tests
# at the chosen split.  usage: bash tools/gpu_vsplit.sh <tag> [splits...]
tag=${1:-vs}
shift || true
mkdir -p gpurun_out
for vs in "$@"; do
  echo "== FGS_VSPLIT=$vs" >> gpurun_out/${tag}_var.txt
  FGS_VSPLIT=$vs timeout 600 python tools/variant_bench.py 5 base >> gpurun_out/${tag}_var.txt 2>&1
done
cat gpurun_out/${tag}_var.txt
