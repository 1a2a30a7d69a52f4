#!/usr/bin/env bash
# quick GPU A/B of an env switch on config 5 and 4 + dense / C5 parity.
# usage: bash tools/gpu_quick2.sh <tag> <ENV=VAL for the B side>
tag=$1; envb=$2
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_fullsize_parity.py -k "dense_cells" -x -q > gpurun_out/${tag}_dense.txt 2>&1
echo "dense rc=$?" >> gpurun_out/${tag}_dense.txt
for c in 5 4; do
  timeout 300 python tools/variant_bench.py $c base >> gpurun_out/${tag}_var.txt 2>&1
  env $envb timeout 300 python tools/variant_bench.py $c base >> gpurun_out/${tag}_var.txt 2>&1
done
timeout 600 python -m pytest tests/test_gpu_fullsize_parity.py -k "config5" -x -q > gpurun_out/${tag}_c5.txt 2>&1
echo "c5 rc=$?" >> gpurun_out/${tag}_c5.txt
