#!/usr/bin/env bash
# quick GPU check of the config-5 path: dense-cell parity, per-stage timing,
# full-size config-5 parity.  usage: bash tools/gpu_quick.sh <tag> [variant tags...]
tag=${1:-q}
shift || true
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_fullsize_parity.py -k "dense_cells" -x -q > gpurun_out/${tag}_dense.txt 2>&1
echo "dense rc=$?" >> gpurun_out/${tag}_dense.txt
timeout 600 python tools/variant_bench.py 5 base "$@" > gpurun_out/${tag}_var.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_fullsize_parity.py -k "config5" -x -q > gpurun_out/${tag}_c5.txt 2>&1
echo "c5 rc=$?" >> gpurun_out/${tag}_c5.txt
