#!/usr/bin/env bash
# One gpurun call: ncu --set full of the config-5 spread / interpolation
# kernels (first 16-vector launch of each).  usage: bash tools/gpu_ncu.sh <tag> [regex] [skip] [count] [bench args]
set -x
tag=${1:-r02}
rx=${2:-"spread_v5_kernel|interp_v5_kernel"}
skip=${3:-2}
cnt=${4:-2}
[ $# -ge 4 ] && shift 4 || set --
mkdir -p gpurun_out
short="python bench.py --steps 2 --warmup 3 --no-cpu --no-lanczos --also= --no-e2e $@"
$short > gpurun_out/${tag}_plain.log 2>&1 &&
ncu --set full --import-source on --clock-control none -k regex:"$rx" \
  -s $skip -c $cnt -o gpurun_out/${tag} -f $short > gpurun_out/${tag}_ncu_full.log 2>&1
echo rc=$?
