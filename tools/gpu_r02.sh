#!/usr/bin/env bash
# One gpurun call: GPU suite, default bench line (config 5), launch list and
# ncu --set full captures of the config-5 spread / interpolation kernels.
# usage: bash tools/gpu_r02.sh <tag> [pytest-args]
set -x
tag=${1:-r02}
shift || true
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q ${@} > gpurun_out/${tag}_gpu_tests.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/${tag}_gpu_tests.txt
timeout 900 python bench.py > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err
short="python bench.py --steps 2 --warmup 3 --no-cpu --no-lanczos --also= --no-e2e"
$short > gpurun_out/${tag}_plain.log 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv --log-file gpurun_out/${tag}_launches.csv $short \
  > gpurun_out/${tag}_ncu_launch.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:"spread_v6_kernel" -s 1 -c 1 \
  -o gpurun_out/${tag}_spread -f $short > gpurun_out/${tag}_ncu_spread.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:"interp_v7_kernel" -s 1 -c 1 --replay-mode application \
  -o gpurun_out/${tag}_interp -f $short > gpurun_out/${tag}_ncu_interp.log 2>&1
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/${tag}_smoke.txt 2>&1
echo done
