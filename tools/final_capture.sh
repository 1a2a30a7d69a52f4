# Round-end evidence: default bench line, C2 launch list, one full ncu
# capture of the C2 step's kernels, GPU suite and smoke.
set -x
mkdir -p gpurun_out
python bench.py > gpurun_out/final_default.json 2> gpurun_out/final_default.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/final_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-lanczos --no-cpu --also "" > gpurun_out/final_launch.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:"spread_v4_2d|interp_v4_2d|assemble_mixed|conv2_cluster" \
  -s 8 -c 4 -o gpurun_out/r01_c2_final -f python bench.py --steps 2 --warmup 3 --no-lanczos --no-cpu --also "" \
  > gpurun_out/final_ncu.log 2>&1
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/final_gpu_tests.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/final_smoke.txt 2>&1
