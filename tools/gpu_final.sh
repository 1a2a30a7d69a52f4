#!/usr/bin/env bash
# Round-end evidence in one gpurun call: GPU suite, smoke, default bench line
# (config 5 + also legs), launch list, ncu of the config-5 kernels, emulated
# N-rank projections.  usage: bash tools/gpu_final.sh <tag>
tag=${1:-r02z}
bash tools/gpu_r02.sh $tag
for w in 2 4 8; do timeout 600 python bench.py --config 5 --emulate $w --steps 3 --warmup 1 >> gpurun_out/${tag}_emu.jsonl 2>>gpurun_out/${tag}_emu.err; done
for w in 2 4 8; do timeout 600 python bench.py --config 5 --weak --emulate $w --steps 3 --warmup 1 >> gpurun_out/${tag}_emu.jsonl 2>>gpurun_out/${tag}_emu.err; done
for w in 2 4 8; do timeout 300 python bench.py --config 4 --emulate $w --steps 10 --warmup 2 >> gpurun_out/${tag}_emu.jsonl 2>>gpurun_out/${tag}_emu.err; done
echo final-done
