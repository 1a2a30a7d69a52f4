timeout 900 python -m pytest tests/test_gpu_shard_group.py -x -q > gpurun_out/r02m_group.txt 2>&1
for w in 8; do timeout 600 python bench.py --config 5 --emulate $w --steps 3 --warmup 1 >> gpurun_out/r02m_emu.jsonl 2>>gpurun_out/r02m_emu.err; done
timeout 300 python bench.py --config 4 --emulate 8 --steps 10 --warmup 2 >> gpurun_out/r02m_emu.jsonl 2>>gpurun_out/r02m_emu.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02m_c4emu_launches.csv python bench.py --config 4 --emulate 8 --steps 1 --warmup 1 > /dev/null 2>&1
