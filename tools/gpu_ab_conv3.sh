timeout 600 python -m pytest tests/test_gpu_shard_group.py tests/test_gpu_fullsize.py -x -q -k "shard_group_equals or full_size_apply" > gpurun_out/r02ad_t.txt 2>&1; echo rc=$? >> gpurun_out/r02ad_t.txt
for c in 5 4; do timeout 300 python tools/variant_bench.py $c base >> gpurun_out/r02ad_var.txt 2>&1; FGS_CONV3_WIDE=0 timeout 300 python tools/variant_bench.py $c base >> gpurun_out/r02ad_var.txt 2>&1; done
python tools/group_stages.py 4 8 > gpurun_out/r02ad_stages.txt 2>&1
FGS_CONV3_WIDE=0 python tools/group_stages.py 4 8 >> gpurun_out/r02ad_stages.txt 2>&1
