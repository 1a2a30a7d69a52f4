for p in "" "1,1,1,1,1,1,1,1,1,1,1,1,1,1,1,1" "1,3,8,3,1" "1,2,4,5,2,1,1" "1,4,6,4,1" "2,4,4,4,2" "1,2,3,4,3,2,1"; do
  echo "parts=$p"
  FGS_PIPE_PARTS=$p python bench.py --steps 6 --warmup 3 --no-cpu --no-lanczos --also= 2>/dev/null | python -c "
import sys, json
j=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('  device', round(j['ms_per_step'],2), 'e2e', round(j['e2e']['ms_per_step'],2), round(j['e2e']['value'],2))"
done
timeout 600 python -m pytest tests/test_gpu_edge.py -x -q 2>&1 | tail -2
