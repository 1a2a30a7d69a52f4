set -e
L=paper_1808_04580_b200/libfgs_b200.so
mkdir -p gpurun_out
for r in 1 2; do for v in A B; do
cp ab/lib$v.so $L
python bench.py --steps 200 --warmup 10 --no-lanczos --no-cpu --also "" 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']['stage_ms_per_step']; print('$v', round(d['value']), round(d['e2e']['value']), {k:round(v*1000,1) for k,v in r.items()})" >> gpurun_out/ab.txt
done; done
cp ab/libB.so $L
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gt.txt 2>&1 || true
tail -3 gpurun_out/gt.txt
