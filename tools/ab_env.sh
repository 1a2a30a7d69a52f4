# A/B of env settings on the C2 bench: bash tools/ab_env.sh "ENV1" "ENV2" ...
mkdir -p gpurun_out
for r in 1 2; do for v in "$@"; do
env $v python bench.py --steps 200 --warmup 10 --no-lanczos --no-cpu --also "" ${BENCH_ARGS} 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']['stage_ms_per_step']; print('$v', round(d['value']), round(d['e2e']['value']), {k:round(v*1000,1) for k,v in r.items()})" >> gpurun_out/abenv.txt
done; done
