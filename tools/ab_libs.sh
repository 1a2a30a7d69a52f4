# A/B two prebuilt libraries (ab/libA.so, ab/libB.so) on a bench config:
#   BENCH_ARGS="--config 4" bash tools/ab_libs.sh
L=paper_1808_04580_b200/libfgs_b200.so
mkdir -p gpurun_out
cp $L ab/lib_orig.so
for r in 1 2; do for v in ${LIBS:-A B}; do
cp ab/lib$v.so $L
python bench.py --steps ${STEPS:-50} --warmup 5 --no-lanczos --no-cpu --also "" ${BENCH_ARGS} 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']['stage_ms_per_step']; print('$v', round(d['value'],1), round(d['e2e']['value'],1), {k:round(v*1000,1) for k,v in r.items()})" >> gpurun_out/ablib.txt
done; done
cp ab/lib_orig.so $L
