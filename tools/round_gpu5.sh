# A/B of compile-time variants + runtime env + the C5-shaped one-GPU joint run
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
if [ -n "$VARIANTS" ]; then VARIANTS="$VARIANTS" bash tools/ab.sh; fi
for bv in 8 16; do
  GSB_POSE_BATCH_VIEWS=$bv timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-joint --no-work-counts --e2e-iters 20 > gpurun_out/c3job_$bv.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/c3job_$bv.json').read().strip().splitlines()[-1]); print('batch_views', $bv, d['c3_job_1gpu']['iters_per_s'], d['c3_job_1gpu']['views_per_s'])"
done
if [ "${C5:-1}" = 1 ]; then timeout 1500 python tools/run_c5.py 404 > gpurun_out/c5_1gpu.json 2> gpurun_out/c5_1gpu.err; tail -c 1500 gpurun_out/c5_1gpu.json; fi
