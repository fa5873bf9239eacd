# A/B of compile-time variants on one box: VARIANTS="label=flags;label=flags" (flags -> GSB_NVCC_EXTRA)
IFS=';' read -ra VS <<< "$VARIANTS"
for rep in 1 2; do
for v in "${VS[@]}"; do
  lab="${v%%=*}"; fl="${v#*=}"
  GSB_NVCC_EXTRA="$fl" python paper_2410_08743_b200/build.py --force > /dev/null 2>gpurun_out/build_$lab.err || { echo "build $lab failed"; tail -5 gpurun_out/build_$lab.err; continue; }
  timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-joint --e2e-iters 20 > gpurun_out/ab_$lab.json 2>gpurun_out/ab_$lab.err
  python -c "import json; d=json.loads(open('gpurun_out/ab_$lab.json').read().strip().splitlines()[-1]); print('$lab', d['value'], d['ms_per_step'], d['stages_ms_per_iter'])" || tail -5 gpurun_out/ab_$lab.err
done
done
python paper_2410_08743_b200/build.py --force > /dev/null
