# A/B of runtime env settings on one box: VARIANTS="label=ENV=val ENV2=val;label2=..." (2 reps)
IFS=';' read -ra VS <<< "$VARIANTS"
for rep in 1 2; do
for v in "${VS[@]}"; do
  lab="${v%%=*}"; envs="${v#*=}"
  env $envs timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-joint --e2e-iters 20 > gpurun_out/ab_$lab.json 2>gpurun_out/ab_$lab.err
  python -c "import json; d=json.loads(open('gpurun_out/ab_$lab.json').read().strip().splitlines()[-1]); print('$lab', d['value'], d['e2e']['value'], d['ms_per_step'])" || tail -5 gpurun_out/ab_$lab.err
done
done
