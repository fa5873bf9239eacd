# compile-time variants (VARIANTS="label=flags;...") on the C3 batch value and the C4 joint step (2 reps)
IFS=';' read -ra VS <<< "$VARIANTS"
for rep in 1 2; do
for v in "${VS[@]}"; do
  lab="${v%%=*}"; fl="${v#*=}"
  GSB_NVCC_EXTRA="$fl" python paper_2410_08743_b200/build.py --force > /dev/null 2>gpurun_out/build_$lab.err || { echo "build $lab failed"; continue; }
  timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-iters 8 > gpurun_out/abj_$lab.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/abj_$lab.json').read().strip().splitlines()[-1]); print('$lab', d['value'], d['joint_c4']['ms_per_step'], d['joint_c4']['final_total_loss'])"
done
done
python paper_2410_08743_b200/build.py --force > /dev/null
