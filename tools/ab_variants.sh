# A/B of build-knob variants of the working tree against .ab_base (tools/ab_git.sh prep) on ONE box.
# VARIANTS="label=-DKNOB=1 -DKNOB2=2;label2=..."  (each built into .ab_<label>/, 2 reps, pose batch line)
set -u
mkdir -p gpurun_out
IFS=';' read -ra VS <<< "$VARIANTS"
labs="base"
declare -A FL; FL[base]=""
for v in "${VS[@]}"; do
  lab="${v%%=*}"; flags="${v#*=}"
  rm -rf .ab_$lab && mkdir -p .ab_$lab
  tar --exclude='./.ab_*' --exclude='./gpurun_out' -cf - . | tar -xf - -C .ab_$lab
  (cd .ab_$lab && GSB_NVCC_EXTRA="$flags" python paper_2410_08743_b200/build.py --force > /dev/null) || echo "build $lab failed"
  labs="$labs $lab"; FL[$lab]="$flags"
done
for rep in 1 2; do
  for lab in $labs; do
    (cd .ab_$lab && GSB_NVCC_EXTRA="${FL[$lab]}" timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-joint --e2e-iters 20) > gpurun_out/abv_$lab.json 2> gpurun_out/abv_$lab.err
    python -c "import json; d=json.loads(open('gpurun_out/abv_$lab.json').read().strip().splitlines()[-1]); print('$lab', d['value'], d['e2e']['value'], d['ms_per_step'], d['stages_ms_per_iter'], d['pose_check']['final_loss'])" || tail -5 gpurun_out/abv_$lab.err
  done
done
