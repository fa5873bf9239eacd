# A/B of the working tree against a git ref on ONE box.
# Here:   bash tools/ab_git.sh prep [REF]   (exports REF into .ab_base/ and builds it there)
# On box: bash tools/ab_git.sh run          (alternates base / head bench lines, 2 reps)
set -u
if [ "${1:-}" = "prep" ]; then
  rm -rf .ab_base && mkdir -p .ab_base
  git archive "${2:-HEAD}" | tar -x -C .ab_base
  (cd .ab_base && python paper_2410_08743_b200/build.py > /dev/null)
  exit $?
fi
mkdir -p gpurun_out
if [ "${1:-}" = "runj" ]; then  # the C4 joint step: ms per step and the final loss (must match bitwise)
  for rep in 1 2; do
    for side in base head; do
      dir=.; [ $side = base ] && dir=.ab_base
      (cd $dir && timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-iters 8) > gpurun_out/abj_$side.json 2> gpurun_out/abj_$side.err
      python -c "import json; d=json.loads(open('gpurun_out/abj_$side.json').read().strip().splitlines()[-1]); j=d['joint_c4']; print('$side', j['ms_per_step'], repr(j['final_total_loss']))" || tail -5 gpurun_out/abj_$side.err
    done
  done
  exit 0
fi
for rep in 1 2; do
  for side in base head; do
    dir=.; [ $side = base ] && dir=.ab_base
    (cd $dir && timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-joint --e2e-iters 20) > gpurun_out/ab_$side.json 2> gpurun_out/ab_$side.err
    python -c "import json; d=json.loads(open('gpurun_out/ab_$side.json').read().strip().splitlines()[-1]); print('$side', d['value'], d['e2e']['value'], d['ms_per_step'], d['stages_ms_per_iter'])" || tail -5 gpurun_out/ab_$side.err
  done
done
