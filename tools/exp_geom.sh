# pose-only K4b register budget: 2 / 3 / 4 CTAs per SM
for mb in 2 3 4; do
  GSB_NVCC_EXTRA="-DGSB_GEOM_POSE_MIN_BLOCKS=$mb" python paper_2410_08743_b200/build.py --force > /dev/null
  timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-joint --e2e-iters 20 > gpurun_out/bg_$mb.json 2>gpurun_out/bg_$mb.err
  python -c "import json; d=json.loads(open('gpurun_out/bg_$mb.json').read().strip().splitlines()[-1]); print('mb=$mb', d['value'], d['ms_per_step'], d['stages_ms_per_iter']['bwd_geom'])"
done
