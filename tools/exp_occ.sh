# occupancy knobs: K1 (GSB_PRE_MIN_BLOCKS) and loss_maps (GSB_LOSS_MIN_BLOCKS)
for cfg in "-DGSB_PRE_MIN_BLOCKS=1 -DGSB_LOSS_MIN_BLOCKS=1" "-DGSB_PRE_MIN_BLOCKS=3 -DGSB_LOSS_MIN_BLOCKS=1" "-DGSB_PRE_MIN_BLOCKS=1 -DGSB_LOSS_MIN_BLOCKS=3"; do
  GSB_NVCC_EXTRA="$cfg" python paper_2410_08743_b200/build.py --force > /dev/null
  timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-joint --e2e-iters 20 > gpurun_out/bo.json 2>gpurun_out/bo.err
  python -c "import json; d=json.loads(open('gpurun_out/bo.json').read().strip().splitlines()[-1]); print('$cfg', d['value'], d['ms_per_step'], d['stages_ms_per_iter']['loss'])"
done
