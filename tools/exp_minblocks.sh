# backward raster register budget: CTAs/SM 5..8 (rebuilds in place)
for mb in 5 6 7 8; do
  GSB_NVCC_EXTRA="-DGSB_BWD_MIN_BLOCKS=$mb" python paper_2410_08743_b200/build.py --force > /dev/null
  timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-joint --e2e-iters 20 > gpurun_out/b_$mb.json 2>gpurun_out/b_$mb.err
  python -c "import json; d=json.loads(open('gpurun_out/b_$mb.json').read().strip().splitlines()[-1]); print('mb=$mb', d['value'], d['ms_per_step'], d['stages_ms_per_iter'])"
done
python paper_2410_08743_b200/build.py --force > /dev/null
python -m pytest tests -m gpu -x -q -p no:faulthandler 2>&1 | tail -2
