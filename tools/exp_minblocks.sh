# backward raster register budget: 6 vs 8 CTAs/SM (rebuilds in place)
python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for mb in 6 8; do
  GSB_NVCC_EXTRA="-DGSB_BWD_MIN_BLOCKS=$mb" python paper_2410_08743_b200/build.py --force > /dev/null
  timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-iters 20 > gpurun_out/b_$mb.json 2>gpurun_out/b_$mb.err
  python -c "import json; d=json.loads(open('gpurun_out/b_$mb.json').read().strip().splitlines()[-1]); print('mb=$mb', d['value'], d['e2e']['value'], d['ms_per_step'], d['stages_ms_per_iter'])"
done
