# K2 counting-sort chunk size sweep (rebuilds in place)
for c in 1024 2048 4096; do
  GSB_NVCC_EXTRA="-DGSB_BIN_CHUNK=$c" python paper_2410_08743_b200/build.py --force > /dev/null
  timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-joint --e2e-iters 20 > gpurun_out/bc_$c.json 2>gpurun_out/bc_$c.err
  python -c "import json; d=json.loads(open('gpurun_out/bc_$c.json').read().strip().splitlines()[-1]); print('chunk=$c', d['value'], d['ms_per_step'], d['stages_ms_per_iter'])"
done
python paper_2410_08743_b200/build.py --force > /dev/null
python -m pytest tests -m gpu -x -q -p no:faulthandler 2>&1 | tail -2
