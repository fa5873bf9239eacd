# throughput vs views per GPU (pose batch width)
for v in 8 16 32 64; do
  GSB_BENCH_VIEWS_PER_GPU=$v timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-joint --e2e-iters 20 > gpurun_out/bv_$v.json 2>gpurun_out/bv_$v.err
  python -c "import json; d=json.loads(open('gpurun_out/bv_$v.json').read().strip().splitlines()[-1]); print('views=$v', d['value'], d['e2e']['value'], d['ms_per_step'])"
done
