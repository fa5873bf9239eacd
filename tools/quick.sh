# quick A/B: GPU parity tests (optionally filtered) + short bench line (one gpurun call)
python -m pytest tests/test_gpu_parity.py -m gpu -q -x ${PYTEST_K:+-k "$PYTEST_K"} 2>&1 | tail -3
for i in 1 2; do
timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-joint --e2e-iters 20 > gpurun_out/q.json 2>gpurun_out/q.err
python -c "import json; d=json.loads(open('gpurun_out/q.json').read().strip().splitlines()[-1]); print(d['value'], d['e2e']['value'], d['ms_per_step'], d['stages_ms_per_iter'])"
done
