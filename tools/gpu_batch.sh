# GPU tests + bench (pose batch) + e2e probe with debug events
python -m pytest tests -m gpu -q -x 2>&1 | tail -15
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/b.json 2>gpurun_out/b.err
tail -3 gpurun_out/b.err
python -c "import json; d=json.loads(open('gpurun_out/b.json').read().strip().splitlines()[-1]); print(d['value'], d['e2e']['value'], d['ms_per_step'], d['stages_ms_per_iter'], d.get('scene'))"
GSB_DEBUG=1 timeout 300 python tools/e2e_probe.py > gpurun_out/e2e_probe.log 2>&1; tail -30 gpurun_out/e2e_probe.log
