# tests + short bench + launch list (one gpurun call)
python -m pytest tests -m gpu -q -x 2>&1 | tail -15
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/b.json 2>gpurun_out/b.err
tail -3 gpurun_out/b.err
python -c "import json; d=json.loads(open('gpurun_out/b.json').read().strip().splitlines()[-1]); print(d['value'], d['e2e']['value'], d['ms_per_step'], d['stages_ms_per_iter'], d.get('scene'))"
if [ "${LAUNCHES:-1}" = 1 ]; then
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python tools/prof_iter.py 3 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/launches.csv | head -40
fi
