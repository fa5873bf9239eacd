set -x
for v in onepass legacy; do
  GSB_HIST_SCAN=$v timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/b_$v.json 2>gpurun_out/b_$v.err
  python -c "import json; d=json.loads(open('gpurun_out/b_$v.json').read().strip().splitlines()[-1]); print('$v', d['value'], d['e2e']['value'], d['stages_ms_per_iter'])"
done
GSB_HIST_SCAN=onepass timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python tools/prof_iter.py 3 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/launches.csv | head -45
