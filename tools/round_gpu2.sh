# tests (full, no -x) + racecheck/memcheck + default bench. TAG names outputs.
TAG=${TAG:-r2}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_$TAG.txt 2>&1; tail -1 gpurun_out/smoke_$TAG.txt
timeout 2400 python -m pytest tests -m gpu -q -rfE -p no:cacheprovider > gpurun_out/pytest_gpu_full_$TAG.txt 2>&1; tail -30 gpurun_out/pytest_gpu_full_$TAG.txt
TOOLS="${SAN_TOOLS:-racecheck memcheck}" bash tools/sanitize.sh
timeout 1200 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; python -c "
import json; d=json.loads(open('gpurun_out/bench_$TAG.json').read().strip().splitlines()[-1]); print(d['value'], d['e2e']['value'], d['stages_ms_per_iter'], d['roofline']['frac'], d.get('c3_job_1gpu',{}).get('iters_per_s'))"
tail -3 gpurun_out/bench_$TAG.err
