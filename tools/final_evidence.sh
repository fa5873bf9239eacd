# End-of-round evidence: GPU suite, sanitizers, default bench + reference arm, launch list, ncu --set full.
TAG=${TAG:-r2final}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_$TAG.txt 2>&1; tail -1 gpurun_out/smoke_$TAG.txt
timeout 2400 python -m pytest tests -m gpu -q -rfE -p no:cacheprovider > gpurun_out/pytest_gpu_$TAG.txt 2>&1; tail -4 gpurun_out/pytest_gpu_$TAG.txt
TOOLS="memcheck racecheck synccheck initcheck" bash tools/sanitize.sh
timeout 1200 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; python -c "
import json; d=json.loads(open('gpurun_out/bench_$TAG.json').read().strip().splitlines()[-1]); print(d['value'], d['e2e']['value'], d['stages_ms_per_iter'], d['roofline']['frac'], d.get('c3_job_1gpu',{}).get('iters_per_s'), d['clocks'])"
timeout 1200 python bench.py --impl reference > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref_$TAG.err; tail -c 300 gpurun_out/bench_ref_$TAG.json
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_batch_$TAG.csv python tools/prof_batch.py 3 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/launches_batch_$TAG.csv | head -22
timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:"backward_raster|composite_kernel|backward_geom|loss_maps|loss_grad|tile_sort_small|tile_scatter|tile_count|scan_onepass" \
  -s 24 -c 9 -o gpurun_out/prof_${TAG}_iter python tools/prof_iter.py 3 > gpurun_out/prof_${TAG}_iter.log 2>&1
tail -1 gpurun_out/prof_${TAG}_iter.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:preprocess -s 8 -c 1 \
  -o gpurun_out/prof_${TAG}_k1multi python tools/prof_batch.py 1 > gpurun_out/prof_${TAG}_k1.log 2>&1
tail -1 gpurun_out/prof_${TAG}_k1.log
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/launches_joint_$TAG.csv python tools/prof_joint.py 6 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/launches_joint_$TAG.csv | head -40
