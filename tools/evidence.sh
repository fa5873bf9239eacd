# Full evidence run for profiles/: GPU tests, default bench, reference arm,
# launch lists and ncu --set full captures. Usage: TAG=r1b bash tools/evidence.sh
TAG=${TAG:-r1}
mkdir -p gpurun_out
python -m pytest tests -m gpu -q 2>&1 | tail -4 > gpurun_out/pytest_gpu_$TAG.txt; cat gpurun_out/pytest_gpu_$TAG.txt
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; tail -c 600 gpurun_out/bench_$TAG.json
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref_$TAG.err; tail -c 300 gpurun_out/bench_ref_$TAG.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_iter_$TAG.csv python tools/prof_iter.py 3 > /dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_batch_$TAG.csv python tools/prof_batch.py 3 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/launches_batch_$TAG.csv | head -24
timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:"backward_raster|composite_kernel|backward_geom|loss_maps|loss_grad|tile_sort_large|tile_scatter|tile_sort_small|tile_count" \
  -s 20 -c 9 -o gpurun_out/prof_${TAG}_iter python tools/prof_iter.py 3 > gpurun_out/prof_${TAG}_iter.log 2>&1
tail -1 gpurun_out/prof_${TAG}_iter.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:preprocess -s 8 -c 1 \
  -o gpurun_out/prof_${TAG}_k1multi python tools/prof_batch.py 1 > gpurun_out/prof_${TAG}_k1.log 2>&1
tail -1 gpurun_out/prof_${TAG}_k1.log
