# One gpurun call: the full -m gpu suite (no -x), compute-sanitizer over the
# sanitizer driver, ncu --set full of the per-view kernels. TAG names outputs.
TAG=${TAG:-r2}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 2400 python -m pytest tests -m gpu -q -rfE > gpurun_out/pytest_gpu_full_$TAG.txt 2>&1; tail -25 gpurun_out/pytest_gpu_full_$TAG.txt
if [ "${SAN:-1}" = 1 ]; then bash tools/sanitize.sh; fi
if [ "${PROF:-1}" = 1 ]; then
timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:"backward_raster|composite_kernel|backward_geom|loss_maps|loss_grad|tile_sort_small|tile_scatter" \
  -s 20 -c 7 -o gpurun_out/prof_${TAG}_iter python tools/prof_iter.py 3 > gpurun_out/prof_${TAG}_iter.log 2>&1
tail -1 gpurun_out/prof_${TAG}_iter.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:preprocess -s 8 -c 1 \
  -o gpurun_out/prof_${TAG}_k1multi python tools/prof_batch.py 1 > gpurun_out/prof_${TAG}_k1.log 2>&1
tail -1 gpurun_out/prof_${TAG}_k1.log
fi
