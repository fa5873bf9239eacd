# ncu --set full captures for profiles/: the per-view kernels from one
# session (tools/prof_iter.py) and the 8-view K1 from a pose batch.
timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:"backward_raster|composite_kernel|backward_geom|loss_maps|loss_grad|tile_sort_large|tile_scatter|tile_sort_small|tile_count" \
  -s 20 -c 9 -o gpurun_out/prof_r1_iter python tools/prof_iter.py 3 > gpurun_out/prof_r1_iter.log 2>&1
tail -1 gpurun_out/prof_r1_iter.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:preprocess -s 8 -c 1 \
  -o gpurun_out/prof_r1_k1multi python tools/prof_batch.py 1 > gpurun_out/prof_r1_k1.log 2>&1
tail -1 gpurun_out/prof_r1_k1.log
