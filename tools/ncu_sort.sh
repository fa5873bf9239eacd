for k in tile_sort_large_kernel tile_sort_small_kernel tile_scatter_kernel; do
timeout 600 ncu --set full --import-source on --clock-control none -k regex:$k -s 1 -c 1 -o gpurun_out/r1e_$k python tools/prof_iter.py 2 > gpurun_out/ncu_$k.log 2>&1
done
ls -la gpurun_out/*.ncu-rep | tail -3
