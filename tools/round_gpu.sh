# One gpurun call: GPU tests, default bench, reference arm, launch list of one
# pose iteration. Usage: TAG=r2a bash tools/round_gpu.sh   (outputs gpurun_out/*_$TAG*)
TAG=${TAG:-r2}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu_$TAG.txt 2>&1
nproc >> gpurun_out/gpu_$TAG.txt; grep -m1 "model name" /proc/cpuinfo >> gpurun_out/gpu_$TAG.txt
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_$TAG.txt 2>&1; tail -2 gpurun_out/smoke_$TAG.txt
if [ "${TESTS:-1}" = 1 ]; then
timeout 1800 python -m pytest tests -m gpu -q -x ${PYTEST_ARGS:-} > gpurun_out/pytest_gpu_$TAG.txt 2>&1; tail -15 gpurun_out/pytest_gpu_$TAG.txt
fi
timeout 1200 python bench.py ${BENCH_ARGS:-} > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; tail -c 3000 gpurun_out/bench_$TAG.json; tail -5 gpurun_out/bench_$TAG.err
if [ "${REF:-1}" = 1 ]; then
timeout 900 python bench.py --impl reference --steps ${REF_STEPS:-10} --warmup 1 > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref_$TAG.err; tail -c 400 gpurun_out/bench_ref_$TAG.json
fi
if [ "${LAUNCHES:-1}" = 1 ]; then
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_batch_$TAG.csv python tools/prof_batch.py 3 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/launches_batch_$TAG.csv | head -30
fi
if [ "${DROPIN:-1}" = 1 ] && [ -x integration/_build/acceptance_b200 ]; then
  for c in 2 3 4 7 8; do timeout 900 integration/_build/acceptance_b200 $c > gpurun_out/dropin_acc_$c.txt 2>&1; tail -1 gpurun_out/dropin_acc_$c.txt; done
  for t in test_rasterizer test_trainer test_losses test_scene; do timeout 900 integration/_build/${t}_b200 > gpurun_out/dropin_$t.txt 2>&1; tail -3 gpurun_out/dropin_$t.txt; done
fi
