mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.txt 2>&1; tail -1 gpurun_out/smoke.txt
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dropin.py tests/test_bootstrap.py -m gpu -q -rfE -p no:cacheprovider > gpurun_out/pytest_hits.txt 2>&1; tail -8 gpurun_out/pytest_hits.txt
timeout 600 compute-sanitizer --tool memcheck --error-exitcode 17 python tools/sanitize_driver.py > gpurun_out/san_mem_hits.log 2>&1; echo memcheck rc=$?; tail -2 gpurun_out/san_mem_hits.log
timeout 600 compute-sanitizer --tool racecheck --error-exitcode 17 python tools/sanitize_driver.py > gpurun_out/san_race_hits.log 2>&1; echo racecheck rc=$?; tail -2 gpurun_out/san_race_hits.log
VARIANTS="hits=;nohits=-DGSB_BWD_HITS=0" bash tools/ab.sh
