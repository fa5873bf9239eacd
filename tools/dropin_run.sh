# the reference's acceptance criteria and doctest suites through the adapter (integration/)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for c in 2 3 4 7 8; do timeout 900 integration/_build/acceptance_b200 $c > gpurun_out/dropin_acc_$c.txt 2>&1; tail -1 gpurun_out/dropin_acc_$c.txt; done
for t in test_rasterizer test_trainer test_losses test_scene; do timeout 900 integration/_build/${t}_b200 > gpurun_out/dropin_$t.txt 2>&1; grep "FAILED:\|test cases" gpurun_out/dropin_$t.txt; done
