mkdir -p gpurun_out/r02d
(free -g; nproc; nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv) > gpurun_out/r02d/box.txt 2>&1
timeout 600 python tools/probe_modes.py > gpurun_out/r02d/probe.log 2>&1; echo "probe rc=$?"
timeout 2700 python -m pytest tests -m gpu -q -p no:cacheprovider -rf --timeout 1500 > gpurun_out/r02d/pytest.log 2>&1; echo "pytest rc=$?"; grep -E "passed|failed|^FAILED|^ERROR" gpurun_out/r02d/pytest.log | tail -30
timeout 300 python -c 'import __graft_entry__ as g; g.smoke()' > gpurun_out/r02d/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/r02d/smoke.log
timeout 900 python bench.py > gpurun_out/r02d/bench.json 2> gpurun_out/r02d/bench.err; echo "bench rc=$?"; tail -c 1500 gpurun_out/r02d/bench.json; tail -5 gpurun_out/r02d/bench.err
timeout 900 python tools/run_reference_tests.py > gpurun_out/r02d/reftests.log 2>&1; echo "reftests rc=$?"; tail -30 gpurun_out/r02d/reftests.log
