mkdir -p gpurun_out/r02c
timeout 600 python tools/probe_modes.py reduce bn > gpurun_out/r02c/probe.log 2>&1; echo "probe rc=$?"
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -rf --timeout 1500 -s > gpurun_out/r02c/pytest.log 2>&1; echo "pytest rc=$?"; grep -E "passed|failed|^FAILED" gpurun_out/r02c/pytest.log | tail -20
timeout 900 python tools/run_reference_tests.py > gpurun_out/r02c/reftests.log 2>&1; echo "reftests rc=$?"; tail -30 gpurun_out/r02c/reftests.log
