mkdir -p gpurun_out/r02b
timeout 600 python tools/probe_modes.py reduce > gpurun_out/r02b/probe.log 2>&1; echo "probe rc=$?"
timeout 1500 python -m pytest tests/test_parity_gpu.py tests/test_parity_signed_gpu.py -q -p no:cacheprovider -x -rf --timeout 900 > gpurun_out/r02b/pytest.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/r02b/pytest.log
SAN_TIMEOUT=300 timeout 1200 tools/sanitize.sh gpurun_out/r02b/san quick "memcheck racecheck synccheck" "reduce"
