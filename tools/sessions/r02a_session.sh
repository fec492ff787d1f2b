mkdir -p gpurun_out/r02a
(free -g; nproc; nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv) > gpurun_out/r02a/box.txt 2>&1
timeout 600 python tools/probe_modes.py > gpurun_out/r02a/probe.log 2>&1; echo "probe rc=$?"
timeout 2700 python -m pytest tests -m gpu -q -p no:cacheprovider -rf --timeout 1500 -s > gpurun_out/r02a/pytest.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/r02a/pytest.log
SAN_TIMEOUT=300 timeout 2400 tools/sanitize.sh gpurun_out/r02a/san quick
