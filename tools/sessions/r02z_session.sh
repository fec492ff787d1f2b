# SPLITM v2 (restarted prefixes in place, stage released early): parity + A/B
O=gpurun_out/r02z; mkdir -p $O
timeout 900 python -m pytest tests/test_parity_signed_gpu.py -x -q -p no:cacheprovider -k "scan" > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest.log
PROBE_AB=TC_SPLITM timeout 600 python tools/probe_modes.py scan > $O/probe.log 2>&1; echo "probe rc=$?"; head -34 $O/probe.log | tail -26
