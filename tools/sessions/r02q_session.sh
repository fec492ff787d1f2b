# SPLIT v3 (prefetched raw granule, in-place patch), BN ticket memset: parity + probes
O=gpurun_out/r02q; mkdir -p $O
timeout 900 python -m pytest tests/test_parity_signed_gpu.py tests/test_batchnorm_gpu.py -x -q -p no:cacheprovider > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -5 $O/pytest.log
PROBE_AB=TC_SPLIT timeout 600 python tools/probe_modes.py scan bn > $O/probe.log 2>&1; echo "probe rc=$?"; cat $O/probe.log
