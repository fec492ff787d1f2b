# SPLIT v4: raw granule from the held SMEM stage
O=gpurun_out/r02s; mkdir -p $O
timeout 900 python -m pytest tests/test_parity_signed_gpu.py -x -q -p no:cacheprovider > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest.log
PROBE_AB=TC_SPLIT timeout 600 python tools/probe_modes.py scan > $O/probe.log 2>&1; echo "probe rc=$?"; grep -v "s=  *[0-9]  *\|s=  *[1-5][0-9] " $O/probe.log
