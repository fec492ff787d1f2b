# branch-free SPLIT outputs, fused BN finish: parity + probes
O=gpurun_out/r02p; mkdir -p $O
timeout 900 python -m pytest tests/test_parity_signed_gpu.py tests/test_batchnorm_gpu.py -x -q -p no:cacheprovider > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -15 $O/pytest.log
timeout 600 python tools/probe_modes.py scan bn > $O/probe.log 2>&1; echo "probe rc=$?"; cat $O/probe.log
