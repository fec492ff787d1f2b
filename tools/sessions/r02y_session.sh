# SPLITM (9 <= s < 64 scans) parity + A/B vs ROWSEG/GENERAL; sanitizers over every mode
O=gpurun_out/r02y; mkdir -p $O
timeout 900 python -m pytest tests/test_parity_signed_gpu.py tests/test_parity_gpu.py -x -q -p no:cacheprovider -k "scan" > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest.log
PROBE_AB=TC_SPLITM timeout 600 python tools/probe_modes.py scan > $O/probe.log 2>&1; echo "probe rc=$?"; head -40 $O/probe.log
SAN_TIMEOUT=400 timeout 3000 tools/sanitize.sh $O/sanitize quick "memcheck racecheck synccheck initcheck" "reduce scan chunk irreg bn"
