# ROWSEG input views: L2 promotion none vs 256 B, evict-normal vs evict-first (A/B)
O=gpurun_out/r03c; mkdir -p $O
timeout 900 python -m pytest tests/test_parity_signed_gpu.py tests/test_parity_gpu.py -x -q -p no:cacheprovider -k "scan or reduce or bf16 or general or c_abi" > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest.log
PROBE_AB=TC_RS_PROMO timeout 900 python tools/probe_modes.py scan > $O/probe_promo_scan.log 2>&1; echo "probe rc=$?"; head -22 $O/probe_promo_scan.log
PROBE_AB=TC_RS_EVICT timeout 900 python tools/probe_modes.py scan > $O/probe_evict_scan.log 2>&1; echo "probe rc=$?"; head -22 $O/probe_evict_scan.log
PROBE_AB_R=TC_RS_EVICT timeout 900 python tools/probe_modes.py reduce > $O/probe_evict_reduce.log 2>&1; echo "probe rc=$?"; head -40 $O/probe_evict_reduce.log
PROBE_AB_R=TC_RS_PROMO timeout 900 python tools/probe_modes.py reduce > $O/probe_promo_reduce.log 2>&1; echo "probe rc=$?"; head -40 $O/probe_promo_reduce.log
