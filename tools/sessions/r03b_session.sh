# ROWSEG scan with two epilogue groups (fp16 out) and the L2 promotion of the
# strided row-segment views: parity, then A/B
O=gpurun_out/r03b; mkdir -p $O
timeout 900 python -m pytest tests/test_parity_signed_gpu.py tests/test_parity_gpu.py -x -q -p no:cacheprovider -k "scan or bf16 or general or c_abi" > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest.log
PROBE_AB=TC_RSS_NG timeout 900 python tools/probe_modes.py scan > $O/probe_ng.log 2>&1; echo "probe rc=$?"; head -24 $O/probe_ng.log
PROBE_AB=TC_RS_PROMO timeout 900 python tools/probe_modes.py scan > $O/probe_promo_scan.log 2>&1; echo "probe rc=$?"; head -24 $O/probe_promo_scan.log
PROBE_AB_R=TC_RS_PROMO timeout 900 python tools/probe_modes.py reduce > $O/probe_promo_reduce.log 2>&1; echo "probe rc=$?"; head -30 $O/probe_promo_reduce.log
