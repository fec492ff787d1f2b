# ROWSEG scan (fp16 out) with up to 16 chunks per row and sector-aligned rows: parity, A/B, full suite
O=gpurun_out/r03n; mkdir -p $O
timeout 900 python -m pytest tests/test_parity_signed_gpu.py tests/test_parity_gpu.py -x -q -p no:cacheprovider -k "scan or c_abi or bf16" > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest.log
PROBE_SCAN_SIZES=3,7,9,17,23,25,29,31,33,39,41,47,49,57,63 PROBE_AB=TC_RSS_ALIGN32 PROBE_AB_VALS=1,0 timeout 600 python tools/probe_modes.py scan > $O/probe_align16.log 2>&1; echo "probe rc=$?"; grep float16 $O/probe_align16.log
