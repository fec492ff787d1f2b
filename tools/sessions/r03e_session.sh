# final-code check: full GPU tests, smoke, bench + reference arm, ROWSEG probe with the shipped rule
O=gpurun_out/r03e; mkdir -p $O
bash tools/gpu_session.sh r03e test bench
PROBE_SIZES=3,5,7,9,12,17,20,24,33,40,49,63,65,100,300 PROBE_AB_R=TC_PROBE_NOP PROBE_AB_VALS=x timeout 600 python tools/probe_modes.py reduce > $O/probe_reduce.log 2>&1; echo "probe rc=$?"
PROBE_SCAN_SIZES=3,5,6,7,9,10,17,33,34,63 PROBE_AB=TC_PROBE_NOP PROBE_AB_VALS=x timeout 600 python tools/probe_modes.py scan > $O/probe_scan.log 2>&1; echo "probe rc=$?"
