# SPLIT reduce with pairwise trees + warp-uniform split pass: parity, A/B vs GENERAL over s;
# ROWSEG fp32-output reduce rule check
O=gpurun_out/r03k; mkdir -p $O
timeout 900 python -m pytest tests/test_parity_signed_gpu.py tests/test_parity_gpu.py -x -q -p no:cacheprovider -k "reduce or general or c_abi or bf16" > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest.log
TC_SPLIT_REDUCE=2 timeout 300 python tools/sanitize.py quick reduce > $O/plain_forced.log 2>&1; echo "plain forced rc=$?"; tail -1 $O/plain_forced.log
PROBE_SIZES=127,1001,4097,8193,12289,32769,100001 PROBE_AB_R=TC_SPLIT_REDUCE PROBE_AB_VALS=2,0 timeout 600 python tools/probe_modes.py reduce > $O/probe_split.log 2>&1; echo "probe rc=$?"; cat $O/probe_split.log
PROBE_SIZES=17,49,63,65,100 PROBE_AB_R=TC_PROBE_NOP PROBE_AB_VALS=x timeout 600 python tools/probe_modes.py reduce > $O/probe_rowseg.log 2>&1; echo "probe rc=$?"; cat $O/probe_rowseg.log
