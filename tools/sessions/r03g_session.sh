# SPLIT reduce (granules of 8, split granule from the SMEM stage) for s > 64 with gcd(s, 64) <= 4:
# parity, then A/B against GENERAL with one-element granules; ROWSEG tie-break A/B
O=gpurun_out/r03g; mkdir -p $O
timeout 900 python -m pytest tests/test_parity_signed_gpu.py tests/test_parity_gpu.py -x -q -p no:cacheprovider -k "reduce or general or c_abi or bf16" > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -15 $O/pytest.log
PROBE_SIZES=65,66,100,127,129,130,300,1001,4097,100001,524291,1000003 PROBE_AB_R=TC_SPLIT_REDUCE PROBE_AB_VALS=1,0 timeout 600 python tools/probe_modes.py reduce > $O/probe_split_reduce.log 2>&1; echo "probe rc=$?"; cat $O/probe_split_reduce.log
PROBE_SIZES=3,5,7,9,11,13,15 PROBE_AB_R=TC_RS_TIE PROBE_AB_VALS=0,1 timeout 600 python tools/probe_modes.py reduce > $O/probe_tie.log 2>&1; echo "probe rc=$?"; cat $O/probe_tie.log
