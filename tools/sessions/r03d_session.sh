# ROWSEG input views: (L2 promotion, load eviction policy) 4-way; GENERAL GR=64 reduce at 2 vs 3 CTAs/SM
O=gpurun_out/r03d; mkdir -p $O
export PROBE_MULTI_VARS=TC_RS_PROMO,TC_RS_EVICT
V="TC_RS_PROMO=256:TC_RS_EVICT=0,TC_RS_PROMO=0:TC_RS_EVICT=0,TC_RS_PROMO=256:TC_RS_EVICT=1,TC_RS_PROMO=0:TC_RS_EVICT=1"
timeout 900 python -m pytest tests/test_parity_signed_gpu.py -x -q -p no:cacheprovider -k "reduce" > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest.log
PROBE_SIZES=3,5,7,9,12,17,20,24,33,40,49,63,65,100,300 PROBE_AB_R=multi PROBE_AB_VALS=$V timeout 900 python tools/probe_modes.py reduce > $O/probe_reduce4.log 2>&1; echo "probe rc=$?"
PROBE_SCAN_SIZES=3,5,6,7,9,10,17,33,34 PROBE_AB=multi PROBE_AB_VALS=$V timeout 900 python tools/probe_modes.py scan > $O/probe_scan4.log 2>&1; echo "probe rc=$?"
PROBE_SIZES=127,129,1001,4097,100001 PROBE_AB_R=TC_CTAS_PER_SM PROBE_AB_VALS=2,3 timeout 900 python tools/probe_modes.py reduce > $O/probe_cps.log 2>&1; echo "probe rc=$?"; cat $O/probe_cps.log
