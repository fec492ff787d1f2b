# ROWSEG L2 rule, remaining sizes: fp16 scans with many chunks per row, fp32 reduces s = 49..65 (repeated)
O=gpurun_out/r03j; mkdir -p $O
export PROBE_MULTI_VARS=TC_RS_PROMO,TC_RS_EVICT
V="TC_RS_PROMO=256:TC_RS_EVICT=0,TC_RS_PROMO=0:TC_RS_EVICT=0,TC_RS_PROMO=256:TC_RS_EVICT=1,TC_RS_PROMO=0:TC_RS_EVICT=1"
PROBE_SCAN_SIZES=11,13,15,31,47,49,63 PROBE_AB=multi PROBE_AB_VALS=$V timeout 600 python tools/probe_modes.py scan > $O/probe_scan4.log 2>&1; echo "probe rc=$?"
PROBE_SIZES=49,63,65,49,63,65,127,129 PROBE_AB_R=multi PROBE_AB_VALS=$V timeout 600 python tools/probe_modes.py reduce > $O/probe_reduce4.log 2>&1; echo "probe rc=$?"
