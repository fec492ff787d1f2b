# ROWSEG scan, fp16 out: rows of whole 32-B sectors vs the 16-B minimum (A/B)
O=gpurun_out/r03m; mkdir -p $O
PROBE_SCAN_SIZES=23,25,27,29,31,39,41,45,47,49,55,57,63 PROBE_AB=TC_RSS_ALIGN32 PROBE_AB_VALS=0,1 timeout 600 python tools/probe_modes.py scan > $O/probe_align.log 2>&1; echo "probe rc=$?"; cat $O/probe_align.log
