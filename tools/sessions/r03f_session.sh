# (1) ROWSEG (with the new L2 rule) vs SPLITM/GENERAL for odd s scans, both outputs;
# (2) CHUNK unit size K for fp16- and fp32-output full / huge-segment scans
O=gpurun_out/r03f; mkdir -p $O
PROBE_SCAN_SIZES=11,13,15,17,21,25,33,49,63 PROBE_AB=TC_RSS_ALL PROBE_AB_VALS=1,0 timeout 600 python tools/probe_modes.py scan > $O/probe_rss_all.log 2>&1; echo "probe rc=$?"; cat $O/probe_rss_all.log
for k in 1 2 3 4; do
  echo "K=$k"; TC_CHUNK_TILES=$k timeout 300 python tools/probe_sizes.py scan 1073741824 524291 2>&1 | sed 's/^/   /'
done > $O/chunk_k.log; cat $O/chunk_k.log
