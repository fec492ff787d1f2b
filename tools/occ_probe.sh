ncu --metrics launch__grid_size,gpu__time_duration.sum --clock-control none -c 30 --csv python tools/perf_probe.py reduce 2>/dev/null | grep -E "seg_kernel" | awk -F'","' '{print $5, $NF}' | head -12
python tools/perf_probe.py reduce 2>&1 | grep float16
TC_CTAS_PER_SM=1 python tools/perf_probe.py reduce 2>&1 | grep float16
python tools/perf_probe.py scan 2>&1 | tail -20
