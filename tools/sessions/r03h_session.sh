# SPLIT reduce: where it overtakes GENERAL (A/B over s), and ncu of s = 4097 vs 100001
O=gpurun_out/r03h; mkdir -p $O
PROBE_SIZES=4097,6001,8193,12289,16385,32769,65537 PROBE_AB_R=TC_SPLIT_REDUCE PROBE_AB_VALS=1,0 timeout 600 python tools/probe_modes.py reduce > $O/probe_split_reduce2.log 2>&1; echo "probe rc=$?"; cat $O/probe_split_reduce2.log
cap() {  # tag, command...
  tag=$1; shift
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:seg_kernel -s 2 -c 1 \
    -o $O/$tag -f "$@" > $O/$tag.log 2>&1; echo "cap $tag rc=$?"
  python tools/ncu_summary.py $O/$tag.ncu-rep > $O/$tag.txt 2>&1
  ncu -i $O/$tag.ncu-rep --page source --csv > $O/$tag.source.csv 2>/dev/null
  rm -f $O/$tag.ncu-rep
}
cap split_4097 python tools/prof_one.py reduce 4097 f16 30 3
cap split_100001 python tools/prof_one.py reduce 100001 f16 30 3
TC_SPLIT_REDUCE=0 cap general_4097 python tools/prof_one.py reduce 4097 f16 30 3
