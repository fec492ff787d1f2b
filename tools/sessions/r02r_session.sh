# line-level ncu of SPLIT (s=300) vs GENERAL GR8 (s=1000), f16; BN graph timing
O=gpurun_out/r02r; mkdir -p $O
cap() {  # tag, regex, command...
  tag=$1; shift; rx=$1; shift
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$rx -s 2 -c 1 \
    -o $O/$tag -f "$@" > $O/$tag.log 2>&1
  python tools/ncu_summary.py $O/$tag.ncu-rep > $O/$tag.txt 2>&1
  ncu -i $O/$tag.ncu-rep --page source --csv > $O/$tag.source.csv 2>/dev/null
  rm -f $O/$tag.ncu-rep
  echo "== $tag"; sed -n 2,3p $O/$tag.txt
}
cap split300 seg_kernel python tools/prof_one.py scan 300 f16 30 3
cap gen1000 seg_kernel python tools/prof_one.py scan 1000 f16 30 3
timeout 600 python tools/probe_modes.py bn > $O/probe_bn.log 2>&1; cat $O/probe_bn.log
