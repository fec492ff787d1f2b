O=gpurun_out/r02sm; mkdir -p $O
cap() {  # tag, regex, command...
  tag=$1; shift; rx=$1; shift
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$rx -s 2 -c 1 \
    -o $O/$tag -f "$@" > $O/$tag.log 2>&1
  python tools/ncu_summary.py $O/$tag.ncu-rep > $O/$tag.txt 2>&1
  ncu -i $O/$tag.ncu-rep --page source --csv > $O/$tag.source.csv 2>/dev/null
  rm -f $O/$tag.ncu-rep
}
TC_SPLITM=2 cap sm33_f16 seg_kernel python tools/prof_one.py scan 33 f16 30 3
TC_SPLITM=2 cap sm33_f32 seg_kernel python tools/prof_one.py scan 33 f32 30 3
