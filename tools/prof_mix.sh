# ncu captures for the line-level stall analysis (tools/ncu_lines.py)
OUT=gpurun_out/mix; mkdir -p $OUT
cap() {  # tag, regex, command...
  tag=$1; shift; rx=$1; shift
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$rx -s 2 -c 1 \
    -o $OUT/$tag -f "$@" > $OUT/$tag.log 2>&1
  python tools/ncu_summary.py $OUT/$tag.ncu-rep --lines 10 > $OUT/$tag.txt 2>&1
  ncu -i $OUT/$tag.ncu-rep --page source --csv > $OUT/$tag.source.csv 2>/dev/null
  rm -f $OUT/$tag.ncu-rep
  echo "== $tag"; sed -n 2,6p $OUT/$tag.txt
}
cap ired64 seg_kernel python tools/prof_irreg.py reduce 64 f32 3
cap fscan16 seg_kernel python tools/prof_one.py scan 1073741824 f16 30 3
cap gscan300 seg_kernel python tools/prof_one.py scan 300 f32 30 3
