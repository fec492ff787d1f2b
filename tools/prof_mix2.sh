OUT=gpurun_out/mix2; mkdir -p $OUT
cap() {
  tag=$1; shift; rx=$1; shift
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$rx -s 2 -c 1 \
    -o $OUT/$tag -f "$@" > $OUT/$tag.log 2>&1
  python tools/ncu_summary.py $OUT/$tag.ncu-rep --lines 10 > $OUT/$tag.txt 2>&1
  ncu -i $OUT/$tag.ncu-rep --page source --csv > $OUT/$tag.source.csv 2>/dev/null
  rm -f $OUT/$tag.ncu-rep
  echo "== $tag"; sed -n 2,6p $OUT/$tag.txt; grep -A9 "stall reasons" $OUT/$tag.txt
}
cap red300 seg_kernel python tools/prof_one.py reduce 300 f16 30 3
cap red2048 seg_kernel python tools/prof_one.py reduce 2048 f16 30 3
