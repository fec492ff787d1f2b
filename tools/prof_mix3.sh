OUT=gpurun_out/mix3; mkdir -p $OUT
tag=ired1024
timeout 600 ncu --set full --clock-control none --import-source on -k regex:seg_kernel -s 2 -c 1 \
  -o $OUT/$tag -f python tools/prof_irreg.py reduce 1024 f32 3 > $OUT/$tag.log 2>&1
python tools/ncu_summary.py $OUT/$tag.ncu-rep --lines 10 > $OUT/$tag.txt 2>&1
ncu -i $OUT/$tag.ncu-rep --page source --csv > $OUT/$tag.source.csv 2>/dev/null
ncu -i $OUT/$tag.ncu-rep --page details --csv > $OUT/$tag.details.csv 2>/dev/null
rm -f $OUT/$tag.ncu-rep
sed -n 2,40p $OUT/$tag.txt
