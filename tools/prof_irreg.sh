# ncu captures of the irregular kernels (run on the GPU box)
OUT=gpurun_out/irr; mkdir -p $OUT
for cfg in ${CFGS:-"reduce 1048576 f32" "reduce 64 f32" "scan 1024 f32"}; do
  set -- $cfg
  tag=$1_$2_$3
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:seg_kernel -s 2 -c 1 \
    -o $OUT/$tag -f python tools/prof_irreg.py $1 $2 $3 3 > $OUT/$tag.log 2>&1
  python tools/ncu_summary.py $OUT/$tag.ncu-rep --lines 25 > $OUT/$tag.txt 2>&1
  ncu -i $OUT/$tag.ncu-rep --page source --csv > $OUT/$tag.source.csv 2>/dev/null
  ncu -i $OUT/$tag.ncu-rep --page source --csv --print-source cuda > $OUT/$tag.cuda.csv 2>/dev/null
  rm -f $OUT/$tag.ncu-rep
  echo "== $tag"; head -30 $OUT/$tag.txt
done
