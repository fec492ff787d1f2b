# ncu --set full capture of the 2^30 full exclusive scan (CHUNK mode); summaries only
set -u
OUT=gpurun_out/${1:-full}; mkdir -p $OUT
export TC_CHUNK_TILES=${TC_CHUNK_TILES:-2}
ncu --set full --clock-control none --import-source on -k regex:seg_kernel -s 2 -c 1 -o $OUT/full_f32 -f python tools/prof_one.py scan 1073741824 f32 30 3 > $OUT/log 2>&1
python tools/ncu_summary.py $OUT/full_f32.ncu-rep --lines 60 > $OUT/full_f32.txt 2>&1
ncu -i $OUT/full_f32.ncu-rep --page source --csv > $OUT/full_f32.source.csv 2>/dev/null
ncu -i $OUT/full_f32.ncu-rep --page details --csv > $OUT/full_f32.details.csv 2>/dev/null
rm -f $OUT/full_f32.ncu-rep
cat $OUT/full_f32.txt
