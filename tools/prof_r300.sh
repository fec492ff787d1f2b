OUT=gpurun_out/r300; mkdir -p $OUT
ncu --set full --clock-control none --import-source on -k regex:seg_kernel -s 2 -c 1 -o $OUT/red300 -f python tools/prof_one.py reduce 300 f16 30 3 > $OUT/log 2>&1
python tools/ncu_summary.py $OUT/red300.ncu-rep --lines 30 > $OUT/red300.txt 2>&1
ncu -i $OUT/red300.ncu-rep --page source --csv > $OUT/red300.source.csv 2>/dev/null
rm -f $OUT/red300.ncu-rep
head -40 $OUT/red300.txt
python tools/src_hot.py $OUT/red300.source.csv | head -30
timeout 900 python bench.py --no-cpu --steps 10 > $OUT/bench.json 2> $OUT/bench.err; tail -2 $OUT/bench.err
python -c "import json; d=json.load(open('$OUT/bench.json')); print(json.dumps(d['extras']['reduce_bf16_input'])); print(json.dumps(d['extras']['non_pow2_segments']))"
