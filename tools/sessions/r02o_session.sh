# ncu: SPLIT scans f16 vs f32, new BN channel kernel
O=gpurun_out/r02o; mkdir -p $O
prof() {  # tag regex cmd...
  local tag=$1 rx=$2; shift 2
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"$rx" -s 2 -c 1 -o $O/prof_$tag -f "$@" > $O/prof_$tag.log 2>&1; echo "prof $tag rc=$?"
  python tools/ncu_summary.py $O/prof_$tag.ncu-rep > $O/prof_$tag.txt 2>&1
  ncu -i $O/prof_$tag.ncu-rep --page source --csv --print-source cuda > $O/prof_${tag}.cuda.csv 2>/dev/null
  ncu -i $O/prof_$tag.ncu-rep --page raw --csv > $O/prof_${tag}.raw.csv 2>/dev/null
  rm -f $O/prof_$tag.ncu-rep
}
prof split_4097_f16 seg_kernel python tools/prof_one.py scan 4097 f16 30 3
prof split_4097_f32 seg_kernel python tools/prof_one.py scan 4097 f32 30 3
prof split_300_f16 seg_kernel python tools/prof_one.py scan 300 f16 30 3
prof bn_56 "bn_chan" python tools/prof_bn.py 256 256 56 56 4
