# reference suite, compute-sanitizer over every mode, ncu of the sub-bar kernels
O=gpurun_out/r02e; mkdir -p $O
timeout 900 python tools/run_reference_tests.py > $O/reftests.log 2>&1; echo "reftests rc=$?"; grep -E "^(FAILED|ERROR)|passed|failed" $O/reftests.log | tail -12
prof() {  # tag regex cmd...
  local tag=$1 rx=$2; shift 2
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"$rx" -s 2 -c 1 -o $O/prof_$tag -f "$@" > $O/prof_$tag.log 2>&1; echo "prof $tag rc=$?"
  python tools/ncu_summary.py $O/prof_$tag.ncu-rep > $O/prof_$tag.txt 2>&1
  ncu -i $O/prof_$tag.ncu-rep --page source --csv --print-source cuda > $O/prof_${tag}.cuda.csv 2>/dev/null
  rm -f $O/prof_$tag.ncu-rep
}
prof irreg_reduce_64_f32 seg_kernel python tools/prof_irreg.py reduce 64 f32 3
prof irreg_reduce_1024_f32 seg_kernel python tools/prof_irreg.py reduce 1024 f32 3
prof bn_56 "bn_" python tools/prof_bn.py 256 256 56 56 4
prof scan_full_f16 seg_kernel python tools/prof_one.py scan 1073741824 f16 30 3
prof scan_100001_f16 seg_kernel python tools/prof_one.py scan 100001 f16 30 3
prof scan_17_f16 rowseg python tools/prof_one.py scan 17 f16 30 3
SAN_TIMEOUT=300 timeout 3000 tools/sanitize.sh $O/san quick
