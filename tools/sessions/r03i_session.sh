# final session of the round: full GPU tests, smoke, bench + reference arm, launch list,
# sanitizers on the reduce modes (SPLIT reduce is new), ncu of the retuned kernels
O=gpurun_out/r03i; mkdir -p $O
bash tools/gpu_session.sh r03i test bench launches
bash tools/sanitize.sh $O/sanitize quick "memcheck racecheck synccheck" "reduce scan"
cap() {  # tag, command...
  tag=$1; shift
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"seg_kernel|rowseg" -s 2 -c 1 \
    -o $O/$tag -f "$@" > $O/$tag.log 2>&1; echo "cap $tag rc=$?"
  python tools/ncu_summary.py $O/$tag.ncu-rep > $O/$tag.txt 2>&1
  rm -f $O/$tag.ncu-rep
}
cap ncu_reduce_17_f16 python tools/prof_one.py reduce 17 f16 30 3
cap ncu_scan_17_f16 python tools/prof_one.py scan 17 f16 30 3
cap ncu_reduce_100001_f16 python tools/prof_one.py reduce 100001 f16 30 3
TC_RS_EVICT=0 cap ncu_reduce_17_f16_evictfirst python tools/prof_one.py reduce 17 f16 30 3
