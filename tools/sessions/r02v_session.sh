# IRREG v7b (no load-use waits in the prefetch) + ncu at mean 1024
O=gpurun_out/r02v; mkdir -p $O
timeout 900 python -m pytest tests/test_irregular_gpu.py -x -q -p no:cacheprovider > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest.log
PROBE_REDUCE_ONLY=1 timeout 600 python tools/probe_irreg.py 16 64 256 1024 16384 1048576 > $O/probe_v7.log 2>&1; echo v7; cat $O/probe_v7.log
cap() {  # tag, regex, command...
  tag=$1; shift; rx=$1; shift
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$rx -s 1 -c 1 \
    -o $O/$tag -f "$@" > $O/$tag.log 2>&1
  python tools/ncu_summary.py $O/$tag.ncu-rep > $O/$tag.txt 2>&1
  ncu -i $O/$tag.ncu-rep --page source --csv > $O/$tag.source.csv 2>/dev/null
  rm -f $O/$tag.ncu-rep
  echo "== $tag"; sed -n 2,3p $O/$tag.txt
}
cap ir1024 irreg_reduce python tools/prof_irreg.py reduce 1024 f32 3
cap ir64 irreg_reduce python tools/prof_irreg.py reduce 64 f32 3
