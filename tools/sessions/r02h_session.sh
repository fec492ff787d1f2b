O=gpurun_out/r02h; mkdir -p $O
timeout 600 python -m pytest tests/test_irregular_gpu.py tests/test_parity_signed_gpu.py -q -p no:cacheprovider -x -rf -k "irreg" > $O/pytest_irreg.log 2>&1; echo "pytest irreg rc=$?"; tail -15 $O/pytest_irreg.log
PROBE_REDUCE_ONLY=1 timeout 300 python tools/probe_irreg.py 16 64 256 1024 16384 1048576 > $O/probe_v4.log 2>&1; echo "probe v4 rc=$?"; cat $O/probe_v4.log
PROBE_REDUCE_ONLY=1 TC_IRREG_GROUPS=3 timeout 300 python tools/probe_irreg.py 64 1024 > $O/probe_v4_g3.log 2>&1; echo "groups=3"; cat $O/probe_v4_g3.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:irreg_reduce -s 2 -c 1 -o $O/prof_irreg64 -f python tools/prof_irreg.py reduce 64 f32 3 > $O/prof_irreg64.log 2>&1; echo "prof rc=$?"
python tools/ncu_summary.py $O/prof_irreg64.ncu-rep > $O/prof_irreg64.txt 2>&1; head -40 $O/prof_irreg64.txt
ncu -i $O/prof_irreg64.ncu-rep --page source --csv > $O/prof_irreg64.source.csv 2>/dev/null
rm -f $O/prof_irreg64.ncu-rep
