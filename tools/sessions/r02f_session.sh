# irregular reduce v2: parity + A/B against the v1 (seg_kernel) path
O=gpurun_out/r02f; mkdir -p $O
timeout 900 python -m pytest tests/test_irregular_gpu.py tests/test_parity_signed_gpu.py -q -p no:cacheprovider -x -rf -k "irreg" > $O/pytest_irreg.log 2>&1; echo "pytest irreg rc=$?"; tail -5 $O/pytest_irreg.log
PROBE_REDUCE_ONLY=1 timeout 600 python tools/probe_irreg.py 16 64 256 1024 16384 1048576 > $O/probe_v2.log 2>&1; echo "probe v2 rc=$?"; cat $O/probe_v2.log
PROBE_REDUCE_ONLY=1 TC_IRREG_V1=1 timeout 600 python tools/probe_irreg.py 64 1024 > $O/probe_v1.log 2>&1; echo "probe v1 rc=$?"; cat $O/probe_v1.log
for c in 2 1; do PROBE_REDUCE_ONLY=1 TC_CTAS_PER_SM=$c timeout 600 python tools/probe_irreg.py 64 1024 > $O/probe_v2_c$c.log 2>&1; echo "ctas=$c"; cat $O/probe_v2_c$c.log; done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:irreg_reduce -s 2 -c 1 -o $O/prof_irreg64 -f python tools/prof_irreg.py reduce 64 f32 3 > $O/prof_irreg64.log 2>&1; echo "prof rc=$?"
python tools/ncu_summary.py $O/prof_irreg64.ncu-rep > $O/prof_irreg64.txt 2>&1; head -45 $O/prof_irreg64.txt
ncu -i $O/prof_irreg64.ncu-rep --page source --csv --print-source cuda > $O/prof_irreg64.cuda.csv 2>/dev/null; rm -f $O/prof_irreg64.ncu-rep
