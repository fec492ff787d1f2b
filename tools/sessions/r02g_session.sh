O=gpurun_out/r02g; mkdir -p $O
timeout 900 python -m pytest tests/test_irregular_gpu.py tests/test_parity_signed_gpu.py -q -p no:cacheprovider -x -rf -k "irreg" > $O/pytest_irreg.log 2>&1; echo "pytest irreg rc=$?"; tail -5 $O/pytest_irreg.log
PROBE_REDUCE_ONLY=1 timeout 600 python tools/probe_irreg.py 16 64 256 1024 16384 1048576 > $O/probe_v3.log 2>&1; echo "probe v3 rc=$?"; cat $O/probe_v3.log
PROBE_REDUCE_ONLY=1 TC_CTAS_PER_SM=1 timeout 600 python tools/probe_irreg.py 64 1024 > $O/probe_v3_c1.log 2>&1; echo "ctas=1"; cat $O/probe_v3_c1.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:irreg_reduce -s 2 -c 1 -o $O/prof_irreg64 -f python tools/prof_irreg.py reduce 64 f32 3 > $O/prof_irreg64.log 2>&1; echo "prof rc=$?"
python tools/ncu_summary.py $O/prof_irreg64.ncu-rep > $O/prof_irreg64.txt 2>&1; head -45 $O/prof_irreg64.txt
rm -f $O/prof_irreg64.ncu-rep
