# IRREG reduce v7 (tile-parallel epilogue groups + k0 pre-pass): parity + A/B; BN unroll/waves A/B
O=gpurun_out/r02u; mkdir -p $O
timeout 900 python -m pytest tests/test_irregular_gpu.py tests/test_parity_signed_gpu.py -k "irreg or irregular" -x -q -p no:cacheprovider > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -5 $O/pytest.log
PROBE_REDUCE_ONLY=1 timeout 600 python tools/probe_irreg.py 16 64 256 1024 16384 1048576 > $O/probe_v7.log 2>&1; echo v7; cat $O/probe_v7.log
TC_IRREG_V1=1 PROBE_REDUCE_ONLY=1 timeout 600 python tools/probe_irreg.py 64 1024 > $O/probe_v1.log 2>&1; echo v1; cat $O/probe_v1.log
for u in 4 8; do for w in 2 4 8; do echo "BN unroll=$u waves=$w"; TC_BN_UNROLL=$u TC_BN_WAVES=$w timeout 300 python tools/probe_modes.py bn 2>&1 | head -2; done; done
