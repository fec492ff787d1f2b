# full GPU suite + smoke + bench after MODE_SPLIT / BN rewrite
O=gpurun_out/r02t; mkdir -p $O
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -rf --timeout 1500 > $O/pytest.log 2>&1; echo "pytest rc=$?"; grep -E "passed|failed|^FAILED|^ERROR" $O/pytest.log | tail -20
timeout 300 python -c 'import __graft_entry__ as g; g.smoke()' > $O/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 $O/smoke.log
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"; tail -5 $O/bench.err
timeout 600 python tools/probe_modes.py bn > $O/probe_bn.log 2>&1; cat $O/probe_bn.log
