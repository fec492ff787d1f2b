# native host stager, BN waves=2: host-path tests, host probe, bench
O=gpurun_out/r02w; mkdir -p $O
timeout 900 python -m pytest tests/test_host_path_gpu.py tests/test_batchnorm_gpu.py tests/test_facades_gpu.py -x -q -p no:cacheprovider > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest.log
timeout 300 python tools/host_probe.py > $O/host_probe.log 2>&1; tail -2 $O/host_probe.log
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"; tail -3 $O/bench.err
python - <<'PY'
import json
d=json.load(open("gpurun_out/r02w/bench.json"))
print("value", d["value"]/1e12, "frac", d["roofline"]["frac"], "e2e", d["e2e"]["value"]/1e9)
print("per_call", json.dumps(d["e2e_per_call"]))
print("bn", json.dumps(d["extras"]["batch_norm_stats"]))
print("irreg", json.dumps(d["extras"]["irregular_segments"]["rows"]))
PY
