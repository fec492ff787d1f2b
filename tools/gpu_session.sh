#!/usr/bin/env bash
# One GPU-box session: tests, bench, launch list, ncu captures.
# usage: tools/gpu_session.sh TAG [parts...]   parts: test bench launches prof probe
set -u
TAG=${1:-r01}; shift || true
PARTS=${*:-"test bench launches prof"}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
nvidia-smi > "$OUT/nvidia-smi.txt" 2>&1
python -c 'import __graft_entry__ as g; g.build()' > "$OUT/build.log" 2>&1 || { echo BUILD FAILED; tail -20 "$OUT/build.log"; }
for p in $PARTS; do
  case $p in
    test)
      timeout 900 python -m pytest tests -m gpu -x -q > "$OUT/pytest_gpu.log" 2>&1; echo "pytest gpu rc=$?"; tail -3 "$OUT/pytest_gpu.log"
      timeout 300 python -c 'import __graft_entry__ as g; g.smoke()' > "$OUT/smoke.log" 2>&1; echo "smoke rc=$?"; tail -2 "$OUT/smoke.log";;
    bench)
      timeout 900 python bench.py > "$OUT/bench.json" 2> "$OUT/bench.err"; echo "bench rc=$?"; tail -c 3000 "$OUT/bench.json"; tail -5 "$OUT/bench.err"
      timeout 600 python bench.py --impl reference > "$OUT/bench_ref.json" 2> "$OUT/bench_ref.err"; echo "bench ref rc=$?"; cut -c1-400 "$OUT/bench_ref.json";;
    launches)
      timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv \
        --log-file "$OUT/launches.csv" python bench.py --steps 2 --warmup 3 --no-cpu --e2e-steps 1 > "$OUT/launches_bench.log" 2>&1; echo "launches rc=$?";;
    prof)
      CFGS=("reduce 16 f16" "reduce 2048 f16" "reduce 65536 f16" "reduce 300 f16" "reduce 17 f16" "scan 256 f16" "scan 16384 f32" "scan 1073741824 f32" "scan 300 f16")
      for cfg in "${CFGS[@]}"; do
        set -- $cfg
        timeout 600 ncu --set full --clock-control none --import-source on -k regex:seg_kernel -s 2 -c 1 \
          -o "$OUT/prof_$1_$2_$3" -f python tools/prof_one.py $1 $2 $3 30 3 > "$OUT/prof_$1_$2_$3.log" 2>&1; echo "prof $cfg rc=$?"
        python tools/ncu_summary.py "$OUT/prof_$1_$2_$3.ncu-rep" > "$OUT/prof_$1_$2_$3.txt" 2>&1
        ncu -i "$OUT/prof_$1_$2_$3.ncu-rep" --page raw --csv > "$OUT/prof_$1_$2_$3.raw.csv" 2>/dev/null
        [ -n "${KEEP_REP:-}" ] || rm -f "$OUT/prof_$1_$2_$3.ncu-rep"
      done;;
    prof2)
      # widened rows: irregular segments (geometric mean 64 / 1024) and batch-norm statistics
      for cfg in "reduce 64 f32" "reduce 1024 f32" "scan 1024 f32"; do
        set -- $cfg
        tag=irreg_$1_$2_$3
        timeout 600 ncu --set full --clock-control none --import-source on -k regex:seg_kernel -s 2 -c 1 \
          -o "$OUT/prof_$tag" -f python tools/prof_irreg.py $1 $2 $3 3 > "$OUT/prof_$tag.log" 2>&1; echo "prof $tag rc=$?"
        python tools/ncu_summary.py "$OUT/prof_$tag.ncu-rep" > "$OUT/prof_$tag.txt" 2>&1
        rm -f "$OUT/prof_$tag.ncu-rep"
      done
      timeout 600 ncu --set full --clock-control none -k regex:"seg_kernel|bn_" -s 3 -c 3 \
        -o "$OUT/prof_bn" -f python tools/prof_bn.py 256 256 56 56 3 > "$OUT/prof_bn.log" 2>&1; echo "prof bn rc=$?"
      python tools/ncu_summary.py "$OUT/prof_bn.ncu-rep" > "$OUT/prof_bn.txt" 2>&1
      rm -f "$OUT/prof_bn.ncu-rep";;
    probe)
      timeout 600 python tools/perf_probe.py > "$OUT/perf_probe.log" 2>&1; echo "probe rc=$?"; cat "$OUT/perf_probe.log";;
  esac
done
