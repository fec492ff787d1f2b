# round-2 evidence session: full GPU suite, smoke, bench + reference arm, launch list, ncu captures
O=gpurun_out/r02x; mkdir -p $O
nvidia-smi > $O/nvidia-smi.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -rf --timeout 1500 > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; grep -E "passed|failed|^FAILED|^ERROR" $O/pytest_gpu.log | tail -8
timeout 300 python -c 'import __graft_entry__ as g; g.smoke()' > $O/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $O/smoke.log
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"; tail -3 $O/bench.err
timeout 600 python bench.py --impl reference > $O/bench_ref.json 2> $O/bench_ref.err; echo "bench ref rc=$?"; cut -c1-300 $O/bench_ref.json
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv \
  --log-file $O/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --e2e-steps 1 > $O/launches_bench.log 2>&1; echo "launches rc=$?"
prof() {  # tag regex cmd...
  local tag=$1 rx=$2; shift 2
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"$rx" -s 2 -c 1 -o $O/prof_$tag -f "$@" > $O/prof_$tag.log 2>&1; echo "prof $tag rc=$?"
  python tools/ncu_summary.py $O/prof_$tag.ncu-rep > $O/prof_$tag.txt 2>&1
  rm -f $O/prof_$tag.ncu-rep
}
prof reduce_16_f16 seg_kernel python tools/prof_one.py reduce 16 f16 30 3
prof reduce_256_f16 seg_kernel python tools/prof_one.py reduce 256 f16 30 3
prof reduce_65536_f16 seg_kernel python tools/prof_one.py reduce 65536 f16 30 3
prof reduce_17_f16 rowseg python tools/prof_one.py reduce 17 f16 30 3
prof scan_256_f16 seg_kernel python tools/prof_one.py scan 256 f16 30 3
prof scan_16384_f32 seg_kernel python tools/prof_one.py scan 16384 f32 30 3
prof scan_full_f32 seg_kernel python tools/prof_one.py scan 1073741824 f32 30 3
prof scan_split_100001_f16 seg_kernel python tools/prof_one.py scan 100001 f16 30 3
prof scan_300_f16 seg_kernel python tools/prof_one.py scan 300 f16 30 3
prof irreg_reduce_1024_f32 irreg_reduce python tools/prof_irreg.py reduce 1024 f32 3
prof irreg_reduce_64_f32 irreg_reduce python tools/prof_irreg.py reduce 64 f32 3
prof bn_56 bn_chan python tools/prof_bn.py 256 256 56 56 4
