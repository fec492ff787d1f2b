#!/usr/bin/env bash
# compute-sanitizer over tools/sanitize.py (every kernel mode, small n), one
# process per (tool, case group) so a slow / stuck case cannot hide the rest.
# usage: tools/sanitize.sh OUTDIR [quick|full] [TOOLS] [PARTS]
set -u
OUT=${1:-gpurun_out/sanitize}; MODE=${2:-quick}
TOOLS=${3:-"memcheck racecheck synccheck initcheck"}
PARTS=${4:-"reduce scan chunk irreg bn"}
TMO=${SAN_TIMEOUT:-420}
mkdir -p "$OUT"
compute-sanitizer --version > "$OUT/version.txt" 2>&1
timeout 300 python tools/sanitize.py $MODE > "$OUT/plain.log" 2>&1; echo "plain rc=$?"; tail -1 "$OUT/plain.log"
for tool in $TOOLS; do
  for part in $PARTS; do
    extra=""
    [ "$tool" = initcheck ] && [ "$part" != reduce ] && [ "$part" != bn ] && continue  # see DESIGN: TMA stores untracked
    [ "$tool" = racecheck ] && extra="--racecheck-report all"
    log="$OUT/${tool}_${part}.log"
    timeout $TMO compute-sanitizer --tool $tool $extra --print-limit 50 --error-exitcode 99 \
      python tools/sanitize.py $MODE $part > "$log" 2>&1
    echo "$tool $part rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|sanitize cases ok' "$log" | tr '\n' ' ' | cut -c1-200)"
  done
done
