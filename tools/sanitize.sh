#!/usr/bin/env bash
# compute-sanitizer memcheck / racecheck / synccheck / initcheck over one small
# case per kernel family (tools/sanitize_cases.py); one log per (tool, case)
# under gpurun_out/sanitize/, summary lines in gpurun_out/sanitize/summary.txt.
cd "$(dirname "$0")/.."
OUT=gpurun_out/sanitize
mkdir -p "$OUT"
: > "$OUT/summary.txt"
CASES=${CASES:-"bottom_cluster bottom_cluster_255 bottom_single stream stream_fast ctile per_op zebra pcg strip"}
TOOLS=${TOOLS:-"memcheck racecheck synccheck initcheck"}
for tool in $TOOLS; do
  for c in $CASES; do
    log="$OUT/${tool}_${c}.log"
    timeout 900 compute-sanitizer --tool "$tool" --error-exitcode 99 --print-limit 20 \
        python tools/sanitize_cases.py "$c" > "$log" 2>&1
    rc=$?
    summ=$(grep -E "ERROR SUMMARY|RACECHECK SUMMARY|Error|case .* ok" "$log" | tail -2 | tr '\n' ' ')
    echo "$tool $c rc=$rc $summ" | tee -a "$OUT/summary.txt"
  done
done
