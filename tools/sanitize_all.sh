#!/bin/bash
# compute-sanitizer over every kernel family (tools/sanitize_cases.py); one log per tool x case in
# gpurun_out/sanitize/, a summary line each.  Run on the GPU box: tools/gpu.sh ... 'bash tools/sanitize_all.sh'
mkdir -p gpurun_out/sanitize
CS=/usr/local/cuda/bin/compute-sanitizer
for c in ${CASES:-linalg slots encode mgd3 mgd4 mlp dp}; do
  for t in ${TOOLS:-memcheck racecheck synccheck initcheck}; do
    log=gpurun_out/sanitize/${t}_${c}.log
    timeout ${TMO:-900} $CS --tool $t --error-exitcode 9 --print-limit 20 python tools/sanitize_cases.py $c > $log 2>&1
    rc=$?
    echo "$t $c rc=$rc $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|case .* ok' $log | tr '\n' ' ')"
  done
done
