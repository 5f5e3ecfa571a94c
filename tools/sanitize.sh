#!/usr/bin/env bash
# compute-sanitizer over every kernel family (tools/sanitize_cases.py):
# memcheck, racecheck, synccheck, initcheck. Summaries -> gpurun_out/san_<tool>_<case>.txt
set -u
OUT=gpurun_out
mkdir -p $OUT
for TOOL in memcheck synccheck racecheck initcheck; do
  for CASE in gemm flash step; do
    # initcheck: GEMM outputs through per-thread stores (TMA bulk stores are
    # invisible to it)
    D=0; [ $TOOL = initcheck ] && D=1
    MIMOSE_GEMM_DIRECT_STORE=$D timeout 900 compute-sanitizer --tool $TOOL --target-processes all \
      --print-limit 20 python tools/sanitize_cases.py $CASE > $OUT/san_${TOOL}_${CASE}.txt 2>&1
    echo "$TOOL $CASE rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|error' $OUT/san_${TOOL}_${CASE}.txt | tail -1)"
  done
done
