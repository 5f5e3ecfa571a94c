#!/usr/bin/env bash
# Source-level ncu of the two flash backward kernels (second iteration) at
# one shape: tools/ncu_flash_bwd.sh TAG SHAPE [P] -> gpurun_out/flb_TAG_{kv,q}_*
set -u
TAG=${1:-r2}
SHAPE=${2:-8x16x1024}
P=${3:-0.1}
OUT=gpurun_out
mkdir -p $OUT
for K in kv q; do
  if [ $K = kv ]; then RX='flash_bwd_kernel<.int.0'; else RX='flash_bwd_kernel<.int.1'; fi
  ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
    -k "regex:$RX" -s 1 -c 1 -o $OUT/flb_${TAG}_$K python tools/flash_once.py --shape $SHAPE --p $P \
    > $OUT/flb_${TAG}_$K.log 2>&1
  ncu -i $OUT/flb_${TAG}_$K.ncu-rep --page source --csv --print-source cuda,sass \
    > $OUT/flb_${TAG}_${K}_source.csv 2>&1
  ncu -i $OUT/flb_${TAG}_$K.ncu-rep --page raw --csv > $OUT/flb_${TAG}_${K}_raw.csv 2>&1
  python tools/ncu_stalls.py $OUT/flb_${TAG}_${K}_source.csv 40 > $OUT/flb_${TAG}_${K}_stalls.txt 2>&1
  python tools/ncu_summary.py $OUT/flb_${TAG}_${K}_raw.csv > $OUT/flb_${TAG}_${K}_summary.txt 2>&1
  rm -f $OUT/flb_${TAG}_$K.ncu-rep
done
