#!/usr/bin/env bash
# Source-level ncu (--set full, stall sampling per SASS line) of the flash
# attention kernels at one shape (second, warm iteration of tools/flash_once.py):
#   tools/ncu_flash.sh TAG SHAPE [P] [CAUSAL]
set -u
TAG=${1:-r2}
SHAPE=${2:-64x12x288}
P=${3:-0.1}
C=${4:-0}
OUT=gpurun_out
mkdir -p $OUT
run() {  # kernel-regex skip count
  local K=$1 SK=$2 N=$3
  ncu --set full --import-source on --clock-control none -k regex:$K -s $SK -c $N \
    -o $OUT/fl_${TAG}_$K python tools/flash_once.py --shape $SHAPE --p $P --causal $C \
    > $OUT/fl_${TAG}_$K.log 2>&1
  ncu -i $OUT/fl_${TAG}_$K.ncu-rep --page raw --csv > $OUT/fl_${TAG}_${K}_raw.csv 2>&1
  ncu -i $OUT/fl_${TAG}_$K.ncu-rep --page source --csv --print-source cuda,sass \
    > $OUT/fl_${TAG}_${K}_source.csv 2>&1
  python tools/ncu_stalls.py $OUT/fl_${TAG}_${K}_source.csv 30 > $OUT/fl_${TAG}_${K}_stalls.txt 2>&1
  python tools/ncu_summary.py $OUT/fl_${TAG}_${K}_raw.csv > $OUT/fl_${TAG}_${K}_summary.txt 2>&1
  rm -f $OUT/fl_${TAG}_$K.ncu-rep
}
run flash_fwd_kernel 1 1
run flash_bwd_kernel 1 1
run flash_keep_mask_kernel 1 1
