# source-level ncu of the first fused attention forward launch of a step at S
set -u
S=${1:-288}
OUT=gpurun_out
ncu --nvtx --nvtx-include "timed_step/" --set full --import-source on --clock-control none \
  -k attn_scores_kernel -c 1 -o $OUT/attn$S python tools/profile_step.py --seq $S > $OUT/attn$S.log 2>&1
ncu -i $OUT/attn$S.ncu-rep --page source --csv --print-source cuda,sass > $OUT/attn${S}_source.csv 2>&1
ncu -i $OUT/attn$S.ncu-rep --page details --csv > $OUT/attn${S}_details.csv 2>&1
rm -f $OUT/attn$S.ncu-rep
