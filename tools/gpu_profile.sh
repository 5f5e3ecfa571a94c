#!/usr/bin/env bash
# One GPU profiling pass (run under gpurun from the repo root):
#   1. per-launch CUDA-event breakdown of a planned step (all kernel classes)
#   2. ncu launch list of the same step (cold-cache, serialised)
#   3. ncu --set full on the first launches of the step (GEMMs + memory stages)
# Outputs go to gpurun_out/prof_<tag>_*. Usage: tools/gpu_profile.sh TAG PRESET SEQ [NCU_COUNT]
set -u
TAG=${1:-r1}
PRESET=${2:-bert-base-mc}
SEQ=${3:-288}
NCU_COUNT=${4:-40}
OUT=gpurun_out
mkdir -p $OUT
python tools/profile_step.py --preset $PRESET --seq $SEQ --gemm-csv $OUT/prof_${TAG}_events.csv \
  --time-steps 10 > $OUT/prof_${TAG}_summary.txt 2>&1
ncu --nvtx --nvtx-include "timed_step/" --metrics gpu__time_duration.sum --clock-control none \
  --csv --log-file $OUT/prof_${TAG}_launches.csv \
  python tools/profile_step.py --preset $PRESET --seq $SEQ > /dev/null 2>&1
python tools/launch_summary.py $OUT/prof_${TAG}_launches.csv > $OUT/prof_${TAG}_launches_summary.txt 2>&1
ncu --nvtx --nvtx-include "timed_step/" --set full --clock-control none --import-source on \
  -c $NCU_COUNT -o $OUT/prof_${TAG}_full \
  python tools/profile_step.py --preset $PRESET --seq $SEQ > $OUT/prof_${TAG}_ncu_full.log 2>&1
ncu -i $OUT/prof_${TAG}_full.ncu-rep --page raw --csv > $OUT/prof_${TAG}_full_raw.csv 2>&1
rm -f $OUT/prof_${TAG}_full.ncu-rep
# backward half of the step
ncu --nvtx --nvtx-include "timed_step/" --set full --clock-control none --import-source on \
  -s ${NCU_BWD_SKIP:-200} -c $NCU_COUNT -o $OUT/prof_${TAG}_fullbwd \
  python tools/profile_step.py --preset $PRESET --seq $SEQ > $OUT/prof_${TAG}_ncu_fullbwd.log 2>&1
ncu -i $OUT/prof_${TAG}_fullbwd.ncu-rep --page raw --csv > $OUT/prof_${TAG}_fullbwd_raw.csv 2>&1
rm -f $OUT/prof_${TAG}_fullbwd.ncu-rep
echo done
