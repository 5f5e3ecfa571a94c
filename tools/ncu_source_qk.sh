set -u
OUT=gpurun_out
ncu --nvtx --nvtx-include "timed_step/" --set full --import-source on --clock-control none -k gemm_bf16_tn_kernel -s 1 -c 1 -o $OUT/qk python tools/profile_step.py --seq 288 > $OUT/qk.log 2>&1
ncu -i $OUT/qk.ncu-rep --page source --csv --print-source cuda,sass > $OUT/qk_source.csv 2>&1
ncu -i $OUT/qk.ncu-rep --page details --csv > $OUT/qk_details.csv 2>&1
rm -f $OUT/qk.ncu-rep
ls -la $OUT
