# source-level ncu of the N-th GEMM launch of one planned step (default: FFN1
# bias+GELU = 4th GEMM of layer 0): tools/ncu_source_kernel.sh TAG SKIP [KERNEL]
set -u
TAG=${1:-ffn1}
SKIP=${2:-3}
KERNEL=${3:-gemm_bf16_tn_kernel}
OUT=gpurun_out
ncu --nvtx --nvtx-include "timed_step/" --set full --import-source on --clock-control none \
  -k $KERNEL -s $SKIP -c 1 -o $OUT/$TAG python tools/profile_step.py --seq 288 > $OUT/$TAG.log 2>&1
ncu -i $OUT/$TAG.ncu-rep --page source --csv --print-source cuda,sass > $OUT/${TAG}_source.csv 2>&1
ncu -i $OUT/$TAG.ncu-rep --page details --csv > $OUT/${TAG}_details.csv 2>&1
rm -f $OUT/$TAG.ncu-rep
