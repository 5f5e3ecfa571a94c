#!/usr/bin/env bash
# One GPU session of kernel diagnostics -> gpurun_out/diag_TAG/:
# flash forward pipeline trace, source-level ncu stalls of the flash kernels
# (S = 288 and 1024), and of the memory-bound stages / the GELU GEMM of one
# planned step.   tools/diag_batch.sh TAG
set -u
TAG=${1:-d}
O=gpurun_out/diag_$TAG
mkdir -p $O
timeout 600 bash tools/trace_flash.sh 288 512 1024 > $O/trace.log 2>&1
mv gpurun_out/flash_trace.txt $O/ 2>/dev/null
timeout 900 bash tools/ncu_flash.sh ${TAG}288 64x12x288 0.1 0 > /dev/null 2>&1
timeout 900 bash tools/ncu_flash.sh ${TAG}1024 8x16x1024 0.1 0 > /dev/null 2>&1
mv gpurun_out/fl_${TAG}* $O/ 2>/dev/null
# memory-bound stages + FFN1 GELU GEMM of one planned step (S = 288)
for K in ln_bwd_kernel:0 colsum_partial_kernel:0 add_ln_fwd_kernel:0 gemm_bf16_tn_kernel:3; do
  N=${K%%:*}; S=${K##*:}
  timeout 600 bash tools/ncu_source_kernel.sh ${TAG}_$N $S $N > /dev/null 2>&1
  python tools/ncu_stalls.py gpurun_out/${TAG}_${N}_source.csv 30 > $O/${N}_stalls.txt 2>&1
  mv gpurun_out/${TAG}_${N}* $O/ 2>/dev/null
done
rm -f $O/*_source.csv.gz
echo done > $O/status.txt
