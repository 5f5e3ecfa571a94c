#!/usr/bin/env bash
# Same-box A/B of a GEMM compile flag: builds the working tree with and
# without -D$FLAG and alternates tools/bench_gemm.py between the two:
#   tools/ab_gemm_flag.sh "MIMOSE_GELU_2BUF=0" [ROUNDS]
# (AB_TOOL / AB_ARGS: another timing script, e.g. tools/bench_flash.py "--p 0.1 --causal 0 --classes")
set -u
ROOT=$(cd "$(dirname "$0")/.." && pwd)
FLAG=$1
ROUNDS=${2:-3}
OUT=$ROOT/gpurun_out/ab_gemm
mkdir -p $OUT
for V in A B; do
  T=/tmp/abg_$V
  rm -rf $T && mkdir -p $T
  cp -r $ROOT/Makefile $ROOT/include $ROOT/paper_2209_02478_b200 $ROOT/tools $ROOT/MEASURED_PEAKS.json $T/
  rm -f $T/paper_2209_02478_b200/*.so
  EXTRA=""; [ $V = A ] && EXTRA="-D$FLAG"
  (cd $T && make -j "$(nproc)" NVFLAGS="$(make -s print-nvflags) $EXTRA" paper_2209_02478_b200/libmimose_cuda.so > build.log 2>&1) || { tail -20 $T/build.log; exit 1; }
done
for i in $(seq $ROUNDS); do
  for V in A B; do (cd /tmp/abg_$V && timeout 300 python ${AB_TOOL:-tools/bench_gemm.py} ${AB_ARGS:-}) >> $OUT/$V.log 2>&1; done
done
for V in A B; do echo "== $V"; sort $OUT/$V.log | awk -F: '{print}' ; done
