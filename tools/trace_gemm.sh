#!/usr/bin/env bash
# Per-tile GEMM pipeline trace from a traced build in a scratch copy:
#   tools/trace_gemm.sh -> gpurun_out/gemm_trace.txt
set -u
ROOT=$(cd "$(dirname "$0")/.." && pwd)
T=/tmp/mimose_gtrace
rm -rf $T && mkdir -p $T
cp -r $ROOT/Makefile $ROOT/include $ROOT/paper_2209_02478_b200 $ROOT/tools $T/
rm -f $T/paper_2209_02478_b200/*.so
(cd $T && make -j "$(nproc)" NVFLAGS="$(make -s print-nvflags) -DMIMOSE_GEMM_TRACE" \
   paper_2209_02478_b200/libmimose_cuda.so > build.log 2>&1) || { tail -20 $T/build.log; exit 1; }
mkdir -p $ROOT/gpurun_out
(cd $T && python tools/gemm_trace.py) > $ROOT/gpurun_out/gemm_trace.txt 2>&1
