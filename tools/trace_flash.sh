#!/usr/bin/env bash
# Pipeline trace of the flash forward (CTA 0 SM clocks per block) from a traced
# build in a scratch copy (the in-tree libraries stay untraced):
#   tools/trace_flash.sh S1 S2 ...  -> gpurun_out/flash_trace.txt
set -u
ROOT=$(cd "$(dirname "$0")/.." && pwd)
T=/tmp/mimose_trace
rm -rf $T && mkdir -p $T
cp -r $ROOT/Makefile $ROOT/include $ROOT/paper_2209_02478_b200 $ROOT/tools $ROOT/tests $T/
rm -f $T/paper_2209_02478_b200/*.so
(cd $T && make -j "$(nproc)" NVFLAGS="$(make -s print-nvflags) -DMIMOSE_FLASH_TRACE" \
   paper_2209_02478_b200/libmimose_cuda.so > build.log 2>&1) || { tail -20 $T/build.log; exit 1; }
mkdir -p $ROOT/gpurun_out
(cd $T && python tools/flash_trace.py "$@") > $ROOT/gpurun_out/flash_trace.txt 2>&1
(cd $T && python tools/flash_trace_bwd.py "$@") > $ROOT/gpurun_out/flash_trace_bwd.txt 2>&1
