#!/usr/bin/env bash
# A/B of the dK/dV kernel's shared-memory split (MIMOSE_FLASH_KV_CFG 0/1/2):
# scratch builds, flash operator tests + timing -> gpurun_out/ab_kv_<cfg>.log
set -u
ROOT=$(cd "$(dirname "$0")/.." && pwd)
for C in "$@"; do
  T=/tmp/mimose_kv_$C
  rm -rf $T && mkdir -p $T
  cp -r $ROOT/Makefile $ROOT/include $ROOT/paper_2209_02478_b200 $ROOT/tools $ROOT/tests $ROOT/oracle $ROOT/MEASURED_PEAKS.json $T/ 2>/dev/null
  rm -f $T/paper_2209_02478_b200/*.so
  (cd $T && make -j "$(nproc)" NVFLAGS="$(make -s print-nvflags) -DMIMOSE_FLASH_KV_CFG=$C" \
     paper_2209_02478_b200/libmimose_cuda.so > build.log 2>&1) || { tail -20 $T/build.log; continue; }
  (cd $T && timeout 300 python -m pytest tests/test_flash_gpu.py -q -x -p no:cacheprovider -k bwd) > $ROOT/gpurun_out/ab_kv_$C.log 2>&1
  for P in 0 0.1; do
    (cd $T && timeout 300 python tools/bench_flash.py --p $P --causal 0 --classes) >> $ROOT/gpurun_out/ab_kv_$C.log 2>&1
  done
done
