#!/usr/bin/env bash
# Same-box A/B of a kernel change: builds a base snapshot (A: ab_base/, made
# here with `git archive HEAD paper_2209_02478_b200/csrc include | tar -x -C
# ab_base` since the GPU box has no .git) and the working tree (B) in scratch
# copies, then alternates the flash operator
# timing (tools/bench_flash.py) between them ROUNDS times, so both see the
# same box, clocks and thermal state:  tools/ab_same_box.sh [ROUNDS] [P]
set -u
ROOT=$(cd "$(dirname "$0")/.." && pwd)
ROUNDS=${1:-3}
P=${2:-0.1}
OUT=$ROOT/gpurun_out/ab_same_box
mkdir -p $OUT
for V in A B; do
  T=/tmp/ab_$V
  rm -rf $T && mkdir -p $T
  cp -r $ROOT/Makefile $ROOT/include $ROOT/paper_2209_02478_b200 $ROOT/tools $ROOT/MEASURED_PEAKS.json $T/
  if [ $V = A ]; then
    [ -d $ROOT/ab_base ] || { echo "no ab_base/ snapshot"; exit 1; }
    cp -r $ROOT/ab_base/. $T/
  fi
  rm -f $T/paper_2209_02478_b200/*.so
  (cd $T && make -j "$(nproc)" paper_2209_02478_b200/libmimose_cuda.so > build.log 2>&1) || { tail -20 $T/build.log; exit 1; }
done
for i in $(seq $ROUNDS); do
  for V in A B; do
    (cd /tmp/ab_$V && timeout 300 python tools/bench_flash.py --p $P --causal 0 --classes) >> $OUT/$V.log 2>&1
  done
done
python - "$OUT" <<'PY'
import json, sys, collections, statistics
out = sys.argv[1]
for V in "AB":
    agg = collections.defaultdict(list)
    for l in open(f"{out}/{V}.log"):
        try: d = json.loads(l)
        except Exception: continue
        for k, v in d.get("kernels_us", {}).items():
            agg[(d["S"], k)].append(v)
    print(V, " ".join(f"S{S}:{k.replace('attn_flash_','')}={statistics.median(v):.1f}" for (S, k), v in sorted(agg.items())))
PY
