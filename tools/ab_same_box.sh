#!/usr/bin/env bash
# Same-box A/B of a kernel change: builds a base snapshot (A: ab_base/, made
# here with `git archive HEAD paper_2209_02478_b200/csrc include | tar -x -C
# ab_base` since the GPU box has no .git) and the working tree (B) in scratch
# copies, then alternates the flash operator
# timing (tools/bench_flash.py) between them ROUNDS times, so both see the
# same box, clocks and thermal state:  tools/ab_same_box.sh [ROUNDS] [P]
# AB_STEP=1: per-kernel-class times of one training step (profile_step)
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
if [ "${AB_STEP:-0}" = 1 ]; then
  # per-kernel-class CUDA-event times of one planned training step instead
  for i in $(seq $ROUNDS); do
    for V in A B; do
      (cd /tmp/ab_$V && timeout 300 python tools/profile_step.py --seq 288 --planner none \
         --gemm-csv /tmp/ab_$V/prof.csv) > /dev/null 2>&1
      python - /tmp/ab_$V/prof.csv >> $OUT/$V.step <<'PY'
import csv, sys, collections, json
agg = collections.Counter()
for r in csv.DictReader(open(sys.argv[1])):
    agg[r["class"]] += float(r["ms"])
    agg["total"] += float(r["ms"])
    if r["class"] == "gemm_dense":  # per shape: M N K ... epi
        d = r["desc"].split()
        agg["  gemm " + " ".join(d[:3] + d[7:8])] += float(r["ms"])
print(json.dumps(agg))
PY
    done
  done
  python - "$OUT" <<'PY'
import json, sys, statistics
out = sys.argv[1]
rows = {V: [json.loads(l) for l in open(f"{out}/{V}.step")] for V in "AB"}
keys = sorted(rows["A"][0], key=lambda k: -rows["A"][0][k])
for k in keys:
    a = statistics.median(r.get(k, 0) for r in rows["A"]); b = statistics.median(r.get(k, 0) for r in rows["B"])
    print(f"{k:20s} A {a:7.3f} ms  B {b:7.3f} ms  ({(b / a - 1) * 100 if a else 0:+.1f} %)")
PY
  exit 0
fi
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
