#!/usr/bin/env bash
# The BASELINE configurations and planner / budget variants as bench lines
# (one JSON line each) -> gpurun_out/bm_<TAG>_<name>.json
set -u
TAG=${1:-r2}
STEPS=${STEPS:-30}
OUT=gpurun_out
mkdir -p $OUT
run() {
  local name=$1; shift
  timeout 1200 python bench.py --steps $STEPS --warmup 5 --no-cpu "$@" > $OUT/bm_${TAG}_$name.json 2> $OUT/bm_${TAG}_$name.err
  echo "$name rc=$?"
}
run bert40 
run bert40_self --budget-basis self
run bert40_self_regen --budget-basis self --ffn-regen-g 1
run bert40_static --planner static-max
run bert40_dtr --planner dtr
run bert40_block --ckpt-unit 0
run bert60 --budget-frac 0.6
run bert80 --budget-frac 0.8
run bert40_normal --dist normal:180:60:64:512
run bert60_normal --dist normal:180:60:64:512 --budget-frac 0.6
run roberta_base_tol0 --preset roberta-base-qa
run roberta_base_tol002 --preset roberta-base-qa --cache-tol 0.02
run roberta_large --preset roberta-large-qa
run gpt2 --preset gpt2-medium-lm
run gpt2_self60 --preset gpt2-medium-lm --budget-basis self --budget-frac 0.6
run bertlarge --preset bert-large-mlm
run bertlarge_self50 --preset bert-large-mlm --budget-basis self --budget-frac 0.5
run small4 --preset small4-h256
