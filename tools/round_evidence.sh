#!/usr/bin/env bash
# Everything profiles/ keeps for a round, in one GPU session:
#   tools/round_evidence.sh TAG   -> gpurun_out/ev_TAG/*
set -u
TAG=${1:-r2}
O=gpurun_out/ev_$TAG
mkdir -p $O
if [ "${SKIP_PYTEST:-0}" != 1 ]; then timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" > $O/status.txt; fi
timeout 900 python bench.py --steps 20 --warmup 5 > $O/bench_n1.json 2> $O/bench_n1.err; echo "bench rc=$?" >> $O/status.txt
timeout 900 python bench.py --steps 100 --warmup 5 --no-cpu > $O/bench_n1_100steps.json 2>> $O/bench_n1.err; echo "bench100 rc=$?" >> $O/status.txt
timeout 900 python bench.py --impl reference --steps 5 --warmup 1 > $O/bench_reference_arm.json 2>> $O/bench_n1.err; echo "ref rc=$?" >> $O/status.txt
timeout 1200 bash tools/gpu_profile.sh $TAG bert-base-mc 288 40 > $O/gpu_profile.log 2>&1; echo "profile rc=$?" >> $O/status.txt
mv gpurun_out/prof_${TAG}_* $O/ 2>/dev/null
for P in 0 0.1; do timeout 600 python tools/bench_flash.py --p $P --classes --json $O/flash_p$P.json > /dev/null 2>&1; done
timeout 1800 bash tools/sanitize.sh > $O/sanitize.log 2>&1; mv gpurun_out/san_* $O/ 2>/dev/null
STEPS=30 timeout 2400 bash tools/bench_matrix.sh $TAG > $O/matrix_status.txt 2>&1; mv gpurun_out/bm_${TAG}_* $O/ 2>/dev/null
for U in 1 0; do timeout 600 python tools/budget_sweep.py --unit $U --out $O/budget_sweep_u$U.json > /dev/null 2>&1; done
echo done >> $O/status.txt
