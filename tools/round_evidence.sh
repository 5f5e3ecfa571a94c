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
# ncu of the flash kernels at the BERT-base and the long-sequence shape
for SH in 64x12x288 8x16x1024; do
  timeout 900 bash tools/ncu_flash.sh ${TAG}_$SH $SH 0.1 > /dev/null 2>&1
  timeout 900 bash tools/ncu_flash_bwd.sh ${TAG}_$SH $SH 0.1 > /dev/null 2>&1
done
mv gpurun_out/fl_${TAG}_* gpurun_out/flb_${TAG}_* $O/ 2>/dev/null
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/status.txt
timeout 1800 bash tools/sanitize.sh > $O/sanitize.log 2>&1; mv gpurun_out/san_* $O/ 2>/dev/null
STEPS=30 timeout 2400 bash tools/bench_matrix.sh $TAG > $O/matrix_status.txt 2>&1; mv gpurun_out/bm_${TAG}_* $O/ 2>/dev/null
for U in 1 0; do timeout 600 python tools/budget_sweep.py --unit $U --out $O/budget_sweep_u$U.json > /dev/null 2>&1; done
# the reference CLI's grid (mimose_main.cpp cmd_compare) over real B200 runs:
# BERT-base MC, S ~ U(64, 512), 4 planners x 3 budgets, 80 iterations each
make -s build/mimose_gpu > /dev/null 2>&1 || g++ -O2 -std=c++17 -Iinclude -I/usr/local/cuda/include \
  paper_2209_02478_b200/cli/mimose_gpu.cpp -o build/mimose_gpu -Lpaper_2209_02478_b200 -lmimose_cuda \
  -lmimose_host -L/usr/local/cuda/lib64 -lcudart -Wl,-rpath,$PWD/paper_2209_02478_b200
timeout 1800 build/mimose_gpu compare --model bert-base-mc --dist uniform:64:512 --batch-multiplier 64 \
  --iters 80 --seed 2024 --budgets 6g,8g,12g --planners mimose,static-max,dtr,none \
  --out $O/cli_compare_bert.csv > $O/cli_compare.log 2>&1; echo "cli compare rc=$?" >> $O/status.txt
echo done >> $O/status.txt
