set -u
for S in 288 400 512; do
  python tools/profile_step.py --seq $S --time-steps 10 2>&1 | grep ms/step
  MIMOSE_ATTN_FWD_MAX=256 python tools/profile_step.py --seq $S --time-steps 10 2>&1 | grep ms/step
done
