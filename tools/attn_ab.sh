set -u
timeout 900 python -m pytest tests/test_trainer_gpu.py -x -q 2>&1 | tail -3
for S in 128 256 288 400 512; do
  python tools/profile_step.py --seq $S --time-steps 10 --attn-unfused 2>&1 | grep ms/step
  python tools/profile_step.py --seq $S --time-steps 10 2>&1 | grep ms/step
done
