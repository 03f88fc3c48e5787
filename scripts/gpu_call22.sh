set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_v6_twist.py tests/test_gpu_v6.py -q -m gpu -x 2>&1 | tail -15
for tw in 1 0; do
echo "== config 2 twist=$tw"; KKT_V6_TWIST=$tw KKT_V6_TIM=1 timeout 600 python scripts/time_large.py --config 2 --reps 3 2>&1 | tail -6
echo "== config 3 twist=$tw"; KKT_V6_TWIST=$tw KKT_V6_TIM=1 timeout 600 python scripts/time_large.py --config 3 --reps 3 2>&1 | tail -6
done
echo "== c4 slab twist=1"; KKT_V6_TIM=1 timeout 900 python scripts/time_large.py --config 4 --nt 128 --T 0.125 --nd 16 --reps 3 2>&1 | tail -6
timeout 1200 python -m pytest tests/test_gpu_large.py -q -m gpu -x 2>&1 | tail -4
