set -x
mkdir -p gpurun_out
run() { echo "== $*"; env "$@" KKT_V6_TIM=1 timeout 600 python scripts/time_large.py --config 2 --reps 3 > gpurun_out/tmp.log 2>&1; grep apply_P_inv_ms gpurun_out/tmp.log | sed 's/.*apply_P_inv_ms/P_inv_ms/' | cut -c1-40; grep cycles gpurun_out/tmp.log | tail -2; }
run A=1
run KKT_V6_NOPOLL=1
run KKT_V6_TWIST=0
echo "== config 3"; KKT_V6_TIM=1 timeout 600 python scripts/time_large.py --config 3 --reps 3 2>&1 | tail -3
timeout 900 python -m pytest tests/test_gpu_v6_twist.py -q -m gpu -x 2>&1 | tail -3
