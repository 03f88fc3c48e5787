set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit,temperature.gpu --format=csv
run() { echo "== $*"; env "$@" KKT_V6_TIM=1 timeout 600 python scripts/time_large.py --config 2 --reps 3 > gpurun_out/tmp.log 2>&1; grep apply_P_inv_ms gpurun_out/tmp.log | sed 's/.*apply_P_inv_ms/P_inv_ms/' | cut -c1-40; grep cycles gpurun_out/tmp.log | tail -2; grep "band windows" gpurun_out/tmp.log | tail -1; }
(cd _head && echo "HEAD build" && run A=1)
run A=1
run KKT_V6_NOPOLL=1
run KKT_V6_TWIST=0
(cd _head && echo "HEAD build again" && run A=1)
timeout 900 python -m pytest tests/test_gpu_v6_twist.py -q -m gpu -x 2>&1 | tail -3
