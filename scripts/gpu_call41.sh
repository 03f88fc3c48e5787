mkdir -p gpurun_out
timeout 2400 python -m pytest tests/test_gpu_v6_twist.py tests/test_gpu_large.py tests/test_gpu_v6.py -q -m gpu -x 2>&1 | tail -15
run() { cfg=$1; shift; echo "== config $cfg $*"; env "$@" KKT_V6_TIM=1 timeout 600 python scripts/time_large.py $cfg --reps 3 --e2e > gpurun_out/tmp.log 2>&1; grep apply_P_inv_ms gpurun_out/tmp.log | sed 's/.*apply_P_inv_ms/P_inv_ms/' | cut -c1-100; grep "elimination form" gpurun_out/tmp.log | tail -1; }
run "--config 2" A=1
run "--config 3" KKT_V6_K=1
run "--config 3" A=1
