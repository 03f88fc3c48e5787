mkdir -p gpurun_out
run() { cfg=$1; shift; echo "== config $cfg $*"; env "$@" KKT_V6_TIM=1 timeout 600 python scripts/time_large.py $cfg --reps 3 > gpurun_out/tmp.log 2>&1; grep apply_P_inv_ms gpurun_out/tmp.log | sed 's/.*apply_P_inv_ms/P_inv_ms/' | cut -c1-60; grep "elimination form\|grouping" gpurun_out/tmp.log | tail -2; tail -3 gpurun_out/tmp.log | grep -i "error\|Traceback" ; }
run "--config 3" A=1
run "--config 3" KKT_V6_THOMAS=0
timeout 2400 python -m pytest tests/test_gpu_v6_twist.py tests/test_gpu_large.py tests/test_gpu_v6.py -q -m gpu -x 2>&1 | tail -15
run "--config 3 --nd 128" A=1
run "--config 3 --nd 128" KKT_V6_THOMAS=0
run "--config 3 --nd 8" A=1
run "--config 3 --nd 8" KKT_V6_THOMAS=0
run "--config 2" A=1
