mkdir -p gpurun_out
run() { cfg=$1; shift; echo "== config $cfg $*"; env "$@" KKT_V6_TIM=1 timeout 600 python scripts/time_large.py $cfg --reps 3 > gpurun_out/tmp.log 2>&1; grep apply_P_inv_ms gpurun_out/tmp.log | sed 's/.*apply_P_inv_ms/P_inv_ms/' | cut -c1-60; grep "cycles/row" gpurun_out/tmp.log | tail -2; tail -3 gpurun_out/tmp.log | grep -i "error\|Traceback" ; }
KKT_V6_THOMAS=1 timeout 1500 python -m pytest tests/test_gpu_v6_twist.py -q -m gpu -x 2>&1 | tail -15
run "--config 2" A=1
run "--config 2" KKT_V6_THOMAS=1
KKT_V6_THOMAS=1 timeout 1500 python -m pytest tests/test_gpu_large.py -q -m gpu -x 2>&1 | tail -15
run "--config 4 --nt 128 --T 0.125 --nd 16" A=1
run "--config 4 --nt 128 --T 0.125 --nd 16" KKT_V6_THOMAS=1
