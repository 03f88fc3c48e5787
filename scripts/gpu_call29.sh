set -x
mkdir -p gpurun_out
run() { cfg=$1; shift; echo "== config $cfg $*"; env "$@" KKT_V6_TIM=1 timeout 900 python scripts/time_large.py $cfg --reps 3 > gpurun_out/tmp.log 2>&1; grep apply_P_inv_ms gpurun_out/tmp.log | sed 's/.*apply_P_inv_ms/P_inv_ms/' | cut -c1-40; grep cycles gpurun_out/tmp.log | tail -2; grep "band windows\|grouping" gpurun_out/tmp.log | tail -2; }
run "--config 2" A=1
run "--config 2" KKT_V6_LATE2=1
run "--config 3" A=1
run "--config 3" KKT_V6_BFRAC=1.1
run "--config 3" KKT_V6_BFRAC=1.1 KKT_V6_K=2
run "--config 4 --nt 128 --T 0.125 --nd 16" A=1
run "--config 4 --nt 128 --T 0.125 --nd 16" KKT_V6_BFRAC=1.1
timeout 1500 python -m pytest tests/test_gpu_v6_twist.py tests/test_gpu_large.py -q -m gpu -x 2>&1 | tail -3
