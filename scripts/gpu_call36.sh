mkdir -p gpurun_out
run() { cfg=$1; shift; echo "== config $cfg $*"; env "$@" KKT_V6_TIM=1 timeout 900 python scripts/time_large.py $cfg --reps 3 > gpurun_out/tmp.log 2>&1; grep apply_P_inv_ms gpurun_out/tmp.log | sed 's/.*apply_P_inv_ms/P_inv_ms/' | cut -c1-60; grep "cycles/row" gpurun_out/tmp.log | tail -2; }
run "--config 2" A=1
run "--config 2" KKT_V6_NOHOLD=1
timeout 1800 python -m pytest tests/test_gpu_v6_twist.py tests/test_gpu_v6.py tests/test_gpu_large.py -q -m gpu -x 2>&1 | tail -5
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3_tl.csv python scripts/time_large.py --config 3 --reps 1 > gpurun_out/ncu_c3.log 2>&1
python scripts/summarize_launches.py gpurun_out/launches_c3_tl.csv | head -30
