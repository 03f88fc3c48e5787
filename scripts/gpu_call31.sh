set -x
mkdir -p gpurun_out
run() { cfg=$1; shift; echo "== config $cfg $*"; env "$@" KKT_V6_TIM=1 timeout 900 python scripts/time_large.py $cfg --reps 3 > gpurun_out/tmp.log 2>&1; grep apply_P_inv_ms gpurun_out/tmp.log | sed 's/.*apply_P_inv_ms/P_inv_ms/' | cut -c1-40; }
run "--config 2" A=1
run "--config 2" KKT_V6_OFF3=1
run "--config 4 --nt 128 --T 0.125 --nd 16" A=1
run "--config 4 --nt 128 --T 0.125 --nd 16" KKT_V6_OFF3=1
KKT_V6_OFF3=1 timeout 1500 python -m pytest tests/test_gpu_v6_twist.py tests/test_gpu_v6.py tests/test_gpu_large.py -q -m gpu -x 2>&1 | tail -3
KKT_V6_OFF3=1 KKT_BENCH_PROFILE=1 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none -c 700 --csv --log-file gpurun_out/launches_c2_off3.csv python bench.py --steps 2 --warmup 1 > gpurun_out/ncu_c2.log 2>&1
python scripts/summarize_launches.py gpurun_out/launches_c2_off3.csv
