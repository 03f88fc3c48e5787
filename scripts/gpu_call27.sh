set -x
mkdir -p gpurun_out _head/gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit,temperature.gpu,serial --format=csv
run() { echo "== $*"; env "$@" KKT_V6_TIM=1 timeout 600 python scripts/time_large.py --config 2 --reps 3 > gpurun_out/tmp.log 2>&1; grep apply_P_inv_ms gpurun_out/tmp.log | sed 's/.*apply_P_inv_ms/P_inv_ms/' | cut -c1-40; grep cycles gpurun_out/tmp.log | tail -2; }
(cd _head && echo "HEAD build" && run A=1)
run A=1
(cd _head && echo "HEAD build again" && run A=1)
run A=2
timeout 900 python -m pytest tests/test_gpu_v6_twist.py -q -m gpu -x 2>&1 | tail -3
KKT_BENCH_PROFILE=1 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none -c 700 --csv --log-file gpurun_out/launches_c2_twist.csv python bench.py --steps 2 --warmup 1 > gpurun_out/ncu_c2.log 2>&1
python scripts/summarize_launches.py gpurun_out/launches_c2_twist.csv
