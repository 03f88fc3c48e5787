set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_v6_twist.py tests/test_gpu_v6.py -q -m gpu -x 2>&1 | tail -5
run() { echo "== $*"; env "$@" KKT_V6_TIM=1 timeout 600 python scripts/time_large.py --config 2 --reps 3 > gpurun_out/tmp.log 2>&1; grep apply_P_inv_ms gpurun_out/tmp.log | sed 's/.*apply_P_inv_ms/P_inv_ms/' | cut -c1-40; grep cycles gpurun_out/tmp.log | tail -2; }
run A=1
run KKT_V6_NOPOLL=1
run KKT_V6_SPIN_NS=100
run KKT_V6_SPIN_NS=300
run KKT_V6_OFF=1
run KKT_V6_TWIST=0
KKT_E2E_TIM=1 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_twist.json 2> gpurun_out/bench_twist.err; grep P_inv_host gpurun_out/bench_twist.err | tail -2; python -c "
import json; d=json.load(open('gpurun_out/bench_twist.json')); print(d['ms_per_step'], d['value'], d['e2e'])"
KKT_BENCH_PROFILE=1 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none -c 700 --csv --log-file gpurun_out/launches_c2_twist.csv python bench.py --steps 2 --warmup 1 > gpurun_out/ncu_c2.log 2>&1
python scripts/summarize_launches.py gpurun_out/launches_c2_twist.csv
