set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_v6_twist.py -q -m gpu -x 2>&1 | tail -15
echo "== config 2 twist"; KKT_V6_TIM=1 timeout 600 python scripts/time_large.py --config 2 --reps 3 > gpurun_out/c2_tim.log 2>&1; grep -v cycles gpurun_out/c2_tim.log | head -20; grep cycles gpurun_out/c2_tim.log | tail -2
echo "== config 3 twist"; KKT_V6_TIM=1 timeout 600 python scripts/time_large.py --config 3 --reps 3 > gpurun_out/c3_tim.log 2>&1; grep -v cycles gpurun_out/c3_tim.log | head -20; grep cycles gpurun_out/c3_tim.log | tail -2
ncu --metrics gpu__time_duration.sum --clock-control none -c 700 --csv --log-file gpurun_out/launches_c2_twist.csv python scripts/time_large.py --config 2 --reps 1 > gpurun_out/ncu_c2.log 2>&1
python scripts/summarize_launches.py gpurun_out/launches_c2_twist.csv
KKT_E2E_TIM=1 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_twist.json 2> gpurun_out/bench_twist.err; grep P_inv_host gpurun_out/bench_twist.err | tail -3; python -c "
import json; d=json.load(open('gpurun_out/bench_twist.json')); print(d['ms_per_step'], d['value'], d['e2e'])"
