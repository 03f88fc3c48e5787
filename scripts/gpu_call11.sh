set -x
echo "== config 2"; python scripts/time_large.py --config 2 --reps 3 2>&1 | tail -1
echo "== config 3"; python scripts/time_large.py --config 3 --reps 3 2>&1 | tail -1
KKT_E2E_TIM=1 python bench.py --steps 3 --warmup 3 --no-extras --no-cpu-baseline 2> gpurun_out/e2e_tim.err | python -c "import sys,json; d=json.loads([l for l in sys.stdin if l.startswith('{')][-1]); print('ms', d['ms_per_step'], 'e2e', d['e2e'])"
grep P_inv_host gpurun_out/e2e_tim.err | tail -3
