set -x
python -m pytest tests/test_gpu_v6.py tests/test_gpu_large.py -q -m gpu -x 2>&1 | tail -6
echo "== config 2"; KKT_V6_TIM=1 python scripts/time_large.py --config 2 --reps 3 2>&1 | tail -3
echo "== config 3 k auto"; KKT_V6_TIM=1 python scripts/time_large.py --config 3 --reps 3 2>&1 | grep -v cycles | tail -3
echo "== config 3 k4"; KKT_V6_K=4 python scripts/time_large.py --config 3 --reps 3 2>&1 | tail -1
echo "== config 3 k5"; KKT_V6_K=5 python scripts/time_large.py --config 3 --reps 3 2>&1 | tail -1
echo "== bench e2e check"; python bench.py --steps 3 --warmup 3 --no-extras --no-cpu-baseline 2>/dev/null | python -c "import sys,json; d=json.loads([l for l in sys.stdin if l.startswith('{')][-1]); print('ms', d['ms_per_step'], 'e2e', d['e2e'], 'stencil', d['roofline_stencil']['frac'], 'roof', d['roofline']['frac'])"
python scripts/sanitize_case.py all > gpurun_out/sanitize_plain2.log 2>&1 && \
timeout 1500 compute-sanitizer --tool memcheck python scripts/sanitize_case.py all > gpurun_out/memcheck_r02.log 2>&1
tail -4 gpurun_out/memcheck_r02.log
