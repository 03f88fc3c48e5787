set -x
echo "== config 2"; KKT_V6_TIM=1 python scripts/time_large.py --config 2 --reps 3 2>&1 | tail -3
echo "== config 3"; python scripts/time_large.py --config 3 --reps 3 2>&1 | tail -1
echo "== c4 slab"; python scripts/time_large.py --config 4 --nt 128 --T 0.125 --nd 16 --reps 3 2>&1 | tail -1
python -m pytest tests/test_gpu_v6.py -q -m gpu -x 2>&1 | tail -4
