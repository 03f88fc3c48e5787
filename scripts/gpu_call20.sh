set -x
for i in 1 2; do echo "== config 3"; python scripts/time_large.py --config 3 --reps 5 2>&1 | tail -1; done
echo "== config 3 noband"; KKT_V6_NOBAND=1 python scripts/time_large.py --config 3 --reps 5 2>&1 | tail -1
echo "== config 2"; python scripts/time_large.py --config 2 --reps 5 2>&1 | tail -1
