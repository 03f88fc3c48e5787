set -x
for ll in 1 0; do
  echo "== config 2, KKT_V6_LL=$ll"; KKT_V6_LL=$ll KKT_V6_TIM=1 python scripts/time_large.py --config 2 --reps 3 2>&1 | tail -5
done
echo "== c4 slab LL=0"; KKT_V6_LL=0 python scripts/time_large.py --config 4 --nt 128 --T 0.125 --nd 16 --reps 3 2>&1 | tail -1
echo "== config 3"; python scripts/time_large.py --config 3 --reps 3 2>&1 | tail -1
for tp in 16 8; do echo "== config 1 K1 tp=$tp"; KKT_K1_TP=$tp python scripts/time_large.py --config 1 --reps 30 2>&1 | tail -1; done
python -m pytest tests/test_gpu_v6.py tests/test_gpu_large.py tests/test_gpu_cpp_shim.py -q -m gpu 2>&1 | tail -5
