set -x
python -m pytest tests/test_gpu_cpp_shim.py tests/test_gpu_v6.py tests/test_gpu_large.py tests/test_gpu_v5.py tests/test_gpu_sharded.py -q -m gpu 2>&1 | tail -30
for k in auto 1 2 4; do
  if [ $k = auto ]; then unset KKT_V6_K; else export KKT_V6_K=$k; fi
  echo "== config 3, KKT_V6_K=$k"; KKT_V6_TIM=1 python scripts/time_large.py --config 3 --reps 3 2>&1 | grep -v "cycles/row" | tail -4
done
unset KKT_V6_K
echo "== config 2"; python scripts/time_large.py --config 2 --reps 3 2>&1 | tail -2
echo "== config 1"; python scripts/time_large.py --config 1 --reps 20 2>&1 | tail -1
python scripts/solve_large.py --config 3 --nd 8 --max-iters 100 --out gpurun_out/solve_c3_nd8.json 2>&1 | tail -1 | cut -c1-600
python scripts/solve_large.py --config 3 --nd 16 --max-iters 100 --out gpurun_out/solve_c3_nd16.json 2>&1 | tail -1 | cut -c1-600
