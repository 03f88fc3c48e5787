set -x
python -m pytest tests/test_gpu_cpp_shim.py tests/test_gpu_v6.py tests/test_gpu_large.py tests/test_gpu_errors.py -q -m gpu 2>&1 | tail -15
for ll in 1 0; do
  echo "== config 3, KKT_V6_LL=$ll"; KKT_V6_LL=$ll python scripts/time_large.py --config 3 --reps 3 2>&1 | tail -1
  echo "== config 2, KKT_V6_LL=$ll"; KKT_V6_LL=$ll python scripts/time_large.py --config 2 --reps 3 2>&1 | tail -1
done
echo "== config 1"; python scripts/time_large.py --config 1 --reps 20 2>&1 | tail -1
echo "== c4 slab"; python scripts/time_large.py --config 4 --nt 128 --T 0.125 --nd 16 --reps 3 2>&1 | tail -1
python bench.py --steps 5 --warmup 3 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; tail -c 1500 gpurun_out/bench_c2.err
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; cat gpurun_out/bench_ref.json | cut -c1-1500
python bench.py --gpus 2 --steps 1 --warmup 1 2>&1 | tail -3
