set -x
( time python -m pytest tests -q -m gpu ) > gpurun_out/pytest_gpu_r02_final.log 2>&1; tail -6 gpurun_out/pytest_gpu_r02_final.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r02.log 2>&1; tail -1 gpurun_out/smoke_r02.log
( time python bench.py --gpus 1 --steps 20 --warmup 5 ) > gpurun_out/bench_r02_driver.json 2> gpurun_out/bench_r02_driver.err; tail -3 gpurun_out/bench_r02_driver.err
( time python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 ) > gpurun_out/bench_r02_reference.json 2> gpurun_out/bench_r02_reference.err; tail -3 gpurun_out/bench_r02_reference.err
python bench.py --config 3 --pinv --steps 5 --warmup 3 --no-extras --no-cpu-baseline > gpurun_out/bench_r02_c3_pinv.json 2>/dev/null
python bench.py --config 1 --steps 5 --warmup 3 --no-extras > gpurun_out/bench_r02_c1_solve.json 2>/dev/null
