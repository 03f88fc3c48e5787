mkdir -p gpurun_out
run() { cfg=$1; shift; echo "== config $cfg $*"; env "$@" timeout 600 python scripts/time_large.py $cfg --reps 3 > gpurun_out/tmp.log 2>&1; grep apply_P_inv_ms gpurun_out/tmp.log | sed 's/.*"apply_K_ms/apply_K_ms/' | cut -c1-100; }
for nd in 8 32 128 256; do run "--config 3 --nd $nd" A=1; done
( time timeout 2400 python -m pytest tests/test_gpu_v6_twist.py tests/test_gpu_large.py tests/test_gpu_v6.py -q -m gpu -x ) > gpurun_out/pytest_gpu_r02_v6_after_preload.log 2>&1; tail -6 gpurun_out/pytest_gpu_r02_v6_after_preload.log
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_r02_final2_driver.json 2> gpurun_out/bench_final2.err; tail -c 300 gpurun_out/bench_r02_final2_driver.json
