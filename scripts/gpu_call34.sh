mkdir -p gpurun_out
e2e() { echo "== e2e $*"; env "$@" KKT_E2E_TIM=1 timeout 900 python scripts/time_large.py --config 2 --reps 3 --e2e > gpurun_out/tmp.log 2>&1; grep "P_inv_host" gpurun_out/tmp.log | tail -1; grep e2e_ms gpurun_out/tmp.log | sed 's/.*apply_P_inv_ms/P_inv_ms/' | cut -c1-70; }
e2e A=1
e2e KKT_E2E_CHUNK_KB=0
e2e KKT_E2E_CHUNK_KB=16384
e2e KKT_E2E_CHUNK_KB=262144
run() { cfg=$1; shift; echo "== config $cfg $*"; env "$@" KKT_V6_TIM=1 timeout 900 python scripts/time_large.py $cfg --reps 3 > gpurun_out/tmp.log 2>&1; grep apply_P_inv_ms gpurun_out/tmp.log | sed 's/.*apply_P_inv_ms/P_inv_ms/' | cut -c1-60; grep "cycles/row\|placement\|grouping" gpurun_out/tmp.log | tail -4; }
run "--config 2" KKT_V6_STAGGER=1500
run "--config 2 --nd 32" KKT_V6_K=1
run "--config 2 --nd 32" A=1
timeout 1500 python -m pytest tests/test_gpu_v6_twist.py tests/test_gpu_v6.py -q -m gpu -x 2>&1 | tail -5
