set -x
mkdir -p gpurun_out
run() { echo "== $*"; env "$@" KKT_V6_TIM=1 timeout 600 python scripts/time_large.py --config 2 --reps 3 > gpurun_out/tmp.log 2>&1; grep apply_P_inv_ms gpurun_out/tmp.log | sed 's/.*apply_P_inv_ms/P_inv_ms/' | cut -c1-40; grep cycles gpurun_out/tmp.log | tail -2; grep "band windows" gpurun_out/tmp.log | tail -1; }
run A=1
run KKT_V6_PHASE_NS=400
run KKT_V6_PHASE_NS=800
run KKT_V6_PHASE_NS=1200
run KKT_V6_BTOL=1e-15
run KKT_V6_BTOL=1e-14
run KKT_V6_TWIST=0
KKT_V6_BTOL=1e-15 timeout 900 python -m pytest tests/test_gpu_large.py -q -m gpu -x 2>&1 | tail -3
