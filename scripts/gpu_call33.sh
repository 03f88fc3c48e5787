set -x
mkdir -p gpurun_out
run() { cfg=$1; shift; echo "== config $cfg $*"; env "$@" KKT_V6_TIM=1 timeout 900 python scripts/time_large.py $cfg --reps 3 > gpurun_out/tmp.log 2>&1; grep apply_P_inv_ms gpurun_out/tmp.log | sed 's/.*apply_P_inv_ms/P_inv_ms/' | cut -c1-60; grep "cycles/row" gpurun_out/tmp.log | tail -2; }
for st in 0 800 1500 2200 3000; do run "--config 2" KKT_V6_STAGGER=$st; done
e2e() { echo "== e2e $*"; env "$@" KKT_E2E_TIM=1 timeout 900 python scripts/time_large.py --config 2 --reps 3 --e2e > gpurun_out/tmp.log 2>&1; grep "P_inv_host" gpurun_out/tmp.log | tail -1; grep e2e_ms gpurun_out/tmp.log | sed 's/.*e2e_ms/e2e_ms/' | cut -c1-30; }
e2e A=1
e2e KKT_E2E_TRAIL_OFF=1
e2e KKT_E2E_SCHED=1
e2e KKT_E2E_SCHED=2
e2e KKT_E2E_SCHED=4
e2e KKT_E2E_SCHED=4 KKT_E2E_TRAIL_OFF=1
