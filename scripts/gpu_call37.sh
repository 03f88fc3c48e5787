mkdir -p gpurun_out
run() { cfg=$1; shift; echo "== config $cfg $*"; env "$@" KKT_V6_TIM=1 timeout 900 python scripts/time_large.py $cfg --reps 3 > gpurun_out/tmp.log 2>&1; grep apply_P_inv_ms gpurun_out/tmp.log | sed 's/.*apply_P_inv_ms/P_inv_ms/' | cut -c1-60; grep "cycles/row\|band windows\|jstar\|grouping" gpurun_out/tmp.log | tail -5; }
run "--config 3" A=1
run "--config 3" KKT_V6_CFRAC=1.01
run "--config 3" KKT_V6_BFRAC=1.01
run "--config 3" KKT_V6_CFRAC=1.01 KKT_V6_K=2
run "--config 3" KKT_V6_CFRAC=1.01 KKT_V6_K=3
run "--config 3 --nd 8" A=1
run "--config 3 --nd 8" KKT_V6_CFRAC=1.01
run "--config 3 --nd 128" A=1
run "--config 3 --nd 128" KKT_V6_CFRAC=1.01
