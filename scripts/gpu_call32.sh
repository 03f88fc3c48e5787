set -x
mkdir -p gpurun_out
run() { cfg=$1; shift; echo "== config $cfg $*"; env "$@" KKT_V6_TIM=1 timeout 900 python scripts/time_large.py $cfg --reps 3 > gpurun_out/tmp.log 2>&1; grep apply_P_inv_ms gpurun_out/tmp.log | sed 's/.*apply_P_inv_ms/P_inv_ms/' | cut -c1-40; cp gpurun_out/tmp.log gpurun_out/tim_$(echo "$cfg $*" | tr -c 'A-Za-z0-9\n' '_').log; }
run "--config 2" A=1
run "--config 2" KKT_V6_OFF3=1
run "--config 3" A=1
run "--config 3" KKT_V6_OFF3=1
run "--config 4 --nt 128 --T 0.125 --nd 16" A=1
run "--config 4 --nt 128 --T 0.125 --nd 16" KKT_V6_OFF3=1
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; tail -c 3000 gpurun_out/bench_default.json
