mkdir -p gpurun_out
run() { cfg=$1; shift; echo "== config $cfg $*"; env "$@" KKT_V6_TIM=1 timeout 600 python scripts/time_large.py $cfg --reps 3 > gpurun_out/tmp.log 2>&1; grep apply_P_inv_ms gpurun_out/tmp.log | sed 's/.*"setup_s/setup_s/' | cut -c1-130; grep "grouping\|jstar" gpurun_out/tmp.log | tail -2; }
for nd in 8 32 128 256; do run "--config 3 --nd $nd" A=1; done
run "--config 4 --nt 128 --T 0.125 --nd 16" A=1
python scripts/time_large.py --config 3 --reps 1 > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r02_final_c3.csv python scripts/time_large.py --config 3 --reps 1 > gpurun_out/ncu_c3.log 2>&1
python scripts/summarize_launches.py gpurun_out/launches_r02_final_c3.csv > gpurun_out/launches_r02_final_c3_summary.txt; head -24 gpurun_out/launches_r02_final_c3_summary.txt
