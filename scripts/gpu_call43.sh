mkdir -p gpurun_out
( time python -m pytest tests -q -m gpu -x ) > gpurun_out/pytest_gpu_r02_final.log 2>&1; tail -6 gpurun_out/pytest_gpu_r02_final.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r02_final.log 2>&1; tail -2 gpurun_out/smoke_r02_final.log
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_r02_final_reference.json 2> gpurun_out/bench_ref.err; tail -c 300 gpurun_out/bench_r02_final_reference.json
KKT_E2E_TIM=1 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_r02_final_driver.json 2> gpurun_out/bench_final.err; tail -c 600 gpurun_out/bench_r02_final_driver.json; grep P_inv_host gpurun_out/bench_final.err | tail -3
KKT_BENCH_PROFILE=1 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r02_final_c2.csv python bench.py --steps 2 --warmup 1 --no-extras --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1
python scripts/summarize_launches.py gpurun_out/launches_r02_final_c2.csv > gpurun_out/launches_r02_final_c2_summary.txt; cat gpurun_out/launches_r02_final_c2_summary.txt
ncu --set full --clock-control none --import-source on -k regex:'v6_(chainw|form_b|mid)' -s 40 -c 8 -o gpurun_out/ncu_v6_c2_r02_final python scripts/time_large.py --config 2 --reps 1 > gpurun_out/ncu_v6.log 2>&1
ls -la gpurun_out/*.ncu-rep
