set -x
( time python -m pytest tests -q -m gpu -x ) > gpurun_out/pytest_gpu_r02.log 2>&1; tail -8 gpurun_out/pytest_gpu_r02.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r02.log 2>&1; tail -2 gpurun_out/smoke_r02.log
python bench.py --steps 2 --warmup 1 --no-extras --no-cpu-baseline > gpurun_out/bench_plain.json 2> gpurun_out/bench_plain.err && \
KKT_BENCH_PROFILE=1 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r02_bench_c2.csv python bench.py --steps 2 --warmup 1 --no-extras --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1
python scripts/time_large.py --config 2 --reps 1 > gpurun_out/tl_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:'v6_(chain|off2|form_b)' -s 30 -c 8 -o gpurun_out/ncu_v6_c2_r02 python scripts/time_large.py --config 2 --reps 1 > gpurun_out/ncu_v6.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:'apply_K_kernel' -s 1 -c 1 -o gpurun_out/ncu_k1_c2_r02 python scripts/time_large.py --config 2 --reps 1 > gpurun_out/ncu_k1c2.log 2>&1
python scripts/prof_solve.py > gpurun_out/ps_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:'apply_K_kernel|cgs_dots_kernel|cgs_update_kernel' -s 12 -c 6 -o gpurun_out/ncu_k1_cgs_r02 python scripts/prof_solve.py > gpurun_out/ncu_k1.log 2>&1
ls -la gpurun_out/*.ncu-rep
