mkdir -p gpurun_out
e2e() { echo "== e2e $*"; env "$@" KKT_E2E_TIM=1 timeout 900 python scripts/time_large.py --config 2 --reps 3 --e2e > gpurun_out/tmp.log 2>&1; grep "P_inv_host" gpurun_out/tmp.log | tail -2; grep e2e_ms gpurun_out/tmp.log | sed 's/.*apply_P_inv_ms/P_inv_ms/' | cut -c1-70; }
e2e A=1
e2e KKT_E2E_CHUNK_KB=0
e2e KKT_E2E_CHUNK_KB=16384
timeout 900 python -m pytest tests/test_gpu_v6_twist.py -q -m gpu -x -k "host_pinv" 2>&1 | tail -3
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x 2>&1 | tail -3
python scripts/time_large.py --config 2 --reps 1 > gpurun_out/tl_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:'v6_(chainw|off3|form_b|mid)' -s 40 -c 10 -o gpurun_out/ncu_v6_c2_r02_late python scripts/time_large.py --config 2 --reps 1 > gpurun_out/ncu_v6.log 2>&1
ls -la gpurun_out/*.ncu-rep
