mkdir -p gpurun_out
( time python -m pytest tests -q -m gpu -x ) > gpurun_out/pytest_gpu_r02_final.log 2>&1; tail -6 gpurun_out/pytest_gpu_r02_final.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r02_final.log 2>&1; tail -2 gpurun_out/smoke_r02_final.log
