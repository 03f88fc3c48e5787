set -x
python -m pytest tests/test_gpu_perdof.py -q -m gpu 2>&1 | tail -5
python - <<'PY'
import time, torch, json
from paper_2305_04421_b200 import problems as P
from paper_2305_04421_b200.solver import HeatKKT
p = P.config(1, coarse="per-dof")
t0 = time.time(); k = HeatKKT(p, mode="fast"); torch.cuda.synchronize(); ts = time.time() - t0
b = torch.from_numpy(P.kkt_rhs(1, p)).cuda(); x = torch.empty_like(b)
o = k.gmres_solve(b, x); torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); o = k.gmres_solve(b, x); e1.record(); torch.cuda.synchronize()
print("PERDOF_C1", json.dumps({"setup_s": ts, "iterations": o.iterations, "converged": o.converged, "relres": o.true_final_relres, "solve_ms": e0.elapsed_time(e1), "coarse_dim": k.coarse_dim(), "history": [float(h) for h in o.residual_history]}))
PY
python scripts/sanitize_case.py both > gpurun_out/sanitize_plain.log 2>&1 && \
timeout 1500 compute-sanitizer --tool racecheck --racecheck-report all python scripts/sanitize_case.py both > gpurun_out/racecheck_r02.log 2>&1
tail -5 gpurun_out/racecheck_r02.log
( time python scripts/golden_large_ops.py --config 4 --nt 8 --nd 4 --out-dir gpurun_out ) > gpurun_out/golden_c4.log 2>&1
tail -5 gpurun_out/golden_c4.log
