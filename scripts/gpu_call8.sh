set -x
python -m pytest tests/test_gpu_perdof.py tests/test_gpu_v6.py -q -m gpu -x 2>&1 | tail -15
echo "== config 2 NG4"; python scripts/time_large.py --config 2 --reps 3 2>&1 | tail -1
echo "== config 2 NG2"; KKT_V6_OFF_NG2=1 python scripts/time_large.py --config 2 --reps 3 2>&1 | tail -1
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
print("PERDOF_C1", json.dumps({"setup_s": ts, "iterations": o.iterations, "converged": o.converged, "relres": o.true_final_relres, "solve_ms": e0.elapsed_time(e1), "coarse_dim": k.coarse_dim()}))
PY
