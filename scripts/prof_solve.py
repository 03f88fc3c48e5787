"""Profile helper: one full FAST (or --mode) GMRES solve of a BASELINE config
between cudaProfilerStart/Stop, after one untimed warm-up solve, so that
`ncu --profile-from-start off` captures exactly the launches of one solve.

    ncu --profile-from-start off --metrics gpu__time_duration.sum \
        --clock-control none --csv --log-file L.csv python scripts/prof_solve.py
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2305_04421_b200 import problems as P  # noqa: E402
from paper_2305_04421_b200.solver import HeatKKT  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=1)
ap.add_argument("--mode", default="fast")
a = ap.parse_args()
p = P.config(a.config)
k = HeatKKT(p, mode=a.mode)
b = torch.from_numpy(P.kkt_rhs(a.config, p)).cuda()
x = torch.empty_like(b)
k.gmres_solve(b, x)
torch.cuda.synchronize()
l0 = k.launch_count()
torch.cuda.profiler.start()
out = k.gmres_solve(b, x)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print(f"solve: {out.iterations} iterations, relres {out.true_final_relres:.3e}, "
      f"{k.launch_count() - l0} launches of this library")
