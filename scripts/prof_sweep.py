"""Profile helper: a few two-level Schur applies (the RASQ sweep + coarse
kernels) and K applies at a BASELINE config, for ncu captures.

    python scripts/prof_sweep.py [--config 1] [--reps 3] [--mode fast]
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
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--mode", default="fast")
a = ap.parse_args()
p = P.config(a.config)
k = HeatKKT(p, mode=a.mode)
r = torch.from_numpy(P.random_vec(3 * p.block, 5)).cuda()
out = torch.empty_like(r)
for _ in range(a.reps):
    k.apply_P_inv(r, out)
    k.apply_K(r, out)
torch.cuda.synchronize()
ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ev0.record()
for _ in range(a.reps):
    k.apply_P_inv(r, out)
ev1.record()
torch.cuda.synchronize()
print(f"P_inv apply: {ev0.elapsed_time(ev1) / a.reps:.3f} ms")
ev0.record()
for _ in range(a.reps):
    k.apply_K(r, out)
ev1.record()
torch.cuda.synchronize()
print(f"K apply: {ev0.elapsed_time(ev1) / a.reps:.3f} ms")
k.set_phase_timing(True)
k.apply_P_inv(r, out)
torch.cuda.synchronize()
print("phase ms (0 K, 1 P_inv, 2 Krylov, 3 sweep kernel):", k.phase_times())
