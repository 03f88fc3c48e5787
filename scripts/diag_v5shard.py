"""Diagnostic: residual-history drift between a single-rank FAST solve and a
2-virtual-rank sharded FAST solve of the same problem, for a v5 grid (nx = 149)
and a v4 grid (nx = 119).  The sharded operators are bitwise the single-rank
ones (tests/test_gpu_sharded.py); only the per-rank dot sums round differently.

    python scripts/diag_v5shard.py
"""
import sys, os
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import numpy as np, torch
from paper_2305_04421_b200 import problems as P
from paper_2305_04421_b200.solver import HeatKKT
from test_gpu_sharded import run_ranks, host
for nx in (150, 120):
    p = P.Problem(Lx=1.0, Ly=1.0, Nx=nx, Ny=140, Nt=16, Nd=4, nu=1.0, omega=1e-1, coarse_variant="scalar", tol=1e-8, restart=20, max_iters=300)
    b = P.random_vec(3 * p.block, 43)
    ref = HeatKKT(p, mode="fast").gmres_solve(b)
    res = run_ranks(p, 2, lambda k, r: (k.gmres_solve(k.local_slab(b)).residual_history))
    h1 = np.array(ref.residual_history); h2 = np.array(res[0])
    n = min(len(h1), len(h2))
    print(nx, "iters", len(h1), len(h2))
    print(" rel diff of history:", [f"{abs(h1[i]-h2[i])/h1[i]:.1e}" for i in range(0, n, max(1, n // 12))])
