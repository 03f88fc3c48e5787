"""Diagnostic: FAST vs STRICT (bitwise the reference) GMRES on the config-3 grid
with a reduced time axis, to tell a method property from a kernel bug when a
solve stagnates.

    python scripts/diag_c3solve.py --nt 512 --nd 256 [--max-iters 200]
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2305_04421_b200 import problems as P  # noqa: E402
from paper_2305_04421_b200.solver import HeatKKT  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--nt", type=int, default=512)
ap.add_argument("--nd", type=int, default=256)
ap.add_argument("--max-iters", type=int, default=200)
ap.add_argument("--modes", default="fast,strict")
ap.add_argument("--T", type=float, default=None, help="final time (keep config 3's dt: T = nt / 4096)")
a = ap.parse_args()
p = P.config(3, Nd=a.nd).replace(Nt=a.nt, max_iters=a.max_iters)
if a.T:
    p = p.replace(T=a.T)
b = torch.from_numpy(P.kkt_rhs(3, p)).cuda()
for mode in a.modes.split(","):
    k = HeatKKT(p, mode=mode)
    t0 = time.time()
    o = k.gmres_solve(b)
    torch.cuda.synchronize()
    h = list(o.residual_history)
    print(f"{mode}: Nt={p.Nt} Nd={p.Nd} its={o.iterations} conv={o.converged} relres={o.true_final_relres:.3e} "
          f"t={time.time() - t0:.1f}s hist[0,10,20,40,-1]={[h[i] for i in (0, 10, 20, 40, -1) if i < len(h)]}",
          flush=True)
    print(mode, "history", [float(f"{v:.6e}") for v in h], flush=True)
    del k
