"""Small P^-1 applications for compute-sanitizer (racecheck / memcheck): one
case on the v4 cluster sweep (nx <= 128) and one on the v6 device-wide sweep
(nx > 128), FAST mode, each applied twice and compared (determinism).

    compute-sanitizer --tool racecheck python scripts/sanitize_case.py [v4|v6|v6b|both|all]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2305_04421_b200 import problems as P  # noqa: E402
from paper_2305_04421_b200.solver import HeatKKT  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "both"
cases = []
if which in ("v4", "both", "all"):
    cases.append(("v4", P.Problem(Lx=1.0, Ly=1.0, Nx=25, Ny=21, Nt=8, Nd=4, omega=1e-2, coarse_variant="scalar")))
if which in ("v6", "both", "all"):
    cases.append(("v6", P.Problem(Lx=1.0, Ly=1.0, Nx=141, Ny=13, Nt=4, Nd=2, omega=1e-2, coarse_variant="scalar")))
if which in ("v6b", "all"):
    # 512-blocks, 24 chains = 3 chain groups: the 4-groups-per-pass off-chain kernel, grouping, packets
    cases.append(("v6b", P.Problem(Lx=1.0, Ly=1.0, Nx=301, Ny=6, Nt=24, Nd=24, nu=0.1, omega=1e-2, coarse_variant="scalar")))
for name, p in cases:
    k = HeatKKT(p, mode="fast")
    r = torch.from_numpy(P.random_vec(3 * p.block, 5)).cuda()
    a = k.apply_P_inv(r).clone()
    b = k.apply_P_inv(r).clone()
    torch.cuda.synchronize()
    print(name, "P_inv twice equal:", bool(torch.equal(a, b)), "finite:", bool(torch.isfinite(a).all()), flush=True)
