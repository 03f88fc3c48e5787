"""Per-dof coarse pieces on intermediate sizes, device STRICT vs the compiled reference."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle.bindings import Ref  # noqa: E402
from paper_2305_04421_b200 import problems as P  # noqa: E402
from paper_2305_04421_b200.solver import HeatKKT  # noqa: E402

for (nx, nd, nt) in [(21, 4, 16), (17, 8, 16), (17, 16, 32), (32, 4, 64)]:
    p = P.Problem(Lx=1.0, Ly=1.0, Nx=nx, Ny=nx, Nt=nt, Nd=nd, omega=1e-2, coarse_variant="per-dof")
    k = HeatKKT(p, mode="strict")
    ref = Ref(p)
    r = P.random_vec(p.block, 31)
    c_ref = ref.coarse_restrict(r)
    s_ref = ref.coarse_solve(c_ref)
    s = k.coarse_solve(c_ref).cpu().numpy()
    d = np.abs(s - s_ref)
    msg = f"nx {nx} nd {nd} dim {k.coarse_dim()} solve_equal {np.array_equal(s, s_ref)} rel {d.max() / np.abs(s_ref).max():.3e}"
    if k.coarse_dim() <= 4096:
        msg += f" S0_equal {np.array_equal(k.coarse_matrix(), ref.coarse_matrix())}"
        S0 = ref.coarse_matrix()
        nz = np.nonzero(S0)
        msg += f" kl {int((nz[0] - nz[1]).max())} ku {int((nz[1] - nz[0]).max())}"
    print(msg, flush=True)
