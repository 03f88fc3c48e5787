"""v6 (nx > 511) diagnostics: full-GMRES solve FAST vs STRICT on a 1023-wide
grid, and a timing run at config 4's row width with a short y axis.

    python scripts/diag_v6.py solve|time
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import numpy as np
    import torch
    from paper_2305_04421_b200 import problems as P
    from paper_2305_04421_b200.solver import HeatKKT
    what = sys.argv[1]
    if what == "solve":
        for restart in (20, 200):
            p = P.Problem(Lx=1.0, Ly=1.0, Nx=1024, Ny=4, Nt=16, Nd=4, nu=1.0, omega=1e-2, precond="two-level",
                          coarse_variant="scalar", tol=1e-8, restart=restart, max_iters=200)
            b = P.kkt_rhs(0, p)
            f = HeatKKT(p, mode="fast").gmres_solve(b)
            s = HeatKKT(p, mode="strict").gmres_solve(b)
            x, y = f.solution.cpu().numpy(), s.solution.cpu().numpy()
            B = p.block
            print(json.dumps({"restart": restart, "fast_its": f.iterations, "strict_its": s.iterations,
                              "fast_relres": f.true_final_relres, "strict_relres": s.true_final_relres,
                              "rel_x": [float(np.linalg.norm(x[k*B:(k+1)*B] - y[k*B:(k+1)*B]) / np.linalg.norm(y[k*B:(k+1)*B])) for k in range(3)],
                              "hist_fast": [float(h) for h in f.residual_history[:12]],
                              "hist_strict": [float(h) for h in s.residual_history[:12]]}), flush=True)
    else:
        ny = int(sys.argv[2]) if len(sys.argv) > 2 else 128
        p = P.config(4).replace(Ny=ny + 1, Nt=128, Nd=16)
        t0 = time.time()
        k = HeatKKT(p, mode="fast")
        torch.cuda.synchronize()
        st = time.time() - t0
        v = torch.randn(3 * p.block, dtype=torch.float64, device="cuda")
        o = torch.empty_like(v)
        k.apply_P_inv(v, o)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        k.apply_P_inv(v, o)
        e1.record()
        torch.cuda.synchronize()
        print(json.dumps({"ny": p.ny_int, "setup_s": st, "P_inv_ms": e0.elapsed_time(e1)}), flush=True)


if __name__ == "__main__":
    main()
