"""Why does GMRES(20) stagnate at config 3 on BASELINE's seeded inputs?

    python scripts/diag_c3_inputs.py [--nd 32] [--out gpurun_out/diag_c3_inputs.json]

On the full config-3 problem (255^2 x 4096, FAST):
  A. P^-1 and K as linear operators: ||Op(a x + b y) - a Op(x) - b Op(y)|| / ||.||
     and run-to-run determinism, on seeded N(0,1) vectors;
  B. one GMRES(20) cycle on BASELINE's right-hand side (noisy target) and on
     the paper's model right-hand side: the recurrence's residual estimate next
     to the recomputed true residual (they agree unless ||y|| blows up);
  C. the right-hand side split into its smooth part (noise off) and its noise
     part: one cycle each, to see which part GMRES cannot reduce.
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import numpy as np
    import torch
    from paper_2305_04421_b200 import problems as P
    from paper_2305_04421_b200.solver import HeatKKT

    ap = argparse.ArgumentParser()
    ap.add_argument("--nd", type=int, default=32)
    ap.add_argument("--nt", type=int, default=None)
    ap.add_argument("--cycles", type=int, default=1)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    p = P.config(3, Nd=a.nd)
    if a.nt:
        p = p.replace(Nt=a.nt, T=a.nt / 4096.0)
    p1 = p.replace(max_iters=20 * a.cycles)
    B = p.block
    rec = {"Nd": p.Nd, "Nt": p.Nt}
    k = HeatKKT(p1, mode="fast")

    def rel(x, y):
        return float((x - y).norm() / y.norm())

    # ---- A
    g = torch.Generator(device="cuda").manual_seed(1)
    x = torch.randn(3 * B, dtype=torch.float64, device="cuda", generator=g)
    y = torch.randn(3 * B, dtype=torch.float64, device="cuda", generator=g)
    al, be = 0.37, -2.25
    for name, op in (("P_inv", k.apply_P_inv), ("K", k.apply_K)):
        ox = op(x).clone()
        oy = op(y).clone()
        oc = op(al * x + be * y).clone()
        lin = al * ox + be * oy
        rec[name + "_linearity_per_block"] = [rel(oc[i * B:(i + 1) * B], lin[i * B:(i + 1) * B]) for i in range(3)]
        rec[name + "_deterministic"] = bool(torch.equal(op(x), ox))
        del ox, oy, oc, lin
    del x, y
    torch.cuda.empty_cache()
    print(json.dumps(rec), flush=True)

    # ---- B, C
    tgt, u0 = P.target_and_u0(3, p)
    ms = p.mass_scale
    b_full = np.zeros(3 * B)
    b_full[:B] = (ms * tgt).reshape(-1)
    del tgt
    xg, yg = P._grid(p)
    X = np.tile(xg, p.ny_int)
    Y = np.repeat(yg, p.nx_int)
    t = np.arange(1, p.Nt + 1, dtype=np.float64) * p.dt
    smooth = np.cos(2 * np.pi * t)[:, None] * (np.sin(np.pi * X) * np.sin(np.pi * Y))[None, :]
    b_smooth = np.zeros(3 * B)
    b_smooth[:B] = (ms * smooth).reshape(-1)
    del smooth
    b_noise = b_full - b_smooth
    b_model, _ = k.model_rhs()
    for name, bh in (("baseline_rhs", b_full), ("smooth_part", b_smooth), ("noise_part", b_noise),
                     ("model_rhs", b_model)):
        b = torch.from_numpy(bh).cuda()
        o = k.gmres_solve(b)
        h = o.residual_history
        rec[name] = {"iterations": o.iterations, "estimate_last": float(h[-1]),
                     "true_relres": o.true_final_relres,
                     "history": [float(v) for v in h]}
        print(name, o.iterations, "estimate", float(h[-1]), "true", o.true_final_relres, flush=True)
        del b, o
        torch.cuda.empty_cache()
    if a.out:
        json.dump(rec, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
