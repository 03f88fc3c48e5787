"""Full GMRES solve of a large BASELINE config (3 by default) on its OWN seeded
inputs (P.kkt_rhs: u~ = sin(pi x) sin(pi y) cos(2 pi t) + 0.01 N(0,1), u0 = 0 at
config 3), through kkt_gmres_solve -- not run_single's model problem.

    python scripts/solve_large.py --config 3 --nd 32 [--out profiles/solve_c3_nd32_r02.json]

Prints one JSON record: iterations, true relative residual, solve time (CUDA
events), per-phase device times, the residual history.
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def slab_rhs(cfg, p, node_first, node_last):
    """b = [f_u; f_z; f] (kkt.cpp:21-48) for nodes node_first..node_last."""
    import numpy as np
    from paper_2305_04421_b200 import problems as P
    tgt, u0 = P.target_and_u0(cfg, p, n_lo=node_first, n_hi=node_last)
    L = (node_last - node_first + 1) * p.n_sp
    b = np.zeros(3 * L)
    b[:L] = (p.mass_scale * tgt).reshape(-1)
    if node_first == 1:
        b[2 * L: 2 * L + p.n_sp] = u0
    return b


def main():
    import numpy as np
    import torch
    from paper_2305_04421_b200 import problems as P
    from paper_2305_04421_b200.solver import HeatKKT

    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--nd", type=int, default=None)
    ap.add_argument("--nt", type=int, default=None)
    ap.add_argument("--mode", default="fast")
    ap.add_argument("--reps", type=int, default=1)
    ap.add_argument("--max-iters", type=int, default=None)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    p = P.config(a.config, Nd=a.nd)
    if a.nt:
        p = p.replace(Nt=a.nt)
    if a.max_iters:
        p = p.replace(max_iters=a.max_iters)
    t0 = time.time()
    b_host = slab_rhs(a.config, p, 1, p.Nt)
    rhs_s = time.time() - t0
    t0 = time.time()
    k = HeatKKT(p, mode=a.mode)
    torch.cuda.synchronize()
    setup_s = time.time() - t0
    b = torch.from_numpy(b_host).cuda()
    del b_host
    x = torch.empty_like(b)
    k.set_phase_timing(True)
    times = []
    for _ in range(a.reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        o = k.gmres_solve(b, x)
        e1.record()
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1) / 1e3)
    ms, cnt = k.phase_times()
    B = p.block
    rec = {"config": a.config, "Nd": p.Nd, "Nt": p.Nt, "nx": p.nx_int, "mode": a.mode,
           "inputs": "BASELINE seeded target (problems.kkt_rhs)", "rhs_gen_s": rhs_s, "setup_s": setup_s,
           "solve_s": times, "iterations": o.iterations, "converged": o.converged,
           "true_final_relres": o.true_final_relres,
           "unknowns_per_s": 3 * B / min(times),
           "phase_ms_total": dict(zip(["K", "P_inv", "krylov", "sweep"], ms)),
           "phase_counts": dict(zip(["K", "P_inv", "krylov", "sweep"], cnt)),
           "norms": {n: float(x[i * B:(i + 1) * B].norm()) for i, n in enumerate("uzw")},
           "mem_GB": torch.cuda.max_memory_allocated() / 1e9,
           "history": [float(h) for h in o.residual_history]}
    free, total = torch.cuda.mem_get_info()
    rec["device_mem_used_GB"] = (total - free) / 1e9
    print(json.dumps({k2: v for k2, v in rec.items() if k2 != "history"}), flush=True)
    if a.out:
        json.dump(rec, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
