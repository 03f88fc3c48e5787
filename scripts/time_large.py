"""Time setup, apply_K and apply_P_inv at the large BASELINE grids (FAST mode).

    python scripts/time_large.py --config 2 [--nt 1024] [--nd 64] [--reps 10]

Inputs are device N(0,1) vectors (timing only; parity lives in tests/).
Prints one JSON line per config.
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    from paper_2305_04421_b200 import problems as P
    from paper_2305_04421_b200.solver import HeatKKT

    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--nt", type=int, default=None)
    ap.add_argument("--nd", type=int, default=None)
    ap.add_argument("--T", type=float, default=None, help="final time (config 4's per-GPU slab: --nt 128 --T 0.125)")
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--mode", default="fast")
    ap.add_argument("--e2e", action="store_true", help="also time apply_P_inv_host from pinned host buffers")
    a = ap.parse_args()
    p = P.config(a.config, Nd=a.nd)
    if a.nt:
        p = p.replace(Nt=a.nt)
    if a.T:
        p = p.replace(T=a.T)
    t0 = time.time()
    k = HeatKKT(p, mode=a.mode)
    torch.cuda.synchronize()
    setup_s = time.time() - t0
    g = torch.Generator(device="cuda").manual_seed(0)
    v = torch.randn(3 * p.block, dtype=torch.float64, device="cuda", generator=g)
    out = torch.empty_like(v)
    st = torch.cuda.current_stream()

    def tm(fn, reps):
        fn()
        torch.cuda.synchronize()
        ts = []
        for _ in range(reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            fn()
            e1.record(st)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        ts.sort()
        return ts[len(ts) // 2]

    k_ms = tm(lambda: k.apply_K(v, out), max(3, a.reps))
    p_ms = tm(lambda: k.apply_P_inv(v, out), a.reps)
    unk = 3 * p.block
    e2e_ms = None
    if a.e2e:
        hin = torch.empty(3 * p.block, dtype=torch.float64).pin_memory()
        hout = torch.empty(3 * p.block, dtype=torch.float64).pin_memory()
        hin.copy_(v)
        ts = []
        for _ in range(a.reps + 1):
            torch.cuda.synchronize()
            t1 = time.perf_counter()
            k.apply_P_inv_host(hin.numpy(), hout.numpy())
            ts.append((time.perf_counter() - t1) * 1e3)
        ts = sorted(ts[1:])
        e2e_ms = ts[len(ts) // 2]
    print(json.dumps({"config": a.config, "Nt": p.Nt, "Nd": p.Nd, "nx": p.nx_int, "setup_s": setup_s,
                      "apply_K_ms": k_ms, "apply_P_inv_ms": p_ms, "e2e_ms": e2e_ms,
                      "P_inv_unknowns_per_s": unk / (p_ms * 1e-3),
                      "finite": bool(torch.isfinite(out).all().item())}), flush=True)


if __name__ == "__main__":
    main()
