"""Run the compiled REFERENCE (oracle/_ref) on a full BASELINE-config solve and
write a golden record under tests/golden/ (test infrastructure).

    python scripts/golden_full_solve.py --config 1 [--coarse scalar]

The record holds the iteration count, convergence flag, true relative
residual, the full residual history, per-block L2 norms, SHA-256 of the raw
little-endian bytes of u, z, w, and a strided sample (every STRIDE-th entry)
of the solution, so that a bitwise (strict-mode) GPU run can be checked by
hash and a fast-mode run by relative error on the sample.  Small configs also
store the whole solution.
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle.bindings import Ref  # noqa: E402
from paper_2305_04421_b200 import problems as P  # noqa: E402

STRIDE = 1009


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, required=True)
    ap.add_argument("--coarse", default="scalar")
    ap.add_argument("--precond", default="two-level")
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    p = P.config(a.config, coarse=a.coarse, precond=a.precond)
    tag = f"c{a.config}_{a.precond}_{a.coarse}"
    out = a.out or os.path.join(ROOT, "tests", "golden", f"solve_{tag}")
    b = P.kkt_rhs(a.config, p)
    t0 = time.time()
    ref = Ref(p)
    t_setup = time.time() - t0
    t0 = time.time()
    r = ref.gmres_solve(b)
    t_solve = time.time() - t0
    x = r["x"]
    B = p.block
    blocks = {"u": x[:B], "z": x[B:2 * B], "w": x[2 * B:]}
    rec = {
        "config": a.config, "precond": a.precond, "coarse": a.coarse,
        "problem": p.__dict__,
        "iterations": r["iterations"], "converged": r["converged"],
        "true_final_relres": r["true_final_relres"],
        "history": [float(h) for h in r["history"]],
        "norms": {k: float(np.linalg.norm(v)) for k, v in blocks.items()},
        "sha256": {k: hashlib.sha256(np.ascontiguousarray(v, dtype="<f8").tobytes()).hexdigest()
                   for k, v in blocks.items()},
        "b_sha256": hashlib.sha256(np.ascontiguousarray(b, dtype="<f8").tobytes()).hexdigest(),
        "stride": STRIDE,
        "setup_seconds": t_setup, "solve_seconds": t_solve,
        "host": os.uname().nodename, "threads": 1,
        "generator": "scripts/golden_full_solve.py (reference compiled by oracle/Makefile)",
    }
    with open(out + ".json", "w") as f:
        json.dump(rec, f, indent=1)
    np.savez_compressed(out + "_sample.npz", idx=np.arange(0, 3 * B, STRIDE, dtype=np.int64),
                        x=x[::STRIDE])
    if 3 * B <= 400_000:
        np.save(out + "_x.npy", x)
    print(json.dumps({k: rec[k] for k in ("iterations", "converged", "true_final_relres",
                                           "setup_seconds", "solve_seconds")}))


if __name__ == "__main__":
    main()
