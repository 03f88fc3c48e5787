"""The paper's studies on the GPU: the reference acceptance
suite's weak-scaling and omega sweeps (tests/acceptance_main.cpp:274-363),
run through the device run_single with the reference's sweep functions'
semantics (paper_2305_04421_b200.experiments), written as the reference's CSV.

    python scripts/paper_sweeps.py [--mode fast|strict] [--out profiles/sweeps_r01]

Base config: the reference defaults (config.hpp:36-50: Lx=1, Ly=2, T=1, nu=1,
two-level per-dof multiplicative, minus sign) with a 17x17 mesh (Nx=Ny=16),
GMRES tol 1e-6, at most 420 iterations, no restart — acceptance_main.cpp:276-280.
The iteration counts the reference itself produced for the same grids
(measured in the survey container) are printed beside ours.
"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2305_04421_b200 import experiments as E  # noqa: E402
from paper_2305_04421_b200 import problems as P  # noqa: E402

# reference iteration counts (acceptance_main.cpp run in the survey)
REF_WEAK = {("two-level", 1e-2): [20, 22, 22, 20], ("two-level", 1e-3): [17, 21, 21, 21],
            ("two-level", 1e-4): [15, 17, 21, 23], ("one-level", 1e-2): [22, 32, 48, 84],
            ("one-level", 1e-3): [17, 20, 28, 46], ("one-level", 1e-4): [15, 17, 21, 25]}
REF_OMEGA = {"two-level": [22, 21, 21, 16, 16], "one-level": [48, 28, 21, 15, 17]}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--mode", default="fast", choices=["fast", "strict"])
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "sweeps_r01"))
    a = ap.parse_args()
    base = P.Problem().replace(Nx=16, Ny=16, tol=1e-6, max_iters=420, restart=None)
    nts = [100, 200, 400, 800]
    omegas = [1e-2, 1e-3, 1e-4]
    t0 = time.perf_counter()
    weak = E.weak_scaling_sweep(base, 20, nts, omegas, ["two-level", "one-level"], mode=a.mode)
    t1 = time.perf_counter()
    om = E.omega_sweep(base, 400, 20, [1e-2, 1e-3, 1e-4, 1e-5, 1e-6], ["two-level", "one-level"],
                       mode=a.mode)
    t2 = time.perf_counter()
    with open(f"{a.out}_weak_{a.mode}.csv", "w") as f:
        f.write(E.to_csv(weak))
    with open(f"{a.out}_omega_{a.mode}.csv", "w") as f:
        f.write(E.to_csv(om))
    print(f"weak-scaling sweep: {len(weak.rows)} runs in {t1 - t0:.1f} s; "
          f"omega sweep: {len(om.rows)} runs in {t2 - t1:.1f} s ({a.mode})")
    ok = True
    for (pc, w), want in REF_WEAK.items():
        got = [r.iterations for r in weak.rows if r.config.precond == pc and r.config.omega == w]
        ok &= all(abs(g - x) <= 1 for g, x in zip(got, want))
        print(f"  weak {pc:9s} omega={w:g}: ours {got}  reference {want}")
    for pc, want in REF_OMEGA.items():  # want: omega = 1e-2 .. 1e-6 (rows are sorted ascending)
        got = [r.iterations for r in sorted(om.rows, key=lambda r: -r.config.omega) if r.config.precond == pc]
        ok &= all(abs(g - x) <= 1 for g, x in zip(got, want))
        print(f"  omega {pc:9s}: ours {got}  reference {want}")
    print("all iteration counts within +-1 of the reference's" if ok else "MISMATCH against the reference")
    return 0 if ok else 1


if __name__ == "__main__":
    sys.exit(main())
