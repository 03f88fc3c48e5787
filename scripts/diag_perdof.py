"""Config-0 per-dof coarse pieces, device STRICT vs the compiled reference."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle.bindings import Ref  # noqa: E402
from paper_2305_04421_b200 import problems as P  # noqa: E402
from paper_2305_04421_b200.solver import HeatKKT  # noqa: E402


def main():
    p = P.config(0, coarse="per-dof", precond="two-level")
    t = time.time()
    k = HeatKKT(p, mode="strict")
    print("device setup", time.time() - t, flush=True)
    t = time.time()
    ref = Ref(p)
    print("ref setup", time.time() - t, flush=True)
    print("dim", k.coarse_dim(), ref.coarse_dim())
    r = P.random_vec(p.block, 31)
    c_ref = ref.coarse_restrict(r)
    c = k.coarse_restrict(r).cpu().numpy()
    print("restrict equal", np.array_equal(c, c_ref), np.abs(c - c_ref).max())
    s_ref = ref.coarse_solve(c_ref)
    s = k.coarse_solve(c_ref).cpu().numpy()
    d = np.abs(s - s_ref)
    print("solve equal", np.array_equal(s, s_ref), d.max() / np.abs(s_ref).max(),
          "first diff", int(np.argmax(d > 0)) if d.max() > 0 else -1)
    for form in ("multiplicative",):
        a = ref.apply_two_level(r, P.FORM[form])
        b = k.apply_two_level(r, form).cpu().numpy()
        print(form, np.array_equal(a, b), np.linalg.norm(a - b) / np.linalg.norm(a))


if __name__ == "__main__":
    main()
