"""Per-dof coarse banded LU on the device vs a numpy restatement of BandedLU
(linalg.cpp:69-125) on the reference's S0: first differing column."""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle.bindings import Ref  # noqa: E402
from paper_2305_04421_b200 import problems as P  # noqa: E402
from paper_2305_04421_b200.solver import lib  # noqa: E402
from paper_2305_04421_b200.solver import HeatKKT  # noqa: E402

nx = int(sys.argv[1]) if len(sys.argv) > 1 else 21
nt = int(sys.argv[2]) if len(sys.argv) > 2 else 16
nd = int(sys.argv[3]) if len(sys.argv) > 3 else 4
os.environ["KKT_KEEP_S0"] = "1"
p = P.Problem(Lx=1.0, Ly=1.0, Nx=nx, Ny=nx, Nt=nt, Nd=nd, omega=1e-2, coarse_variant="per-dof")
k = HeatKKT(p, mode="strict")
S0 = k.coarse_matrix()  # the device assembly (bitwise to the reference's where comparable)
n = S0.shape[0]
kl_, ku_ = C.c_int32(), C.c_int32()
assert lib().kkt_debug_coarse_factor(k._h, C.byref(kl_), C.byref(ku_), None, None) == 0
kl, kuf = kl_.value, ku_.value
ld = kl + kuf + 1
ab = np.zeros(n * ld)
piv = np.zeros(n, dtype=np.int32)
assert lib().kkt_debug_coarse_factor(k._h, None, None, ab.ctypes.data_as(C.c_void_p),
                                     piv.ctypes.data_as(C.c_void_p)) == 0
G = ab.reshape(n, ld)          # G[j, i-j+kuf] = entry(i, j)
nz = np.nonzero(S0)
print("n", n, "kl", kl, "kuf", kuf, "pattern kl", (nz[0] - nz[1]).max(), "ku", (nz[1] - nz[0]).max(), flush=True)
A = S0.copy()
rp = np.zeros(n, dtype=np.int64)
for j in range(n):
    imax, jmax = min(n - 1, j + kl), min(n - 1, j + kuf)
    col = np.abs(A[j:imax + 1, j])
    pj = j + int(np.argmax(col))
    rp[j] = pj
    if pj != j:
        A[[j, pj], j:jmax + 1] = A[[pj, j], j:jmax + 1]
    A[j + 1:imax + 1, j] /= A[j, j]
    u = A[j, j + 1:jmax + 1]
    m = u != 0
    cs = np.arange(j + 1, jmax + 1)[m]
    A[j + 1:imax + 1][:, cs] -= np.outer(A[j + 1:imax + 1, j], u[m])
    # compare column j of the device factor (rows j-kuf..j+kl)
    lo, hi = max(0, j - kuf), min(n - 1, j + kl)
    dev = G[j, lo - j + kuf:hi - j + kuf + 1]
    if rp[j] != piv[j] or not np.array_equal(dev, A[lo:hi + 1, j]):
        bad = np.nonzero(dev != A[lo:hi + 1, j])[0]
        print("first diff at column", j, "piv", rp[j], piv[j], "rows", (bad[:10] + lo).tolist(),
              dev[bad[:3]], A[lo + bad[:3], j])
        break
else:
    print("factor matches")
ref = Ref(p)
r = P.random_vec(p.block, 31)
c = ref.coarse_restrict(r)
xr = ref.coarse_solve(c)
xd = k.coarse_solve(c).cpu().numpy()
print("resid ref", np.linalg.norm(S0 @ xr - c) / np.linalg.norm(c), "dev", np.linalg.norm(S0 @ xd - c) / np.linalg.norm(c),
      "equal", np.array_equal(xr, xd))
