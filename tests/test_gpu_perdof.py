"""GPU parity of the per-dof coarse variant (the reference's default,
config.hpp:47; schur.cpp:266-413) against the compiled reference.

STRICT mode is bitwise identical: S0 assembly, the banded LU with partial
pivoting (linalg.cpp:69-125), restriction, solve, prolongation, the two-level
forms and full GMRES solves.  FAST mode keeps the same coarse path and uses the
fast sweep: rounding-level tolerances written in each test.
"""
import hashlib
import json
import os

import numpy as np
import pytest

from paper_2305_04421_b200 import problems as P

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")

PERDOF = [
    P.Problem(Lx=1.0, Ly=2.0, Nx=8, Ny=6, Nt=12, Nd=3, omega=1e-2, coarse_variant="per-dof",
              tol=1e-10, restart=10, max_iters=200),
    P.Problem(Lx=1.0, Ly=1.0, Nx=9, Ny=9, Nt=16, Nd=4, omega=1e-3, coarse_variant="per-dof",
              tol=1e-7, restart=None, max_iters=200),  # stagnates near 5e-8 (reference too)
    P.Problem(Lx=1.0, Ly=1.0, Nx=2, Ny=7, Nt=6, Nd=6, omega=1e-2, coarse_variant="per-dof",
              tol=1e-10, restart=5, max_iters=100),   # m = 1: constant columns only
    P.Problem(Lx=1.0, Ly=2.0, Nx=13, Ny=11, Nt=24, Nd=8, omega=1e-2, coarse_variant="per-dof",
              tol=1e-10, restart=20, max_iters=200),  # dim 2*8*120 = 1920
]
IDS = ["8x6_nt12_nd3", "9x9_nt16_nd4", "nx1_m1", "13x11_nt24_nd8"]


def rel(a, b):
    nb = np.linalg.norm(b)
    return np.linalg.norm(np.asarray(a) - b) / (nb if nb > 0 else 1.0)


def host(t):
    return t.detach().cpu().numpy()


@pytest.fixture(scope="module", params=list(zip(PERDOF, IDS)), ids=IDS)
def case(request):
    from oracle.bindings import Ref
    from paper_2305_04421_b200.solver import HeatKKT
    p, _ = request.param
    return p, Ref(p), HeatKKT(p, mode="strict"), HeatKKT(p, mode="fast")


def test_coarse_matrix_and_ops_bitwise(case):
    import torch
    p, ref, ks, kf = case
    assert ks.coarse_dim() == ref.coarse_dim() == kf.coarse_dim()
    S0 = ref.coarse_matrix()
    assert np.array_equal(ks.coarse_matrix(), S0)
    r = P.random_vec(p.block, 31)
    c_ref = ref.coarse_restrict(r)
    assert np.array_equal(host(ks.coarse_restrict(r)), c_ref)
    s_ref = ref.coarse_solve(c_ref)
    assert np.array_equal(host(ks.coarse_solve(c_ref)), s_ref)
    assert np.array_equal(host(kf.coarse_solve(c_ref)), s_ref)
    base = P.random_vec(p.block, 32)
    want = ref.coarse_prolong_add(s_ref, base)
    got = ks.coarse_prolong_add(torch.tensor(s_ref, device="cuda"), torch.tensor(base, device="cuda"))
    assert np.array_equal(host(got), want)


@pytest.mark.parametrize("form", ["literal", "multiplicative", "additive"])
def test_two_level_forms(case, form):
    p, ref, ks, kf = case
    r = P.random_vec(p.block, 33)
    want = ref.apply_two_level(r, P.FORM[form])
    assert np.array_equal(host(ks.apply_two_level(r, form)), want), form
    assert rel(host(kf.apply_two_level(r, form)), want) <= 1e-11, form


def test_pinv(case):
    p, ref, ks, kf = case
    r = P.random_vec(3 * p.block, 34)
    want = ref.apply_P_inv(r)
    assert np.array_equal(host(ks.apply_P_inv(r)), want)
    assert rel(host(kf.apply_P_inv(r)), want) <= 1e-11


def test_gmres(case):
    p, ref, ks, kf = case
    b = P.random_vec(3 * p.block, 35)
    want = ref.gmres_solve(b)
    got = ks.gmres_solve(b)
    assert got.iterations == want["iterations"]
    assert np.array_equal(got.residual_history, want["history"])
    assert np.array_equal(host(got.solution), want["x"])
    fast = kf.gmres_solve(b)
    assert abs(fast.iterations - want["iterations"]) <= 1
    assert rel(host(fast.solution), want["x"]) <= max(1e-9, 10 * want["true_final_relres"])


def test_dense_limit_is_a_config_error():
    """coarse_matrix_dense refuses dim > 4096 (schur.cpp:246, check_dense_scale)."""
    from paper_2305_04421_b200.solver import ConfigError, HeatKKT
    p = P.config(0, coarse="per-dof")
    k = HeatKKT(p, mode="fast")
    assert k.coarse_dim() == 2 * p.Nd * p.n_sp
    with pytest.raises(ConfigError):
        k.coarse_matrix()


def _sha(x):
    return hashlib.sha256(np.ascontiguousarray(x, dtype="<f8").tobytes()).hexdigest()


def test_config0_per_dof_against_golden():
    """BASELINE config 0 with the reference's default coarse space (dim 7688,
    banded S0) vs the golden record from the compiled reference."""
    from paper_2305_04421_b200.solver import HeatKKT
    gold = json.load(open(os.path.join(GOLD, "solve_c0_two-level_per-dof.json")))
    p = P.config(0, coarse="per-dof", precond="two-level")
    b = P.kkt_rhs(0, p)
    assert _sha(b) == gold["b_sha256"]
    s = HeatKKT(p, mode="strict").gmres_solve(b)
    x = host(s.solution)
    B = p.block
    assert s.iterations == gold["iterations"]
    assert list(s.residual_history) == gold["history"]
    for i, k in enumerate("uzw"):
        assert _sha(x[i * B:(i + 1) * B]) == gold["sha256"][k], k
    f = HeatKKT(p, mode="fast").gmres_solve(b)
    xf = host(f.solution)
    assert abs(f.iterations - gold["iterations"]) <= 1
    for i in range(3):
        assert rel(xf[i * B:(i + 1) * B], x[i * B:(i + 1) * B]) <= 1e-10


# ---------------------------------------------------------------------------
# the per-dof coarse space beyond desk scale (coarse_kron.cu)
# ---------------------------------------------------------------------------
def test_kron_solve_against_the_reference_at_desk_scale():
    """The Kronecker solve of S0 (FAST, coarse_kron.cu: S0 = (T2 x Ahat^2 + T1 x Ahat + T0 x I)/ms
    in Ahat's eigenbasis, one banded LDL^T per eigenmode) forced at desk scale
    (KKT_PERDOF_KRON=1, read once per process) against the compiled reference's banded-LU
    solve of the same S0: the coarse solve, the three two-level forms, P^-1, a full GMRES
    solve; and BASELINE config 0's per-dof solve against the reference's golden record."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = r'''
import json, os, numpy as np, torch
from paper_2305_04421_b200 import problems as P
from paper_2305_04421_b200.solver import HeatKKT
from oracle.bindings import Ref
def rel(a, b): return float(np.linalg.norm(np.asarray(a) - b) / np.linalg.norm(b))
host = lambda t: t.detach().cpu().numpy()
out = {}
cases = [P.Problem(Lx=1.0, Ly=2.0, Nx=8, Ny=6, Nt=12, Nd=3, omega=1e-2, coarse_variant="per-dof", tol=1e-10, restart=10, max_iters=200),
         P.Problem(Lx=1.0, Ly=1.0, Nx=2, Ny=7, Nt=6, Nd=6, omega=1e-2, coarse_variant="per-dof", tol=1e-10, restart=5, max_iters=100),
         P.Problem(Lx=1.0, Ly=2.0, Nx=13, Ny=11, Nt=24, Nd=8, omega=1e-2, coarse_variant="per-dof", tol=1e-10, restart=20, max_iters=200)]
for i, p in enumerate(cases):
    ref, kf = Ref(p), HeatKKT(p, mode="fast")
    r = P.random_vec(p.block, 31)
    c = ref.coarse_restrict(r)
    o = {"solve": rel(host(kf.coarse_solve(c)), ref.coarse_solve(c))}
    for form in ("literal", "multiplicative", "additive"):
        o[form] = rel(host(kf.apply_two_level(r, form)), ref.apply_two_level(r, P.FORM[form]))
    v = P.random_vec(3 * p.block, 34)
    o["pinv"] = rel(host(kf.apply_P_inv(v)), ref.apply_P_inv(v))
    b = P.random_vec(3 * p.block, 35)
    w, g = ref.gmres_solve(b), kf.gmres_solve(b)
    o["its"] = [g.iterations, w["iterations"]]
    o["sol"] = rel(host(g.solution), w["x"])
    o["relres"] = w["true_final_relres"]
    out[str(i)] = o
p = P.config(0, coarse="per-dof", precond="two-level")
gold = json.load(open(os.path.join("tests", "golden", "solve_c0_two-level_per-dof.json")))
xg = np.load(os.path.join("tests", "golden", "solve_c0_two-level_per-dof_x.npy"))
f = HeatKKT(p, mode="fast").gmres_solve(P.kkt_rhs(0, p))
B = p.block
out["c0"] = {"its": [f.iterations, gold["iterations"]],
             "blocks": [rel(host(f.solution)[k*B:(k+1)*B], xg[k*B:(k+1)*B]) for k in range(3)]}
print("OUT", json.dumps(out))
'''
    r = subprocess.run([sys.executable, "-c", code], env=dict(os.environ, KKT_PERDOF_KRON="1"), capture_output=True,
                       text=True, timeout=900, cwd=root)
    assert r.returncode == 0, r.stderr[-3000:]
    out = json.loads([x for x in r.stdout.splitlines() if x.startswith("OUT")][0][4:])
    for i in ("0", "1", "2"):
        o = out[i]
        assert o["solve"] <= 1e-10, (i, o)
        assert max(o["literal"], o["multiplicative"], o["additive"], o["pinv"]) <= 1e-10, (i, o)
        assert abs(o["its"][0] - o["its"][1]) <= 1, (i, o)
        assert o["sol"] <= max(1e-9, 10 * o["relres"]), (i, o)
    assert abs(out["c0"]["its"][0] - out["c0"]["its"][1]) <= 1, out["c0"]
    assert max(out["c0"]["blocks"]) <= 1e-10, out["c0"]


def test_per_dof_two_level_at_config1():
    """BASELINE config 1 with the reference's DEFAULT coarse variant (per-dof: dimension
    2 * 16 * 16129 = 516,128), which the reference cannot factor (~600 GB of banded LU,
    SURVEY §8a-21) and round 1's dense device build could not hold.  No reference output
    exists at this size, so the coarse solve is checked against its definition --
    S0 = Z^T Shat Z through the device's own restrict / Shat / prolong, which the desk-scale
    tests pin bitwise to the reference -- and the full FAST solve must converge in fewer
    iterations than the scalar coarse space's 44."""
    import torch
    from paper_2305_04421_b200.solver import HeatKKT
    p = P.config(1, coarse="per-dof")
    k = HeatKKT(p, mode="fast")
    d = k.coarse_dim()
    assert d == 2 * p.Nd * p.n_sp == 516128
    g = torch.Generator(device="cuda").manual_seed(7)
    c = torch.randn(d, dtype=torch.float64, device="cuda", generator=g)
    x = k.coarse_solve(c)
    z = torch.zeros(p.block, dtype=torch.float64, device="cuda")
    k.coarse_prolong_add(x, z)
    back = k.coarse_restrict(k.apply_shat(z))          # Z^T Shat Z x
    assert float((back - c).norm() / c.norm()) <= 1e-9
    b = P.kkt_rhs(1, p)
    out = k.gmres_solve(b)
    assert out.converged and out.true_final_relres <= 1.5 * p.tol
    assert out.iterations < 44, out.iterations
    # the solution solves the KKT system (independent residual evaluation), and the sweep is the
    # LU block substitution, not the opt-in spectral one (the Kronecker solve shares its sine matrices)
    assert k.kkt_residual(out.solution, b) <= 1.5 * p.tol
    k.set_phase_timing(True)
    k.apply_P_inv(torch.from_numpy(b).cuda())
    ms, cnt = k.phase_times()
    assert cnt[3] == 1 and ms[3] > 3.0, (ms, cnt)   # one v4 sweep (~4.2 ms); the spectral one takes ~1 ms
