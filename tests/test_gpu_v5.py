"""GPU: the large-grid FAST sweeps against STRICT mode, which is bitwise the
reference's banded LU (test_gpu_parity.py), on grids small enough in time for
STRICT to finish in seconds.  The in-process tests run the default sweep for
128 < nx <= 511, which is sweep v6 (sweep_v6.cu) since it replaced v5 there;
sweep v5 (sweep_v5.cu) itself is checked in subprocesses with
KKT_SWEEP_V6_OFF=1 (the switch is read once per process).

Covers both cluster shapes (kN = 256: 8-CTA clusters; kN = 512: 16-CTA
clusters), chain counts that do not fill a set of 8, the window solves
(1 chain), multi-RHS band solves, one-level RASQ and the fused two-level
residual, rectangular grids (nx != ny).  Tolerance: 1e-10 relative L2 per
block (north_star's solution tolerance), as for the other FAST operators.
"""
import numpy as np
import pytest

from paper_2305_04421_b200 import problems as P

pytestmark = pytest.mark.gpu

CASES = [
    # (Nx, Ny, Nt, Nd, precond)
    (160, 160, 8, 4, "two-level"),    # nx = 159 -> kN 256, 4 chains
    (200, 150, 9, 3, "two-level"),    # rectangular, 3 chains
    (300, 300, 8, 2, "one-level"),    # nx = 299 -> kN 512 (16-CTA clusters)
    (140, 140, 80, 10, "two-level"),  # 10 chains: two chain sets, 17 steps each
    (257, 3, 8, 2, "two-level"),      # nx = 256 -> kN 512 at its smallest; ny = 2
    (256, 40, 8, 4, "two-level"),     # nx = 255: kN 256 full width
    (160, 400, 8, 2, "two-level", 1e-3),  # ny = 399, cy = 20: rows past jstar on resident operators
]


def _problem(Nx, Ny, Nt, Nd, pre, nu=0.1):
    return P.Problem(Lx=1.0, Ly=1.0, Nx=Nx, Ny=Ny, Nt=Nt, Nd=Nd, nu=nu, omega=1e-2, precond=pre,
                     coarse_variant="scalar", tol=1e-8, restart=20)


def _rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


@pytest.mark.parametrize("case", CASES, ids=[f"{c[0]}x{c[1]}_nt{c[2]}_nd{c[3]}_{c[4]}_nu{c[5] if len(c) > 5 else 0.1}"
                                             for c in CASES])
def test_v5_pinv_against_strict(case):
    import torch
    from paper_2305_04421_b200.solver import HeatKKT
    p = _problem(*case)
    v = torch.from_numpy(P.random_kkt(p, 1)).cuda()
    f = HeatKKT(p, mode="fast")
    s = HeatKKT(p, mode="strict")
    got = f.apply_P_inv(v).cpu().numpy()
    want = s.apply_P_inv(v).cpu().numpy()
    B = p.block
    for blk in range(3):
        err = _rel(got[blk * B:(blk + 1) * B], want[blk * B:(blk + 1) * B])
        assert err <= 1e-10, (blk, err)
    # RASQ alone (one-level part) too
    w = v[2 * B:3 * B].contiguous()
    e = _rel(f.apply_rasq(w).cpu().numpy(), s.apply_rasq(w).cpu().numpy())
    assert e <= 1e-10, e


@pytest.mark.parametrize("Nx,Ny", [(160, 160), (300, 220)])
def test_v5_window_and_band_solves(Nx, Ny):
    import torch
    from paper_2305_04421_b200.solver import HeatKKT
    p = _problem(Nx, Ny, 8, 2, "one-level")
    f = HeatKKT(p, mode="fast")
    s = HeatKKT(p, mode="strict")
    g = torch.Generator(device="cuda").manual_seed(3)
    b = torch.randn(5 * p.n_sp, dtype=torch.float64, device="cuda", generator=g)
    for fn in ("forward_solve_window", "adjoint_solve_window"):
        x = getattr(f, fn)(b.clone()).cpu().numpy()
        y = getattr(s, fn)(b.clone()).cpu().numpy()
        assert _rel(x, y) <= 1e-10, fn
    for tr in (False, True):
        x = f.band_solve(b.clone(), transpose=tr).cpu().numpy()
        y = s.band_solve(b.clone(), transpose=tr).cpu().numpy()
        assert _rel(x, y) <= 1e-10, tr


def test_v5_deterministic():
    """Fixed reduction order: two applications are bitwise equal."""
    import torch
    from paper_2305_04421_b200.solver import HeatKKT
    p = _problem(300, 300, 16, 8, "two-level")
    v = torch.from_numpy(P.random_kkt(p, 2)).cuda()
    f = HeatKKT(p, mode="fast")
    a = f.apply_P_inv(v).clone()
    b = f.apply_P_inv(v)
    assert torch.equal(a, b)


def test_v5_resident_rows_used():
    """The tall case converges inside the grid, so part of every sweep runs on
    the resident operators (jstar < ny); KKT_V5_TIM prints it.  Checked in a
    subprocess because the switch is read once per process."""
    import os
    import subprocess
    import sys
    code = ("import torch; from paper_2305_04421_b200 import problems as P; "
            "from paper_2305_04421_b200.solver import HeatKKT; "
            "p = P.Problem(Lx=1.0, Ly=1.0, Nx=160, Ny=400, Nt=8, Nd=2, nu=1e-3, omega=1e-2, "
            "precond='one-level', coarse_variant='scalar', tol=1e-8, restart=20); "
            "HeatKKT(p, mode='fast'); torch.cuda.synchronize()")
    env = dict(os.environ, KKT_V5_TIM="1", KKT_SWEEP_V6_OFF="1")
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600,
                       cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    assert r.returncode == 0, r.stderr[-2000:]
    line = [x for x in r.stderr.splitlines() if x.startswith("v5 jstar")]
    assert line, r.stderr[-2000:]
    js, ny = int(line[0].split()[2]), int(line[0].split()[5])
    assert 0 < js < ny - 1, line[0]


@pytest.mark.parametrize("case", [CASES[0], CASES[3], CASES[6]], ids=["kN256_4ch", "kN256_10ch", "kN256_resident"])
def test_v5_fallback_against_strict(case):
    """Sweep v5 (KKT_SWEEP_V6_OFF=1), kN = 256 cluster chains: P^-1 against STRICT."""
    import os
    import subprocess
    import sys
    Nx, Ny, Nt, Nd, pre = case[:5]
    nu = case[5] if len(case) > 5 else 0.1
    code = (
        "import numpy as np, torch; from paper_2305_04421_b200 import problems as P; "
        "from paper_2305_04421_b200.solver import HeatKKT; "
        f"p = P.Problem(Lx=1.0, Ly=1.0, Nx={Nx}, Ny={Ny}, Nt={Nt}, Nd={Nd}, nu={nu}, omega=1e-2, "
        f"precond='{pre}', coarse_variant='scalar', tol=1e-8, restart=20); "
        "v = torch.from_numpy(P.random_kkt(p, 1)).cuda(); "
        "a = HeatKKT(p, mode='fast').apply_P_inv(v).cpu().numpy(); "
        "b = HeatKKT(p, mode='strict').apply_P_inv(v).cpu().numpy(); "
        "B = p.block; print('REL', max(np.linalg.norm(a[k*B:(k+1)*B] - b[k*B:(k+1)*B]) / np.linalg.norm(b[k*B:(k+1)*B]) for k in range(3)))")
    env = dict(os.environ, KKT_SWEEP_V6_OFF="1")
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600,
                       cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    assert r.returncode == 0, r.stderr[-2000:]
    rel = float([x for x in r.stdout.splitlines() if x.startswith("REL")][0].split()[1])
    assert rel <= 1e-10, rel


@pytest.mark.parametrize("env,label", [({"KKT_SWEEP_V3": "1"}, "v3 group chains (sweep_group.cu)"),
                                       ({"KKT_SWEEP_V3": "1", "KKT_SWEEP_V2": "1"}, "v2 per-row chains (sweep_tma.cu)")],
                         ids=["v3", "v2"])
def test_small_grid_fallback_sweeps_against_strict(env, label):
    """The older small-grid sweeps stay selectable (KKT_SWEEP_V3 / KKT_SWEEP_V2: the
    FAST-parity bisection of scripts/bisect_fast_c1.py runs them): P^-1, RASQ and a
    full solve against STRICT on a config-0-sized problem."""
    import os
    import subprocess
    import sys
    code = (
        "import numpy as np, torch; from paper_2305_04421_b200 import problems as P; "
        "from paper_2305_04421_b200.solver import HeatKKT; "
        "p = P.config(0); v = torch.from_numpy(P.random_kkt(p, 1)).cuda(); "
        "f = HeatKKT(p, mode='fast'); s = HeatKKT(p, mode='strict'); B = p.block; "
        "a = f.apply_P_inv(v).cpu().numpy(); b = s.apply_P_inv(v).cpu().numpy(); "
        "print('REL', max(np.linalg.norm(a[k*B:(k+1)*B] - b[k*B:(k+1)*B]) / np.linalg.norm(b[k*B:(k+1)*B]) for k in range(3))); "
        "a = f.apply_rasq(v[:B]).cpu().numpy(); b = s.apply_rasq(v[:B]).cpu().numpy(); "
        "print('RASQ', np.linalg.norm(a - b) / np.linalg.norm(b)); "
        "rhs = P.kkt_rhs(0, p); of = f.gmres_solve(rhs); os_ = s.gmres_solve(rhs); "
        "print('ITS', of.iterations, os_.iterations); "
        "print('SOL', float((of.solution - os_.solution).norm() / os_.solution.norm()))")
    r = subprocess.run([sys.executable, "-c", code], env=dict(os.environ, **env), capture_output=True, text=True,
                       timeout=600, cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    assert r.returncode == 0, r.stderr[-2000:]
    out = {x.split()[0]: x.split()[1:] for x in r.stdout.splitlines() if x and x.split()[0] in ("REL", "RASQ", "ITS", "SOL")}
    assert float(out["REL"][0]) <= 1e-11, (label, out)
    assert float(out["RASQ"][0]) <= 1e-11, (label, out)
    assert abs(int(out["ITS"][0]) - int(out["ITS"][1])) <= 1, (label, out)
    assert float(out["SOL"][0]) <= 1e-10, (label, out)
