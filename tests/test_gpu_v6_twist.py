"""GPU: the two-sided (twisted) block elimination of sweep v6 (sweep_v6.cu, factor_block.cu
build_twist_middle).  For odd ny the block rows 0..M-1 and ny-1..M+1 run as two half-length
chains that meet in the middle row M = (ny-1)/2; the bottom half is the mirror image of the top
(the same operators), the middle row has its own Schur complement T - 2 cy^2 D_{M-1}^{-1}.  It is
the same direct solve with a re-ordered elimination, so it is gated like every FAST operator:
1e-10 relative L2 per block against STRICT (bitwise the reference's banded LU), plus bitwise
run-to-run determinism, and against the one-sided elimination (KKT_V6_TWIST=0).
"""
import os
import subprocess
import sys

import numpy as np
import pytest

from paper_2305_04421_b200 import problems as P

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

# (Nx, Ny, Nt, Nd, precond, nu): ny = Ny - 1 odd in every case
CASES = [
    (300, 4, 8, 4, "two-level", 0.1),      # ny = 3: one row per half chain (M = 1)
    (520, 8, 12, 6, "two-level", 0.1),     # ny = 7, 512-blocks
    (1024, 6, 8, 4, "two-level", 1.0),     # ny = 5, the full 1024-wide padded row
    (200, 40, 8, 4, "one-level", 0.1),     # ny = 39 on 256-blocks (row grouping k > 1 by default)
    (400, 12, 40, 20, "two-level", 0.1),   # 20 chains: 3 real chain groups, the last half full
    (600, 202, 4, 2, "two-level", 1e-3),   # ny = 201: the block recursion converges inside the half chain
]


def _rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def _problem(Nx, Ny, Nt, Nd, pre, nu):
    return P.Problem(Lx=1.0, Ly=1.0, Nx=Nx, Ny=Ny, Nt=Nt, Nd=Nd, nu=nu, omega=1e-2, precond=pre,
                     coarse_variant="scalar", tol=1e-8, restart=20)


@pytest.mark.parametrize("case", CASES, ids=[f"{c[0]}x{c[1]}_nt{c[2]}_nd{c[3]}_{c[4]}" for c in CASES])
def test_twisted_pinv_against_strict(case):
    import torch
    from paper_2305_04421_b200.solver import HeatKKT
    p = _problem(*case)
    assert (p.Ny - 1) % 2 == 1
    v = torch.from_numpy(P.random_kkt(p, 1)).cuda()
    f = HeatKKT(p, mode="fast")
    s = HeatKKT(p, mode="strict")
    got = f.apply_P_inv(v).clone()
    again = f.apply_P_inv(v)
    assert torch.equal(got, again), "not deterministic"
    got = got.cpu().numpy()
    want = s.apply_P_inv(v).cpu().numpy()
    B = p.block
    for blk in range(3):
        err = _rel(got[blk * B:(blk + 1) * B], want[blk * B:(blk + 1) * B])
        assert err <= 1e-10, (blk, err)
    w = v[2 * B:3 * B].contiguous()
    e = _rel(f.apply_rasq(w).cpu().numpy(), s.apply_rasq(w).cpu().numpy())
    assert e <= 1e-10, e


@pytest.mark.parametrize("Nx,Ny", [(600, 8), (1024, 6), (200, 24)])
def test_twisted_window_and_band_solves(Nx, Ny):
    import torch
    from paper_2305_04421_b200.solver import HeatKKT
    p = _problem(Nx, Ny, 8, 2, "one-level", 0.1)
    f = HeatKKT(p, mode="fast")
    s = HeatKKT(p, mode="strict")
    g = torch.Generator(device="cuda").manual_seed(5)
    b = torch.randn(5 * p.n_sp, dtype=torch.float64, device="cuda", generator=g)
    for fn in ("forward_solve_window", "adjoint_solve_window"):
        x = getattr(f, fn)(b.clone()).cpu().numpy()
        y = getattr(s, fn)(b.clone()).cpu().numpy()
        assert _rel(x, y) <= 1e-10, fn
    for tr in (False, True):
        x = f.band_solve(b.clone(), transpose=tr).cpu().numpy()
        y = s.band_solve(b.clone(), transpose=tr).cpu().numpy()
        assert _rel(x, y) <= 1e-10, tr


@pytest.mark.parametrize("env", [{"KKT_V6_TWIST": "0"}, {"KKT_V6_K": "1"}, {"KKT_V6_K": "4"}, {"KKT_V6_K": "7"},
                                 {"KKT_V6_NOBAND": "1"}, {"KKT_V6_LL": "0"}, {"KKT_V6_K": "1", "KKT_V6_THOMAS": "0"},
                                 {"KKT_V6_K": "1", "KKT_V6_NOBAND": "1"}, {"KKT_V6_K": "1", "KKT_V6_NOHOLD": "1"},
                                 {"KKT_V6_K": "4", "KKT_V6_THOMAS": "0"}, {"KKT_V6_K": "7", "KKT_V6_THOMAS": "0"},
                                 {"KKT_V6_THOMAS": "0"}],
                         ids=["one_sided", "k1", "k4", "k7", "noband", "counter", "k1_lu_form", "k1_noband", "k1_nohold",
                              "k4_lu_form", "k7_lu_form", "lu_form"])
def test_twisted_variants_against_strict(env):
    """The twisted elimination combined with the chain's other re-associations (row grouping k,
    full rows instead of the numerical band), the one-sided elimination (KKT_V6_TWIST=0) and the
    counter handoff (which runs one-sided) on the same inputs: every variant within 1e-10 of
    STRICT and bitwise deterministic.  Subprocesses: the switches are read once per process."""
    code = (
        "import numpy as np, torch; from paper_2305_04421_b200 import problems as P; "
        "from paper_2305_04421_b200.solver import HeatKKT\n"
        "for (Nx, Ny, Nt, Nd, nu) in ((180, 38, 8, 4, 0.1), (300, 330, 4, 2, 1e-3), (500, 24, 32, 16, 0.1)):\n"
        "    p = P.Problem(Lx=1.0, Ly=1.0, Nx=Nx, Ny=Ny, Nt=Nt, Nd=Nd, nu=nu, omega=1e-2, "
        "precond='two-level', coarse_variant='scalar', tol=1e-8, restart=20)\n"
        "    v = torch.from_numpy(P.random_kkt(p, 1)).cuda()\n"
        "    f = HeatKKT(p, mode='fast'); a = f.apply_P_inv(v).clone(); a2 = f.apply_P_inv(v)\n"
        "    b = HeatKKT(p, mode='strict').apply_P_inv(v)\n"
        "    B = p.block\n"
        "    print('REL', max(float((a[k*B:(k+1)*B] - b[k*B:(k+1)*B]).norm() / b[k*B:(k+1)*B].norm()) for k in range(3)), "
        "'DET', bool(torch.equal(a, a2)))\n")
    r = subprocess.run([sys.executable, "-c", code], env=dict(os.environ, KKT_V6_TIM="1", **env), capture_output=True,
                       text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    rows = [x.split() for x in r.stdout.splitlines() if x.startswith("REL")]
    assert len(rows) == 3, r.stdout
    for row in rows:
        assert float(row[1]) <= 1e-10 and row[3] == "True", (env, rows)
    twisted = "v6 twisted elimination" in r.stderr
    assert twisted == (env.get("KKT_V6_TWIST") != "0" and env.get("KKT_V6_LL") != "0"), r.stderr[-1500:]
    # the twisted elimination takes the inverse-block form (no off-chain products), row by row or
    # grouped, unless KKT_V6_THOMAS=0 asks for the L/U factors
    inverse = any("v6 elimination form: inverse blocks" in x for x in r.stderr.splitlines())
    assert inverse == (twisted and env.get("KKT_V6_THOMAS") != "0"), r.stderr[-1500:]


def test_twisted_full_solve_against_one_sided(tmp_path):
    """A whole FAST GMRES solve with the twisted elimination against the same solve with the
    one-sided elimination: same iteration count, residual histories within 1e-8 relative over
    the first 20 iterations and 1e-10 absolute throughout,
    solutions within 1e-7 (both are tol-1e-8 iterates of the same problem)."""
    code = (
        "import sys, json, numpy as np, torch; from paper_2305_04421_b200 import problems as P; "
        "from paper_2305_04421_b200.solver import HeatKKT; "
        "p = P.Problem(Lx=1.0, Ly=1.0, Nx=300, Ny=32, Nt=32, Nd=4, nu=0.1, omega=1e-2, "
        "precond='two-level', coarse_variant='scalar', tol=1e-8, restart=30, max_iters=200); "
        "b = P.kkt_rhs(0, p); o = HeatKKT(p, mode='fast').gmres_solve(b); "
        "np.save(sys.argv[1], o.solution.cpu().numpy()); "
        "print('OUT', json.dumps({'its': o.iterations, 'conv': bool(o.converged), 'hist': list(map(float, o.residual_history))}))")
    import json
    outs = []
    for name, env in (("tw", {}), ("os", {"KKT_V6_TWIST": "0"})):
        path = str(tmp_path / f"{name}.npy")
        r = subprocess.run([sys.executable, "-c", code.replace("sys.argv[1]", repr(path))], env=dict(os.environ, **env),
                           capture_output=True, text=True, timeout=900, cwd=ROOT)
        assert r.returncode == 0, r.stderr[-2000:]
        rec = json.loads([x for x in r.stdout.splitlines() if x.startswith("OUT")][0][4:])
        outs.append((rec, np.load(path)))
    (a, xa), (b, xb) = outs
    assert a["conv"] and b["conv"]
    assert abs(a["its"] - b["its"]) <= 1, (a["its"], b["its"])
    n = min(len(a["hist"]), len(b["hist"]))
    ha, hb = np.asarray(a["hist"][:n]), np.asarray(b["hist"][:n])
    # relative residuals (the first is 1): 1e-8 relative over the first 20 iterations, 1e-10 absolute
    # throughout (measured: <= 4e-14 relative early, <= 2.6e-12 absolute at the 1e-8 end of the history)
    d = np.abs(ha - hb)
    assert np.all(d[:20] <= 1e-8 * hb[:20]), np.max(d[:20] / hb[:20])
    assert np.all(d <= 1e-10), d.max()
    assert _rel(xa, xb) <= 1e-7, _rel(xa, xb)


@pytest.mark.parametrize("env", [{}, {"KKT_E2E_TRAIL_OFF": "1"}, {"KKT_E2E_CHUNK_KB": "100"}, {"KKT_E2E_CHUNK_KB": "0"}],
                         ids=["trailed", "whole_copy", "ragged_chunks", "whole_blocks"])
def test_host_pinv_trailing_download(env):
    """kkt_apply_P_inv_host on a v6 grid with pinned host buffers: the w block's planes go back to
    the host behind each adjoint step of the sweep (rasq_apply's step hook) instead of in one
    copy after it.  The result is bitwise the device-resident application either way, for the
    fused two-level form and for one-level RASQ; pageable buffers take the whole-copy path.  The
    u and z blocks travel in chunks (up, divided, down): one chunk, several ragged ones, or whole."""
    code = (
        "import numpy as np, torch; from paper_2305_04421_b200 import problems as P; "
        "from paper_2305_04421_b200.solver import HeatKKT\n"
        "for pre in ('two-level', 'one-level'):\n"
        "    p = P.Problem(Lx=1.0, Ly=1.0, Nx=300, Ny=12, Nt=24, Nd=6, nu=0.1, omega=1e-2, "
        "precond=pre, coarse_variant='scalar', tol=1e-8, restart=20)\n"
        "    k = HeatKKT(p, mode='fast'); r = P.random_kkt(p, 3)\n"
        "    want = k.apply_P_inv(torch.from_numpy(r).cuda()).cpu().numpy()\n"
        "    rh = torch.from_numpy(r).pin_memory(); oh = torch.zeros(r.size, dtype=torch.float64).pin_memory()\n"
        "    k.apply_P_inv_host(rh.numpy(), oh.numpy())\n"
        "    print('PINNED', bool(np.array_equal(oh.numpy(), want)))\n"
        "    got = k.apply_P_inv_host(r.copy())\n"
        "    print('PAGEABLE', bool(np.array_equal(got, want)))\n")
    r = subprocess.run([sys.executable, "-c", code], env=dict(os.environ, KKT_E2E_TIM="1", **env), capture_output=True,
                       text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    assert r.stdout.count("PINNED True") == 2 and r.stdout.count("PAGEABLE True") == 2, r.stdout
    lines = [x for x in r.stderr.splitlines() if x.startswith("P_inv_host ms")]
    assert len(lines) == 4, r.stderr[-1500:]
    trailed = [("trailed" in x) for x in lines]
    assert trailed == ([False] * 4 if "KKT_E2E_TRAIL_OFF" in env else [True, False, True, False]), lines
    if env.get("KKT_E2E_CHUNK_KB") == "100":  # 299 x 11 x 24 doubles per block in 12,800-double chunks
        assert all("(7 u/z chunks" in x for x in lines), lines
