"""GPU: the reference's error taxonomy through the C-ABI, triggered on the device.

Each case restates one of the reference's own error tests and checks that the
device path raises the same exception class with the same payload as the CPU
oracle (the compiled reference when built, else the C restatement):

  - SingularMatrixError{pivot_index}: the singular literal shift under
    jhat_sign = plus (tests/test_heat_operators.cpp:220-232, config.hpp:61-65,
    linalg.cpp:98-103).
  - GmresDivergenceError{iteration}: non-finite Krylov vectors
    (tests/test_gmres.cpp:141-153, gmres.cpp:84-89).
  - ConfigError: gmres restart < 1 (config.cpp:21) and the other validate() rules.
  - the plus sign on a large grid without diagonal dominance: refused, not
    silently factored without pivoting.
"""
import numpy as np
import pytest

from paper_2305_04421_b200 import problems as P

pytestmark = pytest.mark.gpu


def _oracle():
    from oracle import bindings
    return bindings.Ref if bindings.available("ref") else bindings.Orc


def _kkt(p, mode):
    from paper_2305_04421_b200.solver import HeatKKT
    return HeatKKT(p, mode=mode)


@pytest.mark.parametrize("mode", ["strict", "fast"])
def test_singular_literal_shift_reports_the_pivot(mode):
    from oracle.bindings import OracleError
    from paper_2305_04421_b200.solver import SingularMatrixError
    # single-unknown mesh: A = [2], dt = 0.1, omega = 0.0025 -> Ahat = 2 - 0.1/0.05 = 0
    p = P.Problem(Nt=10, Nd=1, Nx=2, Ny=2, omega=0.0025, jhat_sign="plus")
    with pytest.raises(OracleError) as want:
        _oracle()(p)
    assert want.value.status == 3
    with pytest.raises(SingularMatrixError) as got:
        _kkt(p, mode)
    assert got.value.pivot_index == want.value.index == 0
    assert "pivot" in str(got.value)


@pytest.mark.parametrize("mode", ["strict", "fast"])
def test_singular_pivot_index_past_the_first_row(mode):
    """A 3x1 grid with Ahat = tridiag(-1, 0, -1), which is singular (rows 0 and 2
    are equal): partial pivoting swaps rows 0/1, eliminates, and meets an exactly
    zero pivot at index 2 (linalg.cpp:84-103), as test_linalg.cpp:97-108 pins
    for band_factor."""
    from oracle.bindings import OracleError
    from paper_2305_04421_b200.solver import SingularMatrixError
    # Nx = 4, Ny = 2 on Lx = 4, Ly = 2: dx = dy = 1, dt = 1 (T = Nt), nu = 1 -> cx = cy = 1,
    # A diag = 5; plus sign with omega = 0.04: sigma dt = 5, Ahat diag = 0
    p = P.Problem(Lx=4.0, Ly=2.0, T=2.0, Nx=4, Ny=2, Nt=2, Nd=1, nu=1.0, omega=0.04, jhat_sign="plus")
    with pytest.raises(OracleError) as want:
        _oracle()(p)
    assert want.value.status == 3
    with pytest.raises(SingularMatrixError) as got:
        _kkt(p, mode)
    assert got.value.pivot_index == want.value.index
    assert got.value.pivot_index == 2


@pytest.mark.parametrize("mode", ["strict", "fast"])
def test_nonfinite_krylov_vector_names_the_iteration(mode):
    from oracle.bindings import OracleError
    from paper_2305_04421_b200.solver import GmresDivergenceError
    p = P.Problem(Lx=1.0, Ly=2.0, Nx=8, Ny=6, Nt=12, Nd=3, omega=1e-2, coarse_variant="scalar",
                  tol=1e-10, restart=10, max_iters=200)
    b = P.random_vec(3 * p.block, 26)
    b[5] = np.nan
    with pytest.raises(OracleError) as want:
        _oracle()(p).gmres_solve(b)
    assert want.value.status == 4
    k = _kkt(p, mode)
    with pytest.raises(GmresDivergenceError) as got:
        k.gmres_solve(b)
    assert got.value.iteration == want.value.index == 1
    assert "1" in str(got.value)
    # the context stays usable after the error
    ok = k.gmres_solve(P.random_vec(3 * p.block, 26))
    assert ok.converged


def test_nonfinite_krylov_vector_sharded_ranks_agree():
    """Every rank of a sharded solve raises at the same iteration, although only
    one slab holds the NaN (the decision uses the rank-ordered sums)."""
    import threading
    import torch
    from paper_2305_04421_b200.solver import GmresDivergenceError, HeatKKT, LocalGroup
    p = P.Problem(Lx=1.0, Ly=1.0, Nx=9, Ny=9, Nt=16, Nd=4, omega=1e-3, coarse_variant="scalar",
                  tol=1e-9, restart=8, max_iters=100)
    G = 2
    b = P.random_vec(3 * p.block, 31)
    b[3] = np.nan  # u block, node 1: rank 0's slab only
    grp = LocalGroup(G)
    res = [None] * G

    def work(r):
        try:
            torch.cuda.set_device(0)
            k = HeatKKT(p, mode="fast", rank=r, nranks=G, local_group=grp)
            k.gmres_solve(k.local_slab(b))
            res[r] = "no error"
        except GmresDivergenceError as e:
            res[r] = e.iteration
        except Exception as e:  # noqa: BLE001
            res[r] = repr(e)

    ts = [threading.Thread(target=work, args=(r,)) for r in range(G)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout=120)
    assert not any(t.is_alive() for t in ts), "a rank hung after the other one left"
    assert res == [1, 1], res


def test_restart_below_one_is_a_config_error():
    from oracle.bindings import OracleError
    from paper_2305_04421_b200.solver import ConfigError
    p = P.Problem(Nx=4, Ny=4, Nt=4, Nd=2, restart=0)
    with pytest.raises(OracleError) as want:
        _oracle()(p)
    assert want.value.status == 2
    for bad in (0, -3):
        with pytest.raises(ConfigError, match="restart must be >= 1"):
            _kkt(p.replace(restart=bad), "fast")
    _kkt(p.replace(restart=None), "fast")  # std::nullopt: full GMRES
    _kkt(p.replace(restart=1), "fast")


def test_plus_sign_large_grid_without_dominance_is_refused():
    # nx = 130 > 128 selects the unpivoted block recursion in FAST mode
    base = dict(Lx=1.0, Ly=1.0, Nx=131, Ny=4, Nt=4, Nd=2, nu=1e-4, coarse_variant="scalar", jhat_sign="plus")
    # dt = 0.25, sqrt(omega) = 0.1: the shift 2.5 exceeds 1 -> not diagonally dominant
    with pytest.raises(NotImplementedError, match="diagonally dominant"):
        _kkt(P.Problem(omega=1e-2, **base), "fast")
    # dt = 0.25 < sqrt(omega) = 0.5: dominant, the block recursion is valid and
    # matches the reference's pivoting factorisation (which never swaps here)
    p = P.Problem(omega=0.25, **base)
    r = P.random_vec(3 * p.block, 7)
    want = _oracle()(p).apply_P_inv(r)
    got = _kkt(p, "fast").apply_P_inv(r).cpu().numpy()
    B = p.block
    for k in range(3):
        e = np.linalg.norm(got[k * B:(k + 1) * B] - want[k * B:(k + 1) * B]) / np.linalg.norm(want[k * B:(k + 1) * B])
        assert e <= 1e-10, (k, e)
