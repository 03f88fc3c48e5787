"""f3 on the GPU: the weak-scaling and omega sweeps (experiments.cpp:97-142)
run through the device run_single, against the reference's own sweeps.

STRICT: every CSV column except the two timings (setup_s, solve_s) identical
to the reference's CSV — iterations, convergence, true relres and objective
bitwise.  FAST: the same grid, iterations within +-1 and converged where the
reference converged.
"""
import pytest

from paper_2305_04421_b200 import experiments as E
from paper_2305_04421_b200 import problems as P

pytestmark = pytest.mark.gpu

BASE = P.Problem(Lx=1.0, Ly=2.0, Nx=6, Ny=6, T=1.0, coarse_variant="per-dof", tol=1e-6,
                 max_iters=420, restart=None)
WEAK = dict(steps=4, nts=[8, 12, 10, 16], omegas=[1e-2, 1e-4], preconds=["two-level", "one-level"])
OMEGA = dict(nt=12, nd=3, omegas=[1e-1, 1e-3, 1e-6], preconds=["two-level", "none"])


def _strip_times(text):
    out = []
    for ln in text.splitlines():
        out.append(ln if ln.startswith("#") or ln.startswith("nt,") else ",".join(ln.split(",")[:-2]))
    return out


def _runs(kind, mode):
    if kind == "weak":
        return E.weak_scaling_sweep(BASE, WEAK["steps"], WEAK["nts"], WEAK["omegas"], WEAK["preconds"], mode=mode)
    return E.omega_sweep(BASE, OMEGA["nt"], OMEGA["nd"], OMEGA["omegas"], OMEGA["preconds"], mode=mode)


def _ref_csv(kind):
    from oracle.bindings import Ref
    if kind == "weak":
        return Ref.sweep_csv(BASE, "weak", WEAK["omegas"], WEAK["preconds"], steps=WEAK["steps"], nts=WEAK["nts"])
    return Ref.sweep_csv(BASE, "omega", OMEGA["omegas"], OMEGA["preconds"], nt=OMEGA["nt"], nd=OMEGA["nd"])


@pytest.mark.parametrize("kind", ["weak", "omega"])
def test_sweep_strict_matches_reference_csv(kind):
    want = _ref_csv(kind)
    got = E.to_csv(_runs(kind, "strict"))
    assert _strip_times(got) == _strip_times(want)


@pytest.mark.parametrize("kind", ["weak", "omega"])
def test_sweep_fast_iterations(kind):
    want = [ln.split(",") for ln in _ref_csv(kind).splitlines()[1:] if not ln.startswith("#")]
    got = _runs(kind, "fast")
    assert len(got.rows) == len(want)
    for rec, w in zip(got.rows, want):
        assert (rec.config.Nt, rec.config.precond) == (int(w[0]), w[4])
        assert abs(rec.iterations - int(w[8])) <= 1, (rec.config, rec.iterations, w[8])
        if w[9] == "true":
            assert rec.converged
