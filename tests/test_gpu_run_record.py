"""GPU: the f1 run record — kkt_run_single (experiments.cpp:33-69) against the
reference's run_single on the same config: STRICT bitwise (iterations,
convergence, true relres, objective, solution), FAST within the north-star
tolerances; the model right-hand side and evaluate_objective (kkt.cpp:88-108)
bitwise; the acceptance suite's objective criterion (acceptance_main.cpp:433-457)."""
import numpy as np
import pytest

from paper_2305_04421_b200 import problems as P

pytestmark = pytest.mark.gpu

CASES = [
    P.Problem(Lx=1.0, Ly=2.0, Nx=8, Ny=6, Nt=12, Nd=3, omega=1e-2, coarse_variant="scalar",
              tol=1e-10, restart=10, max_iters=200),
    P.Problem(Lx=1.0, Ly=2.0, Nx=10, Ny=12, Nt=20, Nd=5, omega=1e-3, coarse_variant="per-dof",
              tol=1e-8, restart=None, max_iters=200),
    P.config(0, coarse="scalar"),
]
IDS = ["small_scalar", "small_per_dof", "config0"]


def rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


@pytest.mark.parametrize("p", CASES, ids=IDS)
def test_run_single_vs_reference(p):
    from oracle.bindings import Ref
    from paper_2305_04421_b200.experiments import run_single, to_json_string
    want, text, xw = Ref.run_single(p, want_x=True)
    s = run_single(p, mode="strict", want_solution=True)
    assert s.iterations == want["iterations"] and s.converged == want["converged"]
    assert s.true_final_relres == want["true_final_relres"]
    assert s.objective == want["objective"]
    assert np.array_equal(s.solution, xw)
    f = run_single(p, mode="fast", want_solution=True)
    assert f.converged and abs(f.iterations - want["iterations"]) <= 1
    assert abs(f.objective - want["objective"]) <= 1e-8 * abs(want["objective"])
    B = p.block
    for k in range(3):
        assert rel(f.solution[k * B:(k + 1) * B], xw[k * B:(k + 1) * B]) <= max(1e-9, 10 * p.tol)
    # the JSON record has the reference's keys; only the timings differ
    import json
    a, b = json.loads(to_json_string(s)), json.loads(text)
    assert a.keys() == b.keys()
    for k in a:
        if not k.endswith("_seconds"):
            assert a[k] == b[k], k
    # acceptance criterion 10: objective at or below the zero-control state's
    assert f.objective <= Ref(p).zero_control_objective() * (1.0 + 1e-8)


def test_model_rhs_and_objective_bitwise():
    from oracle.bindings import Ref
    from paper_2305_04421_b200.solver import HeatKKT
    p = CASES[1]
    ref = Ref(p)
    for mode in ("strict", "fast"):
        k = HeatKKT(p, mode=mode)
        b, t = k.model_rhs()
        rb, rt = ref.model_rhs()
        assert np.array_equal(b, rb) and np.array_equal(t, rt)
        u, z = P.random_vec(p.block, 41), P.random_vec(p.block, 42)
        want = ref.evaluate_objective(u, z)
        got = k.evaluate_objective(u, z, t)
        if mode == "strict":
            assert got == want
        else:
            assert abs(got - want) <= 1e-13 * abs(want)
