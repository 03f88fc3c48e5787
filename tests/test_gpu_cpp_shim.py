"""GPU: the reference-side C++ binding (include/kktdd_gpu.hpp) over the C-ABI.

tests/cpp/test_reference_cases.cpp restates a subset of the reference's own
doctest cases (test_heat_operators / test_kkt / test_schur / test_gmres /
test_experiments) against the binding; tests/cpp/run_single_driver.cpp is
run_single's wiring (experiments.cpp:33-69) written with it.  Both are plain
C++20 programs linked to libkktdd_b200.so (built by tests/cpp/Makefile from
__graft_entry__.build()); here they run on the device, in FAST and in STRICT
arithmetic, and the driver's record is compared with the CPU oracle's
run_single.
"""
import json
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))
BUILD = os.path.join(HERE, "cpp", "_build")


def _exe(name):
    path = os.path.join(BUILD, name)
    if not os.path.exists(path):
        r = subprocess.run(["make", "-s", "-C", os.path.join(HERE, "cpp")], capture_output=True, text=True)
        assert r.returncode == 0, r.stderr[-2000:]
    return path


@pytest.mark.parametrize("arith", ["fast", "strict"])
def test_reference_cases_through_the_cpp_binding(arith):
    env = dict(os.environ, KKTDD_ARITH=arith)
    r = subprocess.run([_exe("test_reference_cases")], env=env, capture_output=True, text=True, timeout=900)
    tail = r.stdout[-3000:]
    out_dir = os.path.join(os.path.dirname(HERE), "gpurun_out")
    if os.path.isdir(out_dir):  # keep the full case list next to the other GPU-run artefacts
        open(os.path.join(out_dir, f"cpp_shim_{arith}.log"), "w").write(r.stdout + r.stderr)
    assert r.returncode == 0, tail + r.stderr[-1000:]
    last = r.stdout.strip().splitlines()[-1]
    assert "failed: 0 | assertions" in last and "| failed: 0" in last.split("assertions")[1], last
    ncases = int(last.split("test cases:")[1].split("|")[0])
    assert ncases >= 30, last


@pytest.mark.parametrize("args,problem", [
    (["9", "7", "12", "3", "0.01", "scalar"], dict(Nx=9, Ny=7, Nt=12, Nd=3, omega=1e-2, coarse_variant="scalar")),
    (["4", "5", "8", "2", "0.001", "per-dof"], dict(Nx=4, Ny=5, Nt=8, Nd=2, omega=1e-3, coarse_variant="per-dof")),
])
def test_run_single_driver_matches_the_reference_record(args, problem):
    from oracle import bindings
    from paper_2305_04421_b200 import problems as P
    if not bindings.available("ref"):
        pytest.skip("oracle/_ref not built")
    want, _, _ = bindings.Ref.run_single(P.Problem(**problem))  # the reference's own run_single
    r = subprocess.run([_exe("run_single_driver"), *args, "strict"], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    got = json.loads(r.stdout.strip().splitlines()[-1])
    assert got["kkt_run_single_agrees"] is True
    assert got["iterations"] == want["iterations"] and got["converged"] == bool(want["converged"])
    assert got["true_final_relres"] == want["true_final_relres"]      # STRICT: bitwise the reference
    assert got["objective"] == want["objective"]
    f = subprocess.run([_exe("run_single_driver"), *args], capture_output=True, text=True, timeout=600)
    fast = json.loads(f.stdout.strip().splitlines()[-1])
    assert abs(fast["iterations"] - want["iterations"]) <= 1
    assert abs(fast["objective"] - want["objective"]) <= 1e-6 * abs(want["objective"])


def test_driver_exit_code_for_config_errors():
    # 7 % 3 != 0 -> ConfigError -> exit 1, as the reference CLI (kktdd_cli.cpp:263-267)
    r = subprocess.run([_exe("run_single_driver"), "4", "4", "7", "3", "0.01"], capture_output=True, text=True)
    assert r.returncode == 1 and "not divisible" in r.stderr
