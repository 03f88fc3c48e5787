"""CPU tests of the host side: the C-ABI library loads and exports every
symbol include/kktdd_b200.h declares (no device calls), the struct mirror
matches the header, and the seeded input generator is deterministic and
chunk-independent.
"""
import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest

from paper_2305_04421_b200 import _abi, problems as P

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "kktdd_b200.h")


@pytest.fixture(scope="module")
def lib():
    from paper_2305_04421_b200 import build
    from paper_2305_04421_b200 import solver
    if not os.path.exists(solver.LIB_PATH):
        build.build()
    return solver.lib()


def declared():
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"\b(kkt_[A-Za-z0-9_]+)\s*\(", txt)))


def test_header_declares_the_boundary():
    names = declared()
    for must in ["kkt_ctx_create", "kkt_apply_K", "kkt_apply_P_inv", "kkt_gmres_solve",
                 "kkt_gmres_solve_host", "kkt_apply_rasq", "kkt_apply_two_level", "kkt_apply_shat",
                 "kkt_forward_solve_window", "kkt_adjoint_solve_window", "kkt_coarse_restrict"]:
        assert must in names


def test_library_exports_every_declared_symbol(lib):
    out = subprocess.run(["nm", "-D", "--defined-only", lib._name], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (kkt_[A-Za-z0-9_]+)", out))
    missing = [n for n in declared() if n not in exported]
    assert not missing, missing
    for n in declared():
        getattr(lib, n)  # resolvable through ctypes


def test_library_is_sm100a(lib):
    out = subprocess.run(["cuobjdump", "--list-elf", lib._name], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_desc_defaults_match_reference(lib):
    d = _abi.ProblemDesc()
    lib.kkt_problem_desc_default(C.byref(d))
    ref = P.Problem()  # config.hpp:36-50 defaults mirrored in problems.Problem
    assert (d.Lx, d.Ly, d.T, d.Nx, d.Ny, d.Nt, d.nu, d.omega, d.Nd) == (
        ref.Lx, ref.Ly, ref.T, ref.Nx, ref.Ny, ref.Nt, ref.nu, ref.omega, ref.Nd)
    assert d.precond == P.PRECOND[ref.precond] and d.coarse_variant == P.COARSE[ref.coarse_variant]
    assert d.tol == ref.tol and d.max_iters == ref.max_iters and d.restart == -1  # KKT_NO_RESTART = std::nullopt
    assert d.happy_breakdown_tol == ref.happy_breakdown_tol


def test_status_strings(lib):
    lib.kkt_status_string.restype = C.c_char_p
    assert lib.kkt_status_string(0) == b"ok"
    assert lib.kkt_status_string(_abi.KKT_ESINGULAR) == b"singular matrix"


def test_create_without_device_fails_loudly(lib):
    """No GPU here: context creation must fail with a CUDA status, never fall back."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("a device is present")
    d = _abi.desc_from_problem(P.config(0))
    h = C.c_void_p()
    st = lib.kkt_ctx_create(C.byref(d), None, C.byref(h))
    assert st == _abi.KKT_ECUDA and not h.value


def test_config_errors_precede_the_device(lib):
    """ProblemConfig::validate (config.cpp:5-22) runs before any CUDA call, so the
    reference's ConfigError cases come back as KKT_ECONFIG with its messages even
    without a device -- including gmres restart < 1 (config.cpp:21); only
    KKT_NO_RESTART (-1) means std::nullopt."""
    lib.kkt_create_error.restype = C.c_char_p
    base = P.config(0)
    cases = [(base.replace(restart=0), b"gmres restart must be >= 1"),
             (base.replace(restart=-7), b"gmres restart must be >= 1"),
             (base.replace(Nd=5), b"is not divisible by"),
             (base.replace(omega=0.0), b"omega must be > 0"),
             (base.replace(max_iters=0), b"max_iters must be >= 1"),
             (base.replace(Nx=1), b"mesh needs Nx, Ny >= 2")]
    for p, msg in cases:
        d = _abi.desc_from_problem(p)
        h = C.c_void_p()
        st = lib.kkt_ctx_create(C.byref(d), None, C.byref(h))
        assert st == _abi.KKT_ECONFIG and not h.value, (p, st)
        assert msg in lib.kkt_create_error(), lib.kkt_create_error()
    assert _abi.desc_from_problem(base.replace(restart=None)).restart == -1
    assert "#define KKT_NO_RESTART (-1)" in open(HEADER).read()


def test_solver_refuses_without_cuda():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a device is present")
    from paper_2305_04421_b200.solver import HeatKKT
    with pytest.raises(RuntimeError):
        HeatKKT(P.config(0))


# ---------------------------------------------------------------------------
# input generator
# ---------------------------------------------------------------------------
def test_generator_is_counter_based():
    a = P.normal(7, 1, 1000)
    b = np.concatenate([P.normal(7, 1, 300), P.normal(7, 1, 700, offset=300)])
    assert np.array_equal(a, b)
    c = P.normal(7, 1, 1000, chunk=64)
    assert np.array_equal(a, c)
    assert not np.array_equal(a, P.normal(7, 2, 1000))
    assert abs(a.mean()) < 0.1 and abs(a.std() - 1.0) < 0.1
    u = P.uniform01(3, 0, np.arange(10000, dtype=np.uint64))
    assert u.min() > 0.0 and u.max() <= 1.0


def test_rhs_slices_agree_with_full_field():
    p = P.config(0)
    tgt, u0 = P.target_and_u0(0, p)
    part, _ = P.target_and_u0(0, p, n_lo=17, n_hi=32)
    assert np.array_equal(tgt[16:32], part)
    b = P.kkt_rhs(0, p)
    assert b.size == 3 * p.block
    assert np.array_equal(b[:p.block], (p.mass_scale * tgt).reshape(-1))
    assert not np.any(b[p.block:2 * p.block])


def test_baseline_config_sizes():
    # SURVEY.md §8 size table
    rows = {0: (961, 64, 4, 184512), 1: (16129, 512, 16, 24774144), 2: (261121, 1024, 64, 802163712),
            3: (65025, 4096, 32, 799027200), 4: (1046529, 1024, 128, 3214937088)}
    for cfg, (nsp, nt, nd, unknowns) in rows.items():
        p = P.config(cfg)
        assert (p.n_sp, p.Nt, p.Nd, 3 * p.block) == (nsp, nt, nd, unknowns)
    assert P.config(1).mass_scale == pytest.approx(1.1920928955078125e-07)


def test_config4_modes_recorded():
    a, k, l, m = P._modes_c4(P.SEED + 4)
    assert a.shape == (8,) and k.min() >= 1 and k.max() <= 8 and l.min() >= 1 and m.max() <= 8


def test_bench_roofline_bytes():
    import importlib.util
    spec = importlib.util.spec_from_file_location("bench", os.path.join(ROOT, "bench.py"))
    bench = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(bench)
    p = P.config(1)
    vec = 3 * 512 * 16129 * 8
    # 44 iterations of GMRES(30): j = 0..29 then 0..13
    b, launches = bench.mgs_model(p, 44, mode="strict")   # MGS: (4j + 5) vector passes
    assert b == (4 * (435 + 91) + 5 * 44) * vec and launches == (435 + 91) + 2 * 44
    assert bench.mgs_model(p, 44, ranks=2, mode="strict")[0] == b // 2
    b, launches = bench.mgs_model(p, 44)                  # one-reduction MGS: (2j + 5)
    assert b == (2 * (435 + 91) + 5 * 44) * vec
    assert launches == sum(2 * -(-(j + 1) // 16) + 1 for j in list(range(30)) + list(range(14)))
    # four transform passes: 2 * 2 * Nt * n_sp * (nx + ny) FLOPs
    assert bench.spectral_flops(p) == 4 * 512 * 16129 * 254
    # RASQ sweep: (2Nt + Nd - 1) * 5 planes + (2m+1) * F
    F = 8 * 16129 * (2 * 127 + 1)
    assert bench.sweep_bytes(p) == (2 * 512 + 15) * 5 * 16129 * 8 + 65 * F


def test_mode_names():
    assert _abi.MODES == {"fast": 0, "strict": 1, "spectral": 2}
    txt = open(HEADER).read()
    assert "KKT_MODE_SPECTRAL = 2" in txt



def test_smoke_problem_converges_in_the_oracle():
    """__graft_entry__.smoke() checks the device solve against the oracle on a
    small problem; that problem must converge in the reference too (with
    GMRES(12) it stagnates there, so smoke uses GMRES(30): 36 iterations)."""
    import ast
    from oracle import bindings
    if not bindings.available("orc"):
        pytest.skip("oracle restatement not built")
    src = open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "__graft_entry__.py")).read()
    call = [n for n in ast.walk(ast.parse(src)) if isinstance(n, ast.Call) and getattr(n.func, "attr", "") == "Problem"][0]
    kw = {k.arg: ast.literal_eval(k.value) for k in call.keywords}
    p = P.Problem(**kw)
    out = bindings.Orc(p).gmres_solve(P.kkt_rhs(0, p))
    assert out["converged"] and out["iterations"] < p.max_iters, out["iterations"]
