"""ctypes mirror of the POD structs in include/kktdd_b200.h."""
from __future__ import annotations

import ctypes as C

from .problems import COARSE, FORM, PRECOND, SIGN, Problem

KKT_OK = 0
KKT_EINVAL = 1
KKT_ECONFIG = 2
KKT_ESINGULAR = 3
KKT_EDIVERGED = 4
KKT_ECUDA = 5
KKT_ENCCL = 6
KKT_EUNSUPPORTED = 7

MODE_FAST = 0
MODE_STRICT = 1
MODE_SPECTRAL = 2
MODES = {"fast": MODE_FAST, "strict": MODE_STRICT, "spectral": MODE_SPECTRAL}


class ProblemDesc(C.Structure):
    _fields_ = [
        ("Lx", C.c_double), ("Ly", C.c_double), ("T", C.c_double),
        ("Nx", C.c_int32), ("Ny", C.c_int32), ("Nt", C.c_int32),
        ("nu", C.c_double), ("omega", C.c_double),
        ("Nd", C.c_int32),
        ("precond", C.c_int32), ("coarse_variant", C.c_int32),
        ("two_level_form", C.c_int32), ("jhat_sign", C.c_int32),
        ("tol", C.c_double), ("max_iters", C.c_int32), ("restart", C.c_int32),
        ("happy_breakdown_tol", C.c_double),
    ]


class RuntimeOpts(C.Structure):
    _fields_ = [
        ("mode", C.c_int32), ("device", C.c_int32),
        ("rank", C.c_int32), ("nranks", C.c_int32),
        ("nccl_unique_id", C.c_void_p), ("stream", C.c_void_p),
        ("local_group", C.c_void_p),
    ]


class GmresResult(C.Structure):
    _fields_ = [
        ("converged", C.c_int32), ("iterations", C.c_int32),
        ("true_final_relres", C.c_double), ("history_len", C.c_int32),
    ]


class RunRecordC(C.Structure):
    _fields_ = [
        ("iterations", C.c_int32), ("converged", C.c_int32),
        ("true_final_relres", C.c_double), ("objective", C.c_double),
        ("setup_seconds", C.c_double), ("solve_seconds", C.c_double),
    ]


def desc_from_problem(p: Problem) -> ProblemDesc:
    return ProblemDesc(
        Lx=p.Lx, Ly=p.Ly, T=p.T, Nx=p.Nx, Ny=p.Ny, Nt=p.Nt, nu=p.nu, omega=p.omega, Nd=p.Nd,
        precond=PRECOND[p.precond], coarse_variant=COARSE[p.coarse_variant],
        two_level_form=FORM[p.two_level_form], jhat_sign=SIGN[p.jhat_sign],
        tol=p.tol, max_iters=p.max_iters, restart=(-1 if p.restart is None else int(p.restart)),
        happy_breakdown_tol=p.happy_breakdown_tol,
    )


def dptr(a) -> C.c_void_p:
    """Data pointer of a numpy array or torch tensor."""
    if hasattr(a, "data_ptr"):
        return C.c_void_p(a.data_ptr())
    return a.ctypes.data_as(C.c_void_p)
