"""The end-to-end run record (reference include/kktdd/experiments.hpp:14-31,
src/experiments.cpp:33-69 and :179-208) on the device.

``run_single(problem)`` does what the reference's ``run_single(cfg)`` does —
operators, partition and preconditioner setup, the model problem's right-hand
side (model_problem.hpp), GMRES with apply_K / apply_P_inv, the objective of
the solution — through one C-ABI call, ``kkt_run_single``.  Non-convergence is
recorded, not an error.  ``to_json_string`` writes the reference's JSON record
(same keys, same layout: nlohmann's ``dump(2)`` sorts keys).
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import json
from typing import Optional

import numpy as np

from . import _abi
from .problems import Problem
from .solver import _raise, lib


@dataclasses.dataclass
class RunRecord:
    """RunRecord (experiments.hpp:14-22)."""
    config: Problem
    iterations: int = 0
    converged: bool = False
    true_final_relres: float = 0.0
    objective: float = 0.0
    setup_seconds: float = 0.0
    solve_seconds: float = 0.0
    solution: Optional[np.ndarray] = dataclasses.field(default=None, repr=False)


def run_single(problem: Problem, mode: str = "fast", device: int = 0,
               want_solution: bool = False) -> RunRecord:
    """run_single(cfg) (experiments.cpp:33-69) on one GPU."""
    desc = _abi.desc_from_problem(problem)
    opts = _abi.RuntimeOpts(mode=_abi.MODE_STRICT if mode == "strict" else _abi.MODE_FAST,
                            device=device, rank=0, nranks=1)
    rec = _abi.RunRecordC()
    x = np.empty(3 * problem.block) if want_solution else None
    L = lib()
    st = L.kkt_run_single(C.byref(desc), C.byref(opts), C.byref(rec),
                          x.ctypes.data_as(C.c_void_p) if x is not None else None)
    if st != 0:
        _raise(st, L.kkt_create_error().decode(), -1)
    return RunRecord(problem, rec.iterations, bool(rec.converged), rec.true_final_relres,
                     rec.objective, rec.setup_seconds, rec.solve_seconds, x)


def to_json_string(rec: RunRecord) -> str:
    """to_json_string(RunRecord) (experiments.cpp:179-208)."""
    c = rec.config
    j = {
        "lx": c.Lx, "ly": c.Ly, "t_final": c.T, "nx": c.Nx, "ny": c.Ny, "nt": c.Nt,
        "nu": c.nu, "omega": c.omega, "nd": c.Nd, "precond": c.precond,
        "coarse_variant": c.coarse_variant,
        "two_level_form": c.two_level_form, "jhat_sign": c.jhat_sign,
        "tol": c.tol, "max_iters": c.max_iters, "restart": c.restart,
        "iterations": rec.iterations, "converged": rec.converged,
        "true_final_relres": rec.true_final_relres, "objective": rec.objective,
        "setup_seconds": rec.setup_seconds, "solve_seconds": rec.solve_seconds,
    }
    return json.dumps(j, indent=2, sort_keys=True)
