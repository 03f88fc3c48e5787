"""The end-to-end run record (reference include/kktdd/experiments.hpp:14-31,
src/experiments.cpp:33-69 and :179-208) on the device.

``run_single(problem)`` does what the reference's ``run_single(cfg)`` does —
operators, partition and preconditioner setup, the model problem's right-hand
side (model_problem.hpp), GMRES with apply_K / apply_P_inv, the objective of
the solution — through one C-ABI call, ``kkt_run_single``.  Non-convergence is
recorded, not an error.  ``to_json_string`` writes the reference's JSON record
(same keys, same layout: nlohmann's ``dump(2)`` sorts keys).

The sweeps (experiments.cpp:73-142) run a grid of ``run_single`` on the
device with the reference's grid construction, skip rules and row order;
``to_csv`` writes the reference's CSV (experiments.cpp:144-177) byte for byte
(same columns, ``%.10g`` / ``%.3f`` formatting, ``# skipped`` trailer).
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import json
from typing import Callable, List, Optional, Sequence

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
    if mode not in _abi.MODES:
        raise ValueError(f"mode must be one of {sorted(_abi.MODES)}, got {mode!r}")
    opts = _abi.RuntimeOpts(mode=_abi.MODES[mode], device=device, rank=0, nranks=1)
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


# ---------------------------------------------------------------------------
# f3: the sweeps (experiments.hpp:34-60, experiments.cpp:73-177)
# ---------------------------------------------------------------------------
@dataclasses.dataclass
class SkippedRun:
    """SkippedRun (experiments.hpp:34-38): a grid point that never ran."""
    config: Problem
    reason: str


@dataclasses.dataclass
class SweepResult:
    """SweepResult (experiments.hpp:40-43): rows ordered by (precond, omega, nt)."""
    rows: List[RunRecord] = dataclasses.field(default_factory=list)
    skipped: List[SkippedRun] = dataclasses.field(default_factory=list)


RunProgress = Callable[[RunRecord], None]


def _run_grid(grid: Sequence[Problem], pre_skipped: Sequence[SkippedRun], mode: str,
              device: int, progress: Optional[RunProgress]) -> SweepResult:
    """run_grid (experiments.cpp:73-93): a failing run is recorded as skipped
    with its message; rows sorted by (to_string(precond), omega, Nt)."""
    sweep = SweepResult(skipped=list(pre_skipped))
    for cfg in grid:
        try:
            rec = run_single(cfg, mode=mode, device=device)
        except (ValueError, ArithmeticError) as e:  # the reference's std::exception cases
            sweep.skipped.append(SkippedRun(cfg, str(e)))
            continue
        sweep.rows.append(rec)
        if progress:
            progress(rec)
    sweep.rows.sort(key=lambda r: (r.config.precond, r.config.omega, r.config.Nt))
    return sweep


def weak_scaling_sweep(base: Problem, steps_per_subdomain: int, nt_list: Sequence[int],
                       omega_list: Sequence[float], precond_list: Sequence[str],
                       progress: Optional[RunProgress] = None, mode: str = "fast",
                       device: int = 0) -> SweepResult:
    """weak_scaling_sweep (experiments.cpp:97-124): Nd = Nt / steps for each Nt,
    crossed with the omega and preconditioner lists."""
    from .solver import ConfigError
    if steps_per_subdomain < 1:
        raise ConfigError("steps per subdomain must be >= 1")
    grid, skipped = [], []
    for precond in precond_list:
        for omega in omega_list:
            for nt in nt_list:
                cfg = base.replace(Nt=nt, omega=omega, precond=precond)
                if nt % steps_per_subdomain != 0:
                    skipped.append(SkippedRun(cfg.replace(Nd=1),
                                              f"Nt={nt} not divisible by steps={steps_per_subdomain}"))
                    continue
                grid.append(cfg.replace(Nd=nt // steps_per_subdomain))
    return _run_grid(grid, skipped, mode, device, progress)


def omega_sweep(base: Problem, nt: int, nd: int, omega_list: Sequence[float],
                precond_list: Sequence[str], progress: Optional[RunProgress] = None,
                mode: str = "fast", device: int = 0) -> SweepResult:
    """omega_sweep (experiments.cpp:126-142): regularisation sweep at fixed Nt, Nd."""
    grid = [base.replace(Nt=nt, Nd=nd, omega=omega, precond=precond)
            for precond in precond_list for omega in omega_list]
    return _run_grid(grid, [], mode, device, progress)


def _fmt(v: float, spec: str = "%.10g") -> str:
    return spec % v  # std::snprintf with the same conversion (experiments.cpp:23-27)


def csv_header() -> str:
    """csv_header (experiments.cpp:144-147)."""
    return ("nt,nd,steps_per_subdomain,omega,precond,coarse_variant,two_level_form,jhat_sign,"
            "iters,converged,final_relres,objective,setup_s,solve_s")


def csv_row(rec: RunRecord) -> str:
    """csv_row (experiments.cpp:149-166)."""
    c = rec.config
    return ",".join([str(c.Nt), str(c.Nd), str(c.Nt // c.Nd), _fmt(c.omega), c.precond,
                     c.coarse_variant, c.two_level_form, c.jhat_sign, str(rec.iterations),
                     "true" if rec.converged else "false", _fmt(rec.true_final_relres),
                     _fmt(rec.objective), _fmt(rec.setup_seconds, "%.3f"),
                     _fmt(rec.solve_seconds, "%.3f")])


def to_csv(sweep: SweepResult) -> str:
    """to_csv (experiments.cpp:168-177)."""
    out = csv_header() + "\n"
    for rec in sweep.rows:
        out += csv_row(rec) + "\n"
    for sk in sweep.skipped:
        out += (f"# skipped nt={sk.config.Nt} omega={_fmt(sk.config.omega)} "
                f"precond={sk.config.precond}: {sk.reason}\n")
    return out
