"""B200-native hot path of arXiv 2305.04421's heat-control KKT solve.

The product is libkktdd_b200.so (csrc/, sm_100a CUDA + C-ABI in
include/kktdd_b200.h); ``solver.HeatKKT`` is the Python mirror of the
reference's operator / preconditioner / Krylov interfaces over that ABI.
"""
from .problems import Problem, config, kkt_rhs  # noqa: F401

__all__ = ["Problem", "config", "kkt_rhs", "HeatKKT"]


def __getattr__(name):
    if name == "HeatKKT":
        from .solver import HeatKKT
        return HeatKKT
    raise AttributeError(name)
