"""BASELINE configurations and the seeded, counter-based input generator.

The harness builds every right-hand side on the host through ONE code path
(this module) and hands the same arrays to the device solver and to the CPU
reference, so inputs are bit-identical on both sides.

RHS assembly follows ``assemble_rhs`` (reference proj/src/kkt.cpp:29-48):
``f_u[n,i,j] = ms * target(i*dx, j*dy, n*dt)``, ``f_z = 0``,
``f[1,i,j] = u0(i*dx, j*dy)``; ``b = to_kkt() = [f_u; f_z; f]`` (kkt.cpp:21-27).
Noise is drawn per flat index of the reference layout
(proj/include/kktdd/layout.hpp:24-37) from SplitMix64(seed, stream, index)
-> two uniforms -> Box-Muller, never from an implementation-defined
``std::normal_distribution``.
"""
from __future__ import annotations

import dataclasses
import math
from typing import Optional

import numpy as np

# Enum values mirror include/kktdd_b200.h (and proj/include/kktdd/config.hpp:12-21).
PRECOND = {"none": 0, "one-level": 1, "two-level": 2, "dense-schur": 3, "true-schur": 4}
COARSE = {"scalar": 0, "per-dof": 1}
FORM = {"literal": 0, "multiplicative": 1, "additive": 2}
SIGN = {"plus": 0, "minus": 1}


@dataclasses.dataclass
class Problem:
    """Python mirror of ProblemConfig + GmresParams (config.hpp:23-68).

    Defaults are the reference's (config.hpp:36-50, :24-27)."""

    Lx: float = 1.0
    Ly: float = 2.0
    T: float = 1.0
    Nx: int = 16
    Ny: int = 16
    Nt: int = 100
    nu: float = 1.0
    omega: float = 1e-3
    Nd: int = 5
    precond: str = "two-level"
    coarse_variant: str = "per-dof"
    two_level_form: str = "multiplicative"
    jhat_sign: str = "minus"
    tol: float = 1e-6
    max_iters: int = 420
    restart: Optional[int] = None
    happy_breakdown_tol: float = 1e-14

    # derived quantities, computed with the reference's expressions (config.hpp:52-65)
    @property
    def dx(self) -> float:
        return self.Lx / self.Nx

    @property
    def dy(self) -> float:
        return self.Ly / self.Ny

    @property
    def dt(self) -> float:
        return self.T / self.Nt

    @property
    def nx_int(self) -> int:
        return self.Nx - 1

    @property
    def ny_int(self) -> int:
        return self.Ny - 1

    @property
    def n_sp(self) -> int:
        return self.nx_int * self.ny_int

    @property
    def block(self) -> int:
        return self.Nt * self.n_sp

    @property
    def mass_scale(self) -> float:
        return self.dt * self.dx * self.dy

    def replace(self, **kw) -> "Problem":
        return dataclasses.replace(self, **kw)


# ---------------------------------------------------------------------------
# counter-based RNG: SplitMix64 finaliser over (seed, stream, index)
# ---------------------------------------------------------------------------
_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)
_GAMMA = np.uint64(0x9E3779B97F4A7C15)


def _mix64(z: np.ndarray) -> np.ndarray:
    z = z.astype(np.uint64, copy=True)
    with np.errstate(over="ignore"):
        z ^= z >> np.uint64(30)
        z *= np.uint64(0xBF58476D1CE4E5B9)
        z ^= z >> np.uint64(27)
        z *= np.uint64(0x94D049BB133111EB)
        z ^= z >> np.uint64(31)
    return z


def _key(seed: int, stream: int) -> np.uint64:
    k = _mix64(np.array([(seed * 0x100000001B3 + stream) & 0xFFFFFFFFFFFFFFFF], dtype=np.uint64))
    return k[0]


def uniform01(seed: int, stream: int, index: np.ndarray) -> np.ndarray:
    """Uniform in (0, 1] from the 53 high bits of SplitMix64(key + (i+1)*gamma)."""
    idx = np.asarray(index, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = _key(seed, stream) + (idx + np.uint64(1)) * _GAMMA
    z = _mix64(z)
    return ((z >> np.uint64(11)).astype(np.float64) + 1.0) * (1.0 / 9007199254740992.0)


def normal(seed: int, stream: int, n: int, offset: int = 0, chunk: int = 1 << 22) -> np.ndarray:
    """n standard normals, element i from counters (2i, 2i+1) via Box-Muller."""
    out = np.empty(n, dtype=np.float64)
    for lo in range(0, n, chunk):
        hi = min(n, lo + chunk)
        i = np.arange(lo + offset, hi + offset, dtype=np.uint64)
        u1 = uniform01(seed, stream, 2 * i)
        u2 = uniform01(seed, stream, 2 * i + np.uint64(1))
        out[lo:hi] = np.sqrt(-2.0 * np.log(u1)) * np.cos(2.0 * math.pi * u2)
    return out


# ---------------------------------------------------------------------------
# BASELINE.json configs (restated in BASELINE.md §3)
# ---------------------------------------------------------------------------
SEED = 230504421


def config(idx: int, *, Nd: Optional[int] = None, coarse: str = "scalar",
           precond: str = "two-level") -> Problem:
    common = dict(Lx=1.0, Ly=1.0, T=1.0, precond=precond, coarse_variant=coarse,
                  two_level_form="multiplicative", jhat_sign="minus", max_iters=420)
    if idx == 0:
        return Problem(Nx=32, Ny=32, Nt=64, nu=1.0, omega=1e-2, Nd=4 if Nd is None else Nd,
                       tol=1e-8, restart=30, **common)
    if idx == 1:
        return Problem(Nx=128, Ny=128, Nt=512, nu=1.0, omega=1e-3, Nd=16 if Nd is None else Nd,
                       tol=1e-8, restart=30, **common)
    if idx == 2:
        return Problem(Nx=512, Ny=512, Nt=1024, nu=0.1, omega=1e-2, Nd=64 if Nd is None else Nd,
                       tol=1e-8, restart=None, **common)
    if idx == 3:
        return Problem(Nx=256, Ny=256, Nt=4096, nu=1.0, omega=1e-2, Nd=32 if Nd is None else Nd,
                       tol=1e-8, restart=20, **common)
    if idx == 4:
        return Problem(Nx=1024, Ny=1024, Nt=1024, nu=1.0, omega=1e-4, Nd=128 if Nd is None else Nd,
                       tol=1e-8, restart=20, **common)
    raise ValueError(f"unknown config {idx}")


def _grid(p: Problem):
    """x_i, y_j for the interior points (1-based i, j; layout.hpp:22)."""
    x = np.arange(1, p.nx_int + 1, dtype=np.float64) * p.dx
    y = np.arange(1, p.ny_int + 1, dtype=np.float64) * p.dy
    return x, y


def _modes_c4(seed: int):
    """Config 4's 8 seeded modes: a_q ~ N(0,1); k_q, l_q, m_q in 1..8."""
    a = normal(seed, 7, 8)
    u = uniform01(seed, 8, np.arange(24, dtype=np.uint64))
    ints = (np.floor(u * 8.0).astype(np.int64) + 1).reshape(3, 8)
    return a, ints[0], ints[1], ints[2]


def target_and_u0(cfg_idx: int, p: Problem, seed: int = SEED, n_lo: int = 1, n_hi: Optional[int] = None):
    """(target[n_lo..n_hi] as (nodes, n_sp), u0 as (n_sp,)) for BASELINE config cfg_idx.

    Noise is drawn at the flat reference-layout index (n-1)*n_sp + p so any node
    range gives the same values as the full field."""
    if n_hi is None:
        n_hi = p.Nt
    x, y = _grid(p)
    X = np.tile(x, p.ny_int)            # i inner
    Y = np.repeat(y, p.nx_int)          # j outer
    t = np.arange(n_lo, n_hi + 1, dtype=np.float64) * p.dt
    nodes = n_hi - n_lo + 1
    nsp = p.n_sp
    pi = math.pi
    if cfg_idx in (0, 3):
        sp = np.sin(pi * X) * np.sin(pi * Y)
        tgt = np.cos(2 * pi * t)[:, None] * sp[None, :]
        tgt += 0.01 * normal(seed + cfg_idx, 1, nodes * nsp, offset=(n_lo - 1) * nsp).reshape(nodes, nsp)
        u0 = np.zeros(nsp)
    elif cfg_idx == 1:
        sp = np.sin(2 * pi * X) * np.sin(pi * Y)
        tgt = np.exp(-t)[:, None] * sp[None, :]
        tgt += 0.01 * normal(seed + cfg_idx, 1, nodes * nsp, offset=(n_lo - 1) * nsp).reshape(nodes, nsp)
        u0 = np.sin(pi * X) * np.sin(pi * Y)
    elif cfg_idx == 4:
        a, kq, lq, mq = _modes_c4(seed + cfg_idx)
        tgt = np.zeros((nodes, nsp))
        for q in range(8):
            tgt += a[q] * np.cos(mq[q] * pi * t)[:, None] * (np.sin(kq[q] * pi * X) * np.sin(lq[q] * pi * Y))[None, :]
        u0 = np.zeros(nsp)
    else:
        raise ValueError(f"config {cfg_idx} has no target (config 2 uses random KKT vectors)")
    return tgt, u0


def kkt_rhs(cfg_idx: int, p: Problem, seed: int = SEED) -> np.ndarray:
    """b = [f_u; f_z; f] exactly as assemble_rhs + to_kkt (kkt.cpp:21-48)."""
    tgt, u0 = target_and_u0(cfg_idx, p, seed)
    B = p.block
    b = np.zeros(3 * B)
    b[:B] = (p.mass_scale * tgt).reshape(-1)
    b[2 * B: 2 * B + p.n_sp] = u0
    return b


def random_kkt(p: Problem, k: int, seed: int = SEED) -> np.ndarray:
    """Config 2's k-th seeded N(0,1) KKT vector (all three blocks)."""
    return normal(seed + 2, 100 + k, 3 * p.block)


def random_vec(n: int, seed: int, stream: int = 0) -> np.ndarray:
    """Uniform(-1, 1) test vector (the reference tests' random_vector shape, oracles.hpp:118-123)."""
    return 2.0 * uniform01(seed, stream, np.arange(n, dtype=np.uint64)) - 1.0
