"""Python host side of the B200 hot path: a thin mirror of the reference's
operator / preconditioner / Krylov interfaces (proj/include/kktdd/*.hpp) over
the C-ABI of libkktdd_b200.so (include/kktdd_b200.h).

``HeatKKT`` bundles what the reference keeps in ``HeatOperators``
(heat_operators.hpp:26-39), ``TimePartition`` (time_partition.hpp:26-42) and
``SchurSolver`` (schur.hpp:304-331).  Its methods keep the reference's names,
argument meaning and error behaviour (reference exception -> Python exception
of the same name).  Vectors are CUDA ``torch`` tensors (device memory) in the
reference layout; the ``*_host`` solve takes numpy arrays.

There is no CPU fallback: constructing a ``HeatKKT`` without the built library
or without a CUDA device raises.
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import os
from typing import Optional

import numpy as np

from . import _abi
from ._abi import GmresResult, ProblemDesc, RuntimeOpts, desc_from_problem, dptr
from .problems import Problem

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "_lib", "libkktdd_b200.so")
_P = C.c_void_p


class ConfigError(ValueError):
    """ConfigError (config.hpp:82-85)."""


class SingularMatrixError(ArithmeticError):
    """SingularMatrixError (linalg.hpp:14-19); ``pivot_index`` as in the reference."""

    def __init__(self, msg, pivot_index):
        super().__init__(msg)
        self.pivot_index = pivot_index


class GmresDivergenceError(ArithmeticError):
    """GmresDivergenceError (gmres.hpp:22-27); ``iteration`` as in the reference."""

    def __init__(self, msg, iteration):
        super().__init__(msg)
        self.iteration = iteration


class DeviceError(RuntimeError):
    pass


_lib = None


def lib():
    """Load libkktdd_b200.so; raises if it has not been built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"{LIB_PATH} is missing: build it with `python -m paper_2305_04421_b200.build` "
                "(there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        L.kkt_last_error.restype = C.c_char_p
        L.kkt_last_error.argtypes = [_P]
        L.kkt_last_error_index.argtypes = [_P]
        L.kkt_create_error.restype = C.c_char_p
        L.kkt_status_string.restype = C.c_char_p
        _lib = L
    return _lib


class LocalGroup:
    """In-process rank group (kkt_local_group_create): the ranks are host threads
    of this process sharing one device; exchanges are host-synchronised."""

    def __init__(self, nranks: int):
        h = _P()
        st = lib().kkt_local_group_create(C.c_int32(nranks), C.byref(h))
        if st != 0:
            raise RuntimeError("kkt_local_group_create failed")
        self.handle = h
        self.nranks = nranks

    def __del__(self):
        if getattr(self, "handle", None):
            lib().kkt_local_group_destroy(self.handle)
            self.handle = None


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    st = lib().kkt_nccl_unique_id(buf)
    if st != 0:
        _raise(st, lib().kkt_create_error().decode(), -1)
    return buf.raw


def exported_symbols():
    """Names declared in include/kktdd_b200.h (for the load/export test)."""
    import re
    hdr = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include",
                       "kktdd_b200.h")
    txt = open(hdr).read()
    return sorted(set(re.findall(r"\b(kkt_[A-Za-z0-9_]+)\s*\(", txt)))


def _raise(status, msg, index):
    if status == _abi.KKT_ECONFIG:
        raise ConfigError(msg)
    if status == _abi.KKT_ESINGULAR:
        raise SingularMatrixError(msg, index)
    if status == _abi.KKT_EDIVERGED:
        raise GmresDivergenceError(msg, index)
    if status == _abi.KKT_EINVAL:
        raise ValueError(msg)
    if status == _abi.KKT_EUNSUPPORTED:
        raise NotImplementedError(msg)
    raise DeviceError(f"status {status}: {msg}")


@dataclasses.dataclass
class GmresOutcome:
    """GmresResult (gmres.hpp:13-19)."""
    solution: object
    converged: bool
    iterations: int
    residual_history: np.ndarray
    true_final_relres: float


class HeatKKT:
    """Device context: HeatOperators + TimePartition + SchurSolver on one GPU."""

    def __init__(self, problem: Problem, mode: str = "fast", device: int = 0, stream=None,
                 rank: int = 0, nranks: int = 1, nccl_id: Optional[bytes] = None,
                 local_group=None):
        import torch
        if not torch.cuda.is_available():
            raise RuntimeError("HeatKKT needs a CUDA device (no CPU fallback)")
        self.problem = problem
        self.mode = mode
        self.device = torch.device("cuda", device)
        self._torch = torch
        L = lib()
        self._desc = desc_from_problem(problem)
        if stream is None:
            # a dedicated stream; every call is fenced against torch's current
            # stream on both sides (_pre/_post), so tensors flow in and out in
            # stream order without host synchronisation
            stream = torch.cuda.Stream(device=self.device)
        self.stream = stream
        self._nccl_id = C.create_string_buffer(nccl_id, 128) if nccl_id is not None else None
        if mode not in _abi.MODES:
            raise ValueError(f"mode must be one of {sorted(_abi.MODES)}, got {mode!r}")
        opts = RuntimeOpts(mode=_abi.MODES[mode],
                           device=device, rank=rank, nranks=nranks,
                           nccl_unique_id=C.cast(self._nccl_id, C.c_void_p) if self._nccl_id else None,
                           stream=C.c_void_p(stream.cuda_stream),
                           local_group=local_group.handle if local_group is not None else None)
        self.rank, self.nranks = rank, nranks
        h = _P()
        st = L.kkt_ctx_create(C.byref(self._desc), C.byref(opts), C.byref(h))
        if st != 0:
            _raise(st, L.kkt_create_error().decode(), L.kkt_create_error_index())
        self._h = h
        blk, nsp, nf, nl, lb = C.c_int64(), C.c_int32(), C.c_int32(), C.c_int32(), C.c_int64()
        L.kkt_layout(h, C.byref(blk), C.byref(nsp), C.byref(nf), C.byref(nl), C.byref(lb))
        self.global_block = blk.value
        self.block = lb.value          # rank-local block: vectors are local slabs
        self.n_sp = nsp.value
        self.node_first, self.node_last = nf.value, nl.value

    def local_slab(self, v):
        """This rank's slab [u; z; w] (or one block) of a global vector."""
        v = np.asarray(v)
        G, L, off = self.global_block, self.block, (self.node_first - 1) * self.n_sp
        if v.size == 3 * G:
            return np.concatenate([v[k * G + off:k * G + off + L] for k in range(3)])
        assert v.size == G
        return v[off:off + L].copy()

    # -- plumbing ----------------------------------------------------------
    def close(self):
        h = getattr(self, "_h", None)
        if h:
            lib().kkt_ctx_destroy(h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _pre(self):
        self.stream.wait_stream(self._torch.cuda.current_stream(self.device))

    def _post(self):
        self._torch.cuda.current_stream(self.device).wait_stream(self.stream)

    def _call(self, fn, *args):
        self._pre()
        st = getattr(lib(), fn)(self._h, *args)
        self._post()
        self._check(st)

    def _check(self, st):
        if st != 0:
            L = lib()
            _raise(st, L.kkt_last_error(self._h).decode(), L.kkt_last_error_index(self._h))

    def _dev(self, x, n=None):
        t = self._torch
        if not isinstance(x, t.Tensor):
            x = t.as_tensor(np.asarray(x, dtype=np.float64))
        x = x.to(device=self.device, dtype=t.float64).contiguous()
        if n is not None and x.numel() != n:
            raise ValueError(f"vector length {x.numel()}, expected {n}")
        return x

    def _empty(self, n):
        return self._torch.empty(n, dtype=self._torch.float64, device=self.device)

    def _unary(self, fn, x, n, out=None):
        x = self._dev(x, n)
        out = self._empty(n) if out is None else out
        self._call(fn, dptr(x), dptr(out))
        return out

    def synchronize(self):
        self._call("kkt_synchronize")

    def launch_count(self) -> int:
        c = C.c_int64()
        lib().kkt_launch_count(self._h, C.byref(c))
        return c.value

    def reset_launch_count(self):
        lib().kkt_reset_launch_count(self._h)

    def set_phase_timing(self, on: bool):
        lib().kkt_set_phase_timing(self._h, C.c_int32(int(on)))

    def phase_times(self):
        ms = (C.c_double * 4)()
        cnt = (C.c_int64 * 4)()
        lib().kkt_phase_times(self._h, ms, cnt)
        return list(ms), list(cnt)

    # -- heat operators (heat_operators.hpp:41-61) ----------------------------
    def apply_J(self, u, out=None): return self._unary("kkt_apply_J", u, self.block, out)
    def apply_JT(self, w, out=None): return self._unary("kkt_apply_JT", w, self.block, out)
    def apply_L(self, z, out=None): return self._unary("kkt_apply_L", z, self.block, out)
    def apply_LT(self, w, out=None): return self._unary("kkt_apply_LT", w, self.block, out)
    def apply_Mu(self, u, out=None): return self._unary("kkt_apply_Mu", u, self.block, out)
    def apply_Mu_inv(self, u, out=None): return self._unary("kkt_apply_Mu_inv", u, self.block, out)
    def apply_Mz(self, z, out=None): return self._unary("kkt_apply_Mz", z, self.block, out)
    def apply_Jhat(self, u, out=None): return self._unary("kkt_apply_Jhat", u, self.block, out)
    def apply_JhatT(self, w, out=None): return self._unary("kkt_apply_JhatT", w, self.block, out)

    def forward_solve_window(self, b):
        """In place on a multiple of n_sp (heat_operators.cpp:139-153)."""
        if b.numel() % self.n_sp:
            raise ValueError("forward_solve_window: length not a multiple of n_sp")
        self._call("kkt_forward_solve_window", dptr(b), C.c_int32(b.numel() // self.n_sp))
        return b

    def adjoint_solve_window(self, b):
        if b.numel() % self.n_sp:
            raise ValueError("adjoint_solve_window: length not a multiple of n_sp")
        self._call("kkt_adjoint_solve_window", dptr(b), C.c_int32(b.numel() // self.n_sp))
        return b

    def band_solve(self, b, transpose=False):
        """In place Ahat^{-1} b (or Ahat^{-T} b) per n_sp plane (BandedLU solves)."""
        fn = "kkt_band_solve_transpose" if transpose else "kkt_band_solve"
        self._call(fn, dptr(b), C.c_int32(b.numel() // self.n_sp))
        return b

    # -- KKT level (kkt.hpp:48-65) -------------------------------------------
    def apply_K(self, v, out=None): return self._unary("kkt_apply_K", v, 3 * self.block, out)
    def apply_P_inv(self, r, out=None): return self._unary("kkt_apply_P_inv", r, 3 * self.block, out)

    def apply_P_inv_host(self, r_host: np.ndarray, out_host: Optional[np.ndarray] = None) -> np.ndarray:
        """apply_P_inv from host buffers; H2D/D2H copies inside the call."""
        r_host = np.ascontiguousarray(r_host, dtype=np.float64)
        if r_host.size != 3 * self.block:
            raise ValueError(f"vector length {r_host.size}, expected {3 * self.block}")
        if out_host is None:
            out_host = np.empty_like(r_host)
        self._call("kkt_apply_P_inv_host", r_host.ctypes.data_as(_P), out_host.ctypes.data_as(_P))
        return out_host

    def kkt_residual(self, v, rhs) -> float:
        v = self._dev(v, 3 * self.block)
        rhs = self._dev(rhs, 3 * self.block)
        out = C.c_double()
        self._call("kkt_residual", dptr(v), dptr(rhs), C.byref(out))
        return out.value

    def evaluate_objective(self, u, z, target) -> float:
        """evaluate_objective (kkt.cpp:88-108) with the target sampled at the nodes."""
        u, z, target = (self._dev(a, self.block) for a in (u, z, target))
        out = C.c_double()
        self._call("kkt_evaluate_objective", dptr(u), dptr(z), dptr(target), C.byref(out))
        return out.value

    def model_rhs(self):
        """assemble_rhs(ops, model_initial_condition, model_target).to_kkt() and the
        target samples (kkt.cpp:21-48, model_problem.hpp) for this slab, on the host."""
        b = np.empty(3 * self.block)
        t = np.empty(self.block)
        self._check(lib().kkt_model_rhs(self._h, b.ctypes.data_as(_P), t.ctypes.data_as(_P)))
        return b, t

    # -- Schur level (schur.hpp) ------------------------------------------------
    def apply_shat(self, v, out=None): return self._unary("kkt_apply_shat", v, self.block, out)
    def apply_rasq(self, r, out=None): return self._unary("kkt_apply_rasq", r, self.block, out)
    def schur_apply(self, r, out=None): return self._unary("kkt_schur_apply", r, self.block, out)

    def apply_two_level(self, r, form: str = "multiplicative", out=None):
        from .problems import FORM
        r = self._dev(r, self.block)
        out = self._empty(self.block) if out is None else out
        self._call("kkt_apply_two_level", dptr(r), dptr(out), C.c_int32(FORM[form]))
        return out

    def coarse_dim(self) -> int:
        d = C.c_int32()
        self._check(lib().kkt_coarse_dim(self._h, C.byref(d)))
        return d.value

    def coarse_restrict(self, r):
        r = self._dev(r, self.block)
        c = self._empty(self.coarse_dim())
        self._call("kkt_coarse_restrict", dptr(r), dptr(c))
        return c

    def coarse_solve(self, c):
        c = self._dev(c, self.coarse_dim()).clone()
        self._call("kkt_coarse_solve", dptr(c))
        return c

    def coarse_prolong_add(self, c, out):
        c = self._dev(c, self.coarse_dim())
        self._call("kkt_coarse_prolong_add", dptr(c), dptr(out))
        return out

    def coarse_matrix(self) -> np.ndarray:
        d = self.coarse_dim()
        m = np.empty(d * d)
        self._check(lib().kkt_coarse_matrix(self._h, m.ctypes.data_as(_P)))
        return m.reshape(d, d)

    # -- Krylov (gmres.hpp) ---------------------------------------------------
    def gmres_solve(self, b, x=None) -> GmresOutcome:
        """Right-preconditioned GMRES with apply_K and apply_P_inv (gmres.cpp:21-155)."""
        b = self._dev(b, 3 * self.block)
        x = self._empty(3 * self.block) if x is None else x
        hist = np.empty(self.problem.max_iters)
        res = GmresResult()
        self._call("kkt_gmres_solve", dptr(b), dptr(x), C.byref(res), hist.ctypes.data_as(_P),
                   C.c_int32(hist.size))
        return GmresOutcome(x, bool(res.converged), res.iterations, hist[: res.history_len].copy(),
                            res.true_final_relres)

    def gmres_solve_host(self, b_host: np.ndarray, x_host: Optional[np.ndarray] = None) -> GmresOutcome:
        """Same solve from host buffers; H2D/D2H copies inside the call."""
        b_host = np.ascontiguousarray(b_host, dtype=np.float64)
        if x_host is None:
            x_host = np.empty_like(b_host)
        hist = np.empty(self.problem.max_iters)
        res = GmresResult()
        self._call("kkt_gmres_solve_host", b_host.ctypes.data_as(_P), x_host.ctypes.data_as(_P),
                   C.byref(res), hist.ctypes.data_as(_P), C.c_int32(hist.size))
        return GmresOutcome(x_host, bool(res.converged), res.iterations, hist[: res.history_len].copy(),
                            res.true_final_relres)
