"""TEST INFRASTRUCTURE ONLY — ctypes bindings of the CPU oracles.

* ``Ref``: the UNMODIFIED reference library (oracle/_ref/libkktdd_ref.so,
  built by oracle/Makefile from /root/reference/proj/src plus
  oracle/ref_driver.cpp).
* ``Orc``: the plain-C restatement (oracle/_build/libkkt_oracle.so, from
  oracle/kkt_oracle.c).

Both expose the same method names, so tests can pin the restatement against
the reference and the CUDA path against either.  Only tests/,
``__graft_entry__.smoke()`` and bench.py's reference / cpu_baseline legs may
import this module; the product package never does.
"""
from __future__ import annotations

import ctypes as C
import os
import sys

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(_HERE))
from paper_2305_04421_b200._abi import GmresResult, RunRecordC, desc_from_problem  # noqa: E402
from paper_2305_04421_b200.problems import Problem  # noqa: E402

REF_SO = os.path.join(_HERE, "_ref", "libkktdd_ref.so")
ORC_SO = os.path.join(_HERE, "_build", "libkkt_oracle.so")

_P = C.c_void_p


class OracleError(RuntimeError):
    def __init__(self, status, msg, index):
        super().__init__(f"status {status}: {msg} (index {index})")
        self.status = status
        self.index = index


def _arr(a):
    return a.ctypes.data_as(_P)


class _Base:
    prefix = ""
    path = ""
    _lib = None

    @classmethod
    def lib(cls):
        if cls._lib is None:
            if not os.path.exists(cls.path):
                raise FileNotFoundError(f"{cls.path} missing: run `make -C oracle`")
            lib = C.CDLL(cls.path)
            p = cls.prefix
            getattr(lib, p + "error").restype = C.c_char_p
            getattr(lib, p + "block").restype = C.c_int64
            getattr(lib, p + "block").argtypes = [_P]
            getattr(lib, p + "destroy").argtypes = [_P]
            cls._lib = lib
        return cls._lib

    def __init__(self, problem: Problem):
        self.problem = problem
        self._desc = desc_from_problem(problem)
        h = _P()
        self._call("create", C.byref(self._desc), C.byref(h))
        self.h = h
        self.block = int(getattr(self.lib(), self.prefix + "block")(self.h))
        self.n_sp = problem.n_sp

    def __del__(self):
        h = getattr(self, "h", None)
        if h:
            getattr(self.lib(), self.prefix + "destroy")(h)
            self.h = None

    def _call(self, name, *args):
        lib = self.lib()
        st = getattr(lib, self.prefix + name)(*args)
        if st != 0:
            msg = getattr(lib, self.prefix + "error")().decode()
            idx = getattr(lib, self.prefix + "error_index")()
            raise OracleError(st, msg, idx)
        return st

    # -- unary block operators --------------------------------------------
    def _unary(self, name, v, n):
        v = np.ascontiguousarray(v, dtype=np.float64)
        assert v.size == n, (v.size, n)
        out = np.empty(n)
        self._call(name, self.h, _arr(v), _arr(out))
        return out

    def apply_K(self, v):
        return self._unary("apply_K", v, 3 * self.block)

    def apply_P_inv(self, r):
        return self._unary("apply_P_inv", r, 3 * self.block)

    def schur_apply(self, r):
        return self._unary("schur_apply", r, self.block)

    def apply_rasq(self, r):
        return self._unary("apply_rasq", r, self.block)

    def apply_shat(self, v):
        return self._unary("apply_shat", v, self.block)

    def apply_two_level(self, r, form=1):
        r = np.ascontiguousarray(r, dtype=np.float64)
        out = np.empty(self.block)
        self._call("apply_two_level", self.h, _arr(r), _arr(out), C.c_int(form))
        return out

    def op(self, name, v):
        """apply_J / JT / L / LT / Mu / Mu_inv / Mz / Jhat / JhatT."""
        return self._unary("apply_" + name, v, self.block)

    def forward_solve_window(self, b):
        b = np.array(b, dtype=np.float64, copy=True)
        self._call("forward_solve_window", self.h, _arr(b), C.c_int(b.size // self.n_sp))
        return b

    def adjoint_solve_window(self, b):
        b = np.array(b, dtype=np.float64, copy=True)
        self._call("adjoint_solve_window", self.h, _arr(b), C.c_int(b.size // self.n_sp))
        return b

    def band_solve(self, b, transpose=False):
        b = np.array(b, dtype=np.float64, copy=True)
        self._call("band_solve", self.h, _arr(b), C.c_int(b.size // self.n_sp), C.c_int(int(transpose)))
        return b

    def ahat_factor(self):
        lib = self.lib()
        kl, ku = C.c_int(), C.c_int()
        g = C.c_double()
        self._call("ahat_factor", self.h, C.byref(kl), C.byref(ku), None, None, C.byref(g))
        n = self.n_sp
        ab = np.empty(n * (kl.value + ku.value + 1))
        piv = np.empty(n, dtype=np.int32)
        self._call("ahat_factor", self.h, C.byref(kl), C.byref(ku), _arr(ab), _arr(piv), C.byref(g))
        return kl.value, ku.value, ab, piv, g.value

    # -- coarse space -----------------------------------------------------
    def coarse_dim(self):
        return int(getattr(self.lib(), self.prefix + "coarse_dim")(self.h))

    def coarse_restrict(self, r):
        r = np.ascontiguousarray(r, dtype=np.float64)
        c = np.empty(self.coarse_dim())
        self._call("coarse_restrict", self.h, _arr(r), _arr(c))
        return c

    def coarse_solve(self, c):
        c = np.array(c, dtype=np.float64, copy=True)
        self._call("coarse_solve", self.h, _arr(c))
        return c

    def coarse_prolong_add(self, c, out):
        c = np.ascontiguousarray(c, dtype=np.float64)
        out = np.array(out, dtype=np.float64, copy=True)
        self._call("coarse_prolong_add", self.h, _arr(c), _arr(out))
        return out

    def coarse_matrix(self):
        d = self.coarse_dim()
        m = np.empty(d * d)
        self._call("coarse_matrix", self.h, _arr(m))
        return m.reshape(d, d)

    # -- Krylov -----------------------------------------------------------
    def gmres_solve(self, b):
        b = np.ascontiguousarray(b, dtype=np.float64)
        x = np.empty_like(b)
        hist = np.empty(self.problem.max_iters)
        res = GmresResult()
        self._call("gmres_solve", self.h, _arr(b), _arr(x), C.byref(res), _arr(hist),
                   C.c_int(hist.size))
        return dict(x=x, converged=bool(res.converged), iterations=res.iterations,
                    true_final_relres=res.true_final_relres, history=hist[: res.history_len].copy())

    def kkt_residual(self, v, rhs):
        out = C.c_double()
        self._call("kkt_residual", self.h, _arr(np.ascontiguousarray(v)), _arr(np.ascontiguousarray(rhs)),
                   C.byref(out))
        return out.value

    @classmethod
    def gmres_dense(cls, A, b, M=None, tol=1e-6, max_iters=420, restart=None):
        A = np.ascontiguousarray(A, dtype=np.float64)
        n = A.shape[0]
        b = np.ascontiguousarray(b, dtype=np.float64)
        x = np.empty(n)
        hist = np.empty(max_iters)
        res = GmresResult()
        Mp = _arr(np.ascontiguousarray(M, dtype=np.float64)) if M is not None else None
        lib = cls.lib()
        st = getattr(lib, cls.prefix + "gmres_dense")(
            C.c_int(n), _arr(A), Mp, _arr(b), C.c_double(tol), C.c_int(max_iters),
            C.c_int(restart or 0), _arr(x), C.byref(res), _arr(hist), C.c_int(max_iters))
        if st != 0:
            raise OracleError(st, getattr(lib, cls.prefix + "error")().decode(),
                              getattr(lib, cls.prefix + "error_index")())
        return dict(x=x, converged=bool(res.converged), iterations=res.iterations,
                    true_final_relres=res.true_final_relres, history=hist[: res.history_len].copy())


class Ref(_Base):
    """The compiled reference (oracle/_ref/libkktdd_ref.so)."""
    prefix = "ref_"
    path = REF_SO
    _lib = None

    # -- the f1 record (experiments.cpp:33-69, :179-208) ------------------
    @classmethod
    def run_single(cls, problem: Problem, want_x=False):
        """The reference's own run_single(cfg): (record dict, JSON text, x or None)."""
        desc = desc_from_problem(problem)
        rec = RunRecordC()
        B = problem.block
        x = np.empty(3 * B) if want_x else None
        buf = C.create_string_buffer(1 << 14)
        lib = cls.lib()
        st = lib.ref_run_single(C.byref(desc), C.byref(rec), _arr(x) if want_x else None, buf,
                                C.c_int(len(buf)))
        if st != 0:
            raise OracleError(st, lib.ref_error().decode(), lib.ref_error_index())
        d = {k: getattr(rec, k) for k, _ in RunRecordC._fields_}
        d["converged"] = bool(d["converged"])
        return d, buf.value.decode(), x

    # -- the f3 sweeps (experiments.cpp:97-177) ----------------------------
    @classmethod
    def sweep_csv(cls, base: Problem, kind: str, omegas, preconds, steps=0, nts=(), nt=0, nd=0):
        """to_csv(weak_scaling_sweep(...)) (kind "weak") or to_csv(omega_sweep(...))
        (kind "omega") of the reference itself."""
        from paper_2305_04421_b200.problems import PRECOND
        desc = desc_from_problem(base)
        ia = (C.c_int * max(1, len(nts)))(*nts)
        oa = (C.c_double * max(1, len(omegas)))(*omegas)
        pa = (C.c_int * max(1, len(preconds)))(*[PRECOND[p] for p in preconds])
        buf = C.create_string_buffer(1 << 16)
        lib = cls.lib()
        st = lib.ref_sweep_csv(0 if kind == "weak" else 1, C.byref(desc), steps, nt, nd, ia, len(nts), oa,
                               len(omegas), pa, len(preconds), buf, C.c_int(len(buf)))
        if st != 0:
            raise OracleError(st, lib.ref_error().decode(), lib.ref_error_index())
        return buf.value.decode()

    def model_rhs(self):
        """(b, target samples) of assemble_rhs(ops, model_initial_condition, model_target)."""
        b = np.empty(3 * self.block)
        t = np.empty(self.block)
        self._call("model_rhs", self.h, _arr(b), _arr(t))
        return b, t

    def evaluate_objective(self, u, z):
        out = C.c_double()
        self._call("evaluate_objective", self.h, _arr(np.ascontiguousarray(u, dtype=np.float64)),
                   _arr(np.ascontiguousarray(z, dtype=np.float64)), C.byref(out))
        return out.value

    def zero_control_objective(self):
        out = C.c_double()
        self._call("zero_control_objective", self.h, C.byref(out))
        return out.value


class Orc(_Base):
    """The plain-C restatement (oracle/_build/libkkt_oracle.so)."""
    prefix = "orc_"
    path = ORC_SO
    _lib = None


def available(kind: str) -> bool:
    return os.path.exists(REF_SO if kind == "ref" else ORC_SO)
