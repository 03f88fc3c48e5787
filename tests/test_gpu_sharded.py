"""GPU: the time-slab sharded path on ONE device.

G virtual ranks run as host threads of this process with an in-process group
(kkt_local_group_create): each owns Nd/G subdomains and its node slab, and the
plane halos, coarse all-gather and dot all-gathers go through the same code
as the NCCL backend, host-synchronised between launches (no kernel waits on
another rank).  The sharded operators must equal the single-rank slabs
bitwise; the sharded solve must match the single-rank solve to 1e-10 with the
same iteration count (dots are summed per rank, then across ranks).
"""
import threading

import numpy as np
import pytest

from paper_2305_04421_b200 import problems as P

pytestmark = pytest.mark.gpu


def run_ranks(p, G, fn):
    import torch
    from paper_2305_04421_b200.solver import HeatKKT, LocalGroup
    grp = LocalGroup(G)
    out, errs = [None] * G, []

    def worker(r):
        try:
            torch.cuda.set_device(0)
            k = HeatKKT(p, mode="fast", rank=r, nranks=G, local_group=grp)
            out[r] = fn(k, r)
            torch.cuda.synchronize()
        except Exception as e:  # surfaced below
            errs.append(e)

    th = [threading.Thread(target=worker, args=(r,)) for r in range(G)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    assert not errs, errs
    return out


def host(t):
    return t.detach().cpu().numpy()


CASES = [
    (P.config(0), 2),
    (P.config(0), 4),
    (P.Problem(Lx=1.0, Ly=2.0, Nx=9, Ny=7, Nt=24, Nd=6, omega=1e-2, coarse_variant="scalar",
               tol=1e-10, restart=8, max_iters=300), 3),
    # nx = 149: the large-grid sweep (sweep_v5.cu), 2 subdomains per rank
    (P.Problem(Lx=1.0, Ly=1.0, Nx=150, Ny=140, Nt=16, Nd=4, nu=1.0, omega=1e-1, coarse_variant="scalar",
               tol=1e-8, restart=20, max_iters=300), 2),
]
IDS = ["c0_G2", "c0_G4", "desk_G3", "v5_G2"]


@pytest.fixture(scope="module")
def single():
    from paper_2305_04421_b200.solver import HeatKKT
    cache = {}

    def get(p):
        key = repr(p)
        if key not in cache:
            cache[key] = HeatKKT(p, mode="fast")
        return cache[key]
    return get


@pytest.mark.parametrize("p,G", CASES, ids=IDS)
def test_sharded_operators_bitwise(p, G, single):
    k1 = single(p)
    v = P.random_vec(3 * p.block, 41)
    want_K = host(k1.apply_K(v))
    want_P = host(k1.apply_P_inv(v))
    s = P.random_vec(p.block, 42)
    want_S = host(k1.apply_shat(s))
    want_J = host(k1.apply_J(s))
    want_JT = host(k1.apply_JT(s))
    want_R = host(k1.apply_rasq(s))

    def fn(k, r):
        return (host(k.apply_K(k.local_slab(v))), host(k.apply_P_inv(k.local_slab(v))),
                host(k.apply_shat(k.local_slab(s))), host(k.apply_J(k.local_slab(s))),
                host(k.apply_JT(k.local_slab(s))), host(k.apply_rasq(k.local_slab(s))),
                k.local_slab(want_K), k.local_slab(want_P), k.local_slab(want_S),
                k.local_slab(want_J), k.local_slab(want_JT), k.local_slab(want_R))

    for r, res in enumerate(run_ranks(p, G, fn)):
        for i, name in enumerate(["K", "P_inv", "shat", "J", "JT", "rasq"]):
            assert np.array_equal(res[i], res[i + 6]), (r, name)


# The v5 case is checked operator by operator only (bitwise, above): on this
# saddle-point system the Krylov recurrence amplifies the rounding of the
# per-rank dot sums ~1e3-fold per iteration (scripts/diag_v5shard.py:
# the v4 grid nx = 119 shows the same 1e-3 history drift by iteration 4), so
# its iteration count is not a parity property of the sweep.
@pytest.mark.parametrize("p,G", CASES[:3], ids=IDS[:3])
def test_sharded_gmres_matches_single_rank(p, G, single):
    b = P.kkt_rhs(0, p) if p.Nx == 32 else P.random_vec(3 * p.block, 43)
    ref = single(p).gmres_solve(b)
    x1 = host(ref.solution)

    def fn(k, r):
        o = k.gmres_solve(k.local_slab(b))
        return o.iterations, host(o.solution), k.local_slab(x1), o.true_final_relres, list(o.residual_history)

    res = run_ranks(p, G, fn)
    for r, (it, xs, want, relres, hist) in enumerate(res):
        assert abs(it - ref.iterations) <= 1, (r, it, ref.iterations)
        # two iterates meeting the stopping test differ by about the attained residual
        tol = max(1e-10, 10 * ref.true_final_relres)
        assert np.linalg.norm(xs - want) <= tol * np.linalg.norm(want), r
        assert hist == res[0][4]  # every rank runs the same scalar recurrence
    assert abs(res[0][3] - ref.true_final_relres) <= 1e-3 * ref.true_final_relres + 1e-14


def test_sharding_rejects_bad_splits():
    from paper_2305_04421_b200.solver import ConfigError, HeatKKT, LocalGroup
    grp = LocalGroup(3)
    with pytest.raises(ConfigError):
        HeatKKT(P.config(0), rank=0, nranks=3, local_group=grp)  # 3 does not divide Nd = 4
    with pytest.raises(NotImplementedError):
        HeatKKT(P.config(0), mode="strict", rank=0, nranks=2, local_group=LocalGroup(2))
