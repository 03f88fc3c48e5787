"""CPU, world_size 2 over gloo: the time-slab sharding plan and its exchanges.

Two processes each own half of the subdomains (tests/sharding_plan.py,
the host mirror of the CUDA context's slab logic) and exchange exactly what the
device path exchanges: the u/w halo planes of K, the r plane of the sweep's
shared node, the per-rank coarse columns (all-gather) and one partial per dot
(all-gather, rank-ordered sum).  Each rank's slab results are checked against
the single-process oracle restricted to the slab.
"""
import os
import socket

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _stencil_slab(p, x, prev, nxt, lower):
    """The reference's band row order (-nx, -1, 0, +1, +nx; linalg.cpp:45-54)
    plus the time coupling, on a slab with neighbour planes `prev` / `nxt`."""
    nx, ny, nsp = p.nx_int, p.ny_int, p.n_sp
    cx = p.dt * p.nu / (p.dx * p.dx)
    cy = p.dt * p.nu / (p.dy * p.dy)
    diag = 1.0 + 2.0 * cx + 2.0 * cy
    X = x.reshape(-1, ny, nx)
    acc = np.zeros_like(X)
    acc[:, 1:, :] += (-cy) * X[:, :-1, :]
    acc[:, :, 1:] += (-cx) * X[:, :, :-1]
    acc += diag * X
    acc[:, :, :-1] += (-cx) * X[:, :, 1:]
    acc[:, :-1, :] += (-cy) * X[:, 1:, :]
    out = acc.reshape(-1, nsp)
    Xn = x.reshape(-1, nsp)
    if lower:
        out[1:] -= Xn[:-1]
        if prev is not None:
            out[0] -= prev
    else:
        out[:-1] -= Xn[1:]
        if nxt is not None:
            out[-1] -= nxt
    return out.reshape(-1)


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    import sys
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from oracle.bindings import Orc
    from paper_2305_04421_b200 import problems as P
    import sharding_plan as S

    try:
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                                world_size=world)
        p = P.Problem(Lx=1.0, Ly=2.0, Nx=9, Ny=7, Nt=24, Nd=6, omega=1e-2, coarse_variant="scalar")
        sl = S.plan(p, rank, world)
        nsp, B = p.n_sp, p.block
        o = Orc(p)
        v = P.random_vec(3 * B, 51)
        mine = S.local_slab(p, v, sl)
        L = sl.block
        u, z, w = mine[:L], mine[L:2 * L], mine[2 * L:]

        def halo(to_prev, to_next):
            """send to_prev -> rank-1, to_next -> rank+1; receive (from_prev, from_next)"""
            reqs, fp, fn = [], None, None
            if sl.prev is not None:
                fp = torch.empty(nsp, dtype=torch.float64)
                reqs.append(dist.isend(torch.from_numpy(np.ascontiguousarray(to_prev)), sl.prev))
                reqs.append(dist.irecv(fp, sl.prev))
            if sl.next is not None:
                fn = torch.empty(nsp, dtype=torch.float64)
                reqs.append(dist.isend(torch.from_numpy(np.ascontiguousarray(to_next)), sl.next))
                reqs.append(dist.irecv(fn, sl.next))
            for r in reqs:
                r.wait()
            return (fp.numpy() if fp is not None else None), (fn.numpy() if fn is not None else None)

        # ---- K on the slab (kkt.cpp:50-65): u plane forward, w plane backward
        u_prev, _ = halo(np.zeros(nsp), u[(sl.ntl - 1) * nsp:])   # rank+1 gets our last u plane
        _, w_next = halo(w[:nsp], np.zeros(nsp))                   # rank-1 gets our first w plane
        ms, dt = p.mass_scale, p.dt
        ou = _stencil_slab(p, w, None, w_next, lower=False) + ms * u
        oz = (p.omega * ms) * z - dt * w
        ow = _stencil_slab(p, u, u_prev, None, lower=True) - dt * z
        got = np.concatenate([ou, oz, ow])
        want = S.local_slab(p, o.apply_K(v), sl)
        ok_K = bool(np.array_equal(got, want))

        # ---- the sweep's shared node: r's last plane travels to rank+1
        r = P.random_vec(B, 52)
        rl = S.local_slab(p, r, sl)
        r_prev, _ = halo(np.zeros(nsp), rl[(sl.ntl - 1) * nsp:])
        ok_shared = True
        if sl.prev is not None:
            node = sl.s0 * (p.Nt // p.Nd)          # shared node s*m of the first local subdomain
            assert node == sl.n0 - 1
            ok_shared = bool(np.array_equal(r_prev, r[(node - 1) * nsp:node * nsp]))

        # ---- coarse restriction: own columns, all-gather, rank-ordered sum
        m = p.Nt // p.Nd
        cols = []
        for s in range(p.Nd):
            ns = (s + 1) * m - (1 if s == 0 else s * m) + 1
            skip = 0 if s == 0 else 1
            lin = [-1.0 + 2.0 * k / (ns - 1) for k in range(ns)][skip:]
            cols.append((s, [1.0] * (ns - skip)))
            cols.append((s, lin))
        c_local = np.zeros(len(cols))
        for ci, (s, phi) in enumerate(cols):
            if sl.s0 <= s < sl.s0 + sl.ndl:
                first = 1 if s == 0 else s * m + 1
                acc = 0.0
                for k, ph in enumerate(phi):
                    n = first + k
                    ns_val = rl[(n - sl.n0) * nsp:(n - sl.n0 + 1) * nsp].sum()
                    acc += ph * ns_val
                c_local[ci] = acc
        gathered = [torch.empty(len(cols), dtype=torch.float64) for _ in range(world)]
        dist.all_gather(gathered, torch.from_numpy(c_local))
        c_all = sum(g.numpy() for g in gathered)
        c_ref = o.coarse_restrict(r)
        ok_coarse = bool(np.allclose(c_all, c_ref, rtol=1e-12, atol=1e-12 * np.abs(c_ref).max()))

        # ---- Krylov dot: one partial per rank, all-gathered, summed in rank order
        a = P.random_vec(3 * B, 53)
        part = float(np.dot(S.local_slab(p, a, sl), mine))
        parts = [torch.empty(1, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(parts, torch.tensor([part], dtype=torch.float64))
        total = sum(float(x.item()) for x in parts)
        ok_dot = abs(total - float(np.dot(a, v))) <= 1e-12 * abs(float(np.dot(np.abs(a), np.abs(v))))

        q.put((rank, ok_K, ok_shared, ok_coarse, ok_dot, sl.n0, sl.ntl))
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put((rank, repr(e)))


def test_two_rank_slab_exchanges_match_single_process():
    import torch.multiprocessing as mp
    from oracle import bindings
    if not bindings.available("orc"):
        import subprocess
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "oracle"], check=True)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=300) for _ in procs]
    for pr in procs:
        pr.join(timeout=60)
    res = sorted(res)
    for r in res:
        assert len(r) == 7, r
        rank, ok_K, ok_shared, ok_coarse, ok_dot, n0, ntl = r
        assert ok_K, f"rank {rank}: slab K differs from the oracle"
        assert ok_shared, f"rank {rank}: shared-node halo wrong"
        assert ok_coarse, f"rank {rank}: coarse all-gather wrong"
        assert ok_dot, f"rank {rank}: dot all-gather wrong"
    assert [x[5] for x in res] == [1, 13] and [x[6] for x in res] == [12, 12]


def test_plan_matches_partition():
    from paper_2305_04421_b200 import problems as P
    import sharding_plan as S
    p = P.config(1)
    slabs = [S.plan(p, g, 8) for g in range(8)]
    assert [s.n0 for s in slabs] == [1 + 64 * g for g in range(8)]
    assert sum(s.ntl for s in slabs) == p.Nt and all(s.ndl == 2 for s in slabs)
    with pytest.raises(ValueError):
        S.plan(P.config(0), 0, 3)
    v = np.arange(3 * p.block, dtype=np.float64)
    parts = [S.local_slab(p, v, s) for s in slabs]
    assert np.array_equal(S.assemble(p, parts), v)
