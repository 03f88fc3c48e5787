"""TEST HELPER (not product code): time-slab sharding plan — a host-side mirror of what
kkt_ctx_create computes for a rank (csrc/capi.cu, setup()).

Rank g of G owns the whole subdomains [g*Nd/G, (g+1)*Nd/G) of the reference's
TimePartition (time_partition.cpp:61-86) and therefore the node slab
[g*Nt/G + 1, (g+1)*Nt/G].  Per GMRES iteration the ranks exchange:
  * K (kkt.cpp:50-65): u's last plane -> rank g+1 (its J coupling u_{n-1}),
    w's first plane -> rank g-1 (its J^T coupling w_{n+1});
  * the sweep: r's last plane -> rank g+1 (the shared node s*m of its first
    subdomain, time_partition.cpp:77);
  * the coarse space: each rank restricts its own columns; all-gather;
  * Krylov dots: one partial per rank, all-gathered, summed in rank order.
"""
from __future__ import annotations

import dataclasses

import numpy as np

from paper_2305_04421_b200.problems import Problem


@dataclasses.dataclass(frozen=True)
class Slab:
    rank: int
    nranks: int
    s0: int      # first local subdomain (0-based)
    ndl: int     # local subdomains
    n0: int      # first local node (1-based, global numbering)
    ntl: int     # local nodes
    n_sp: int

    @property
    def block(self) -> int:
        return self.ntl * self.n_sp

    @property
    def prev(self):
        return self.rank - 1 if self.rank > 0 else None

    @property
    def next(self):
        return self.rank + 1 if self.rank + 1 < self.nranks else None


def plan(p: Problem, rank: int, nranks: int) -> Slab:
    if nranks < 1 or not 0 <= rank < nranks:
        raise ValueError("bad rank / nranks")
    if p.Nd % nranks:
        raise ValueError(f"nranks={nranks} must divide Nd={p.Nd}")
    m = p.Nt // p.Nd
    ndl = p.Nd // nranks
    s0 = rank * ndl
    return Slab(rank, nranks, s0, ndl, s0 * m + 1, ndl * m, p.n_sp)


def local_slab(p: Problem, v: np.ndarray, sl: Slab) -> np.ndarray:
    """[u; z; w] (or one block) of a global vector restricted to the slab."""
    B = p.block
    off = (sl.n0 - 1) * p.n_sp
    if v.size == 3 * B:
        return np.concatenate([v[k * B + off:k * B + off + sl.block] for k in range(3)])
    return v[off:off + sl.block].copy()


def assemble(p: Problem, parts) -> np.ndarray:
    """Inverse of local_slab over all ranks' parts (rank order)."""
    k = 3 if parts[0].size == 3 * (parts[0].size // 3) and sum(x.size for x in parts) == 3 * p.block else 1
    if k == 1:
        return np.concatenate(parts)
    blocks = [np.concatenate([x[j * (x.size // 3):(j + 1) * (x.size // 3)] for x in parts]) for j in range(3)]
    return np.concatenate(blocks)
