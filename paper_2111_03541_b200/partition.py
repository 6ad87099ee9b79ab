"""Mesh partitioning for the multi-GPU path (no paper design exists).

Owner computes: rank r owns the contiguous control-point range [lo, hi) (for the structured
generators, whose numbering has z slowest, this is a z-slab) and assembles exactly the global rows
of those points, from every element touching them (its own elements plus one ghost layer).  Rows
therefore need no interface exchange; only the residual norms are reduced across ranks.
Host-side index bookkeeping only; all assembly runs in libfem.so.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass
class SubMesh:
    dim: int
    etype: str
    order: int
    coords: np.ndarray  # global coordinates (all points)
    conn: np.ndarray  # int32 [n_loc][E_r], global point ids
    bsets: list
    elem_ids: np.ndarray  # global ids of the local elements

    @property
    def n_nodes(self):
        return int(self.coords.shape[1])

    @property
    def n_elems(self):
        return int(self.conn.shape[1])

    @property
    def n_loc(self):
        return int(self.conn.shape[0])


@dataclass
class Part:
    rank: int
    own: tuple
    mesh: SubMesh


def owned_range(n_nodes: int, nparts: int, rank: int):
    """Balanced contiguous ranges: the first n % P parts get one extra point."""
    base, extra = divmod(n_nodes, nparts)
    lo = rank * base + min(rank, extra)
    hi = lo + base + (1 if rank < extra else 0)
    return lo, hi


def part_for_rank(mesh, nparts: int, rank: int) -> Part:
    lo, hi = owned_range(mesh.coords.shape[1], nparts, rank)
    conn = mesh.conn
    touch = np.zeros(conn.shape[1], dtype=bool)
    for a in range(conn.shape[0]):
        touch |= (conn[a] >= lo) & (conn[a] < hi)
    eids = np.nonzero(touch)[0]
    local_of = np.full(conn.shape[1], -1, dtype=np.int64)
    local_of[eids] = np.arange(eids.size)
    bsets = []
    for be, bf in mesh.bsets:
        keep = touch[be]
        bsets.append((np.ascontiguousarray(local_of[be[keep]], dtype=np.int32),
                      np.ascontiguousarray(bf[keep], dtype=np.int8)))
    sub = SubMesh(mesh.dim, mesh.etype, mesh.order, mesh.coords,
                  np.ascontiguousarray(conn[:, eids], dtype=np.int32), bsets, eids)
    return Part(rank, (lo, hi), sub)


def partition_nodes(mesh, nparts: int):
    return [part_for_rank(mesh, nparts, r) for r in range(nparts)]
