"""Mesh partitioning for the multi-GPU path (the paper names distributed assembly as future
work).  Host-side index bookkeeping only: all assembly runs in libfem.so.

Owner computes.  The control points are split into `nparts` spatially compact parts by recursive coordinate
bisection (RCB: cut the longest extent of the point cloud at the count-weighted median, recursively), so a
part is a box-like region whatever the numbering (the perturbed variants permute node and element ids at
random, which a contiguous id range would scatter over the whole domain).  Rank r assembles exactly the
rows of its own points, from every element touching them (its interior elements plus one ghost layer), so
rows need no interface exchange; only the residual norms are reduced across ranks.

Local numbering.  A rank holds only its own points and the halo points of its elements: local ids are the
owned points in increasing global id, then the halo points in increasing global id.  The local mesh is
therefore self-contained (coordinates, connectivity, state and rows all scale as 1/N), the rank's CSR uses
the paper's κ-major numbering g(κ, α) = κ·n_local + α of the relabelled points (B-3), and
`node_ids` maps local point ids back to the global ones (a permutation restricted to the part).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass
class SubMesh:
    dim: int
    etype: str
    order: int
    coords: np.ndarray  # float64 [dim][n_local]: owned points, then halo points
    conn: np.ndarray    # int32 [n_loc][E_r], local point ids
    bsets: list
    elem_ids: np.ndarray  # global ids of the local elements (ascending)

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
    own: tuple            # (0, n_owned): owned points are local ids [0, n_owned)
    mesh: SubMesh
    node_ids: np.ndarray  # int64 [n_local]: global id of each local point

    @property
    def n_owned(self):
        return self.own[1] - self.own[0]

    def local_state(self, state):
        """The rank's slice of a global state array [levels][κ̂][N] (owned + halo points, local order)."""
        return np.ascontiguousarray(state[..., self.node_ids])

    def global_rows(self, kappa_hat: int, n_global: int):
        """Global row id g(κ, α) = κ·N + α of every local row κ·n_owned + i."""
        own = self.node_ids[: self.n_owned]
        return (np.arange(kappa_hat)[:, None] * n_global + own[None, :]).ravel()

    def global_cols(self, local_cols, n_global: int):
        """Map local column ids κ·n_local + j to global κ·N + node_ids[j]."""
        nl = len(self.node_ids)
        k, j = np.divmod(np.asarray(local_cols, dtype=np.int64), nl)
        return k * n_global + self.node_ids[j]


def rcb_parts(coords: np.ndarray, nparts: int) -> np.ndarray:
    """Recursive coordinate bisection of the points: part id (int32) per point, part sizes within one point
    of N·(share of the part).  Each cut splits the longest extent of the current point set (ties: the
    highest axis, so a cube splits into z-slabs first) at the position that gives the two sides point
    counts proportional to the numbers of parts they receive.  Ties in the coordinate are broken by the
    global id, so the result is deterministic."""
    n = coords.shape[1]
    part = np.zeros(n, dtype=np.int32)

    def split(idx: np.ndarray, p0: int, np_: int):
        if np_ == 1 or idx.size == 0:
            part[idx] = p0
            return
        x = coords[:, idx]
        ext = x.max(axis=1) - x.min(axis=1)
        axis = int(np.flatnonzero(ext >= ext.max() * (1 - 1e-12))[-1])
        nl = np_ // 2
        k = (idx.size * nl) // np_
        order = np.lexsort((idx, x[axis]))
        split(idx[order[:k]], p0, nl)
        split(idx[order[k:]], p0 + nl, np_ - nl)

    split(np.arange(n, dtype=np.int64), 0, nparts)
    return part


def part_for_rank(mesh, nparts: int, rank: int, parts: np.ndarray | None = None) -> Part:
    """The rank's local mesh (owned + halo points, elements touching an owned point) in local numbering."""
    if parts is None:
        parts = rcb_parts(mesh.coords, nparts)
    conn = mesh.conn
    own_mask = parts == rank
    touch = own_mask[conn].any(axis=0)
    eids = np.nonzero(touch)[0]
    owned = np.nonzero(own_mask)[0]
    used = np.unique(conn[:, eids])
    halo = used[~own_mask[used]]
    node_ids = np.concatenate([owned, halo]).astype(np.int64)
    local_of = np.full(mesh.coords.shape[1], -1, dtype=np.int64)
    local_of[node_ids] = np.arange(node_ids.size)
    elem_local = np.full(conn.shape[1], -1, dtype=np.int64)
    elem_local[eids] = np.arange(eids.size)
    bsets = []
    for be, bf in mesh.bsets:
        keep = touch[be]
        bsets.append((np.ascontiguousarray(elem_local[be[keep]], dtype=np.int32),
                      np.ascontiguousarray(bf[keep], dtype=np.int8)))
    sub = SubMesh(mesh.dim, mesh.etype, mesh.order, np.ascontiguousarray(mesh.coords[:, node_ids]),
                  np.ascontiguousarray(local_of[conn[:, eids]], dtype=np.int32), bsets, eids)
    return Part(rank, (0, int(owned.size)), sub, node_ids)


def partition_nodes(mesh, nparts: int):
    parts = rcb_parts(mesh.coords, nparts)
    return [part_for_rank(mesh, nparts, r, parts) for r in range(nparts)]
