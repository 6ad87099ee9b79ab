"""Seeded structured / perturbed-unstructured mesh generators (SURVEY §8(d) "Synthetic inputs").

Conventions (readings L7/L8/L19):
  * coords: float64 SoA, shape (dim, N); conn: int32 SoA, shape (n_loc, E) (VTK local node order).
  * tri  (P1): (0,0),(1,0),(0,1) reference vertices, counter-clockwise.
  * tet  (P1): v0..v3; (P2): + edge nodes (0,1),(1,2),(0,2),(0,3),(1,3),(2,3)  [VTK quadratic tetra].
  * hex  (Q1): (---),(+--),(++-),(-+-),(--+),(+-+),(+++),(-++)  [VTK hexahedron].
  * hex (Q2, 27 nodes) / hexs (serendipity, 20 nodes), reading L28: the 8 corners as Q1, the 12 edge
    midpoints of VTK's quadratic hexahedron (0,1),(1,2),(2,3),(3,0),(4,5),(5,6),(6,7),(7,4),(0,4),(1,5),
    (2,6),(3,7), then (27 only) the face centres in facet order x-,x+,y-,y+,z-,z+ and the centre.
  * Facet k: tri edge (k, k+1 mod 3); tet face opposite vertex k; hex faces
    x-(0,4,7,3) x+(1,2,6,5) y-(0,1,5,4) y+(3,7,6,2) z-(0,3,2,1) z+(4,5,6,7).
The facet vertex lists below are only used to *select* boundary facets lying on a plane; the
facet integration itself is done independently by each implementation.
"""
from __future__ import annotations

import itertools
from dataclasses import dataclass, field

import numpy as np

FACET_VERTS = {
    "tri": [(0, 1), (1, 2), (2, 0)],
    "tet": [(1, 2, 3), (0, 2, 3), (0, 1, 3), (0, 1, 2)],
    "hex": [(0, 4, 7, 3), (1, 2, 6, 5), (0, 1, 5, 4), (3, 7, 6, 2), (0, 3, 2, 1), (4, 5, 6, 7)],
}
FACET_VERTS["hexs"] = FACET_VERTS["hex"]

_HEX_CORNERS = [(-1, -1, -1), (1, -1, -1), (1, 1, -1), (-1, 1, -1), (-1, -1, 1), (1, -1, 1), (1, 1, 1), (-1, 1, 1)]
_HEX_EDGES = [(0, 1), (1, 2), (2, 3), (3, 0), (4, 5), (5, 6), (6, 7), (7, 4), (0, 4), (1, 5), (2, 6), (3, 7)]


def quad_cube_ref_nodes(n_loc: int):
    """Reference coordinates r_a ∈ {-1,0,1}³ of the 20/27 nodes of a quadratic cube (reading L28)."""
    r = [tuple(c) for c in _HEX_CORNERS]
    for a, b in _HEX_EDGES:
        r.append(tuple((_HEX_CORNERS[a][d] + _HEX_CORNERS[b][d]) // 2 for d in range(3)))
    if n_loc == 27:
        for f in range(6):
            c = [0, 0, 0]
            c[f // 2] = 1 if f & 1 else -1
            r.append(tuple(c))
        r.append((0, 0, 0))
    return np.array(r[:n_loc], dtype=np.int64)


@dataclass
class Mesh:
    dim: int
    etype: str  # "tri" | "tet" | "hex"
    order: int
    coords: np.ndarray  # (dim, N) float64
    conn: np.ndarray  # (n_loc, E) int32
    bsets: list = field(default_factory=list)  # list of (elem int32[], facet int8[])
    bset_names: list = field(default_factory=list)

    @property
    def n_nodes(self) -> int:
        return int(self.coords.shape[1])

    @property
    def n_elems(self) -> int:
        return int(self.conn.shape[1])

    @property
    def n_loc(self) -> int:
        return int(self.conn.shape[0])


def _soa(a, dtype):
    return np.ascontiguousarray(np.asarray(a, dtype=dtype))


def tri_square(n: int) -> Mesh:
    """Unit square, n x n squares, each split into two CCW P1 triangles (reading L19):
    (v_ij, v_{i+1,j}, v_{i+1,j+1}) and (v_ij, v_{i+1,j+1}, v_{i,j+1})."""
    i, j = np.meshgrid(np.arange(n + 1), np.arange(n + 1), indexing="xy")
    coords = np.stack([i.ravel() / n, j.ravel() / n])
    nid = lambda a, b: a + (n + 1) * b  # noqa: E731
    si, sj = np.meshgrid(np.arange(n), np.arange(n), indexing="xy")
    si, sj = si.ravel(), sj.ravel()
    v00, v10, v11, v01 = nid(si, sj), nid(si + 1, sj), nid(si + 1, sj + 1), nid(si, sj + 1)
    ta = np.stack([v00, v10, v11])
    tb = np.stack([v00, v11, v01])
    conn = np.empty((3, 2 * n * n), dtype=np.int64)
    conn[:, 0::2] = ta
    conn[:, 1::2] = tb
    return Mesh(2, "tri", 1, _soa(coords, np.float64), _soa(conn, np.int32))


def hex_box(nx: int, ny: int, nz: int, lx=1.0, ly=1.0, lz=1.0) -> Mesh:
    """Structured Q1 hex box [0,lx]x[0,ly]x[0,lz]; node id = i + (nx+1)(j + (ny+1)k),
    element id = i + nx(j + ny k), VTK local order."""
    I, J, K = np.meshgrid(np.arange(nx + 1), np.arange(ny + 1), np.arange(nz + 1), indexing="ij")
    I, J, K = (a.transpose(2, 1, 0).ravel() for a in (I, J, K))  # x fastest
    coords = np.stack([I * (lx / nx), J * (ly / ny), K * (lz / nz)])
    ei, ej, ek = np.meshgrid(np.arange(nx), np.arange(ny), np.arange(nz), indexing="ij")
    ei, ej, ek = (a.transpose(2, 1, 0).ravel() for a in (ei, ej, ek))
    nid = lambda a, b, c: a + (nx + 1) * (b + (ny + 1) * c)  # noqa: E731
    corners = [(0, 0, 0), (1, 0, 0), (1, 1, 0), (0, 1, 0), (0, 0, 1), (1, 0, 1), (1, 1, 1), (0, 1, 1)]
    conn = np.stack([nid(ei + a, ej + b, ek + c) for (a, b, c) in corners])
    return Mesh(3, "hex", 1, _soa(coords, np.float64), _soa(conn, np.int32))


_P2_EDGES = [(0, 1), (1, 2), (0, 2), (0, 3), (1, 3), (2, 3)]


def hex_box_quadratic(nx: int, ny: int, nz: int, lx=1.0, ly=1.0, lz=1.0, serendipity: bool = False) -> Mesh:
    """Structured box of quadratic cubes (NEXT-2): 27-node Lagrange ("hex", order 2) or 20-node serendipity
    ("hexs", order 2).  Nodes are the points of the doubled lattice (id by x fastest) — all of them for the
    27-node cube; for serendipity only the points with at most one odd lattice coordinate (vertices and edge
    midpoints), renumbered in the same order."""
    mx, my, mz = 2 * nx, 2 * ny, 2 * nz
    I, J, K = np.meshgrid(np.arange(mx + 1), np.arange(my + 1), np.arange(mz + 1), indexing="ij")
    I, J, K = (a.transpose(2, 1, 0).ravel() for a in (I, J, K))
    keep = ((I & 1) + (J & 1) + (K & 1) <= 1) if serendipity else np.ones(I.shape, bool)
    new_id = np.full(I.shape, -1, dtype=np.int64)
    new_id[keep] = np.arange(int(keep.sum()))
    coords = np.stack([I[keep] * (lx / mx), J[keep] * (ly / my), K[keep] * (lz / mz)])
    ei, ej, ek = np.meshgrid(np.arange(nx), np.arange(ny), np.arange(nz), indexing="ij")
    ei, ej, ek = (a.transpose(2, 1, 0).ravel() for a in (ei, ej, ek))
    ref = quad_cube_ref_nodes(20 if serendipity else 27)
    lid = lambda a, b, c: a + (mx + 1) * (b + (my + 1) * c)  # noqa: E731
    conn = np.stack([new_id[lid(2 * ei + 1 + r[0], 2 * ej + 1 + r[1], 2 * ek + 1 + r[2])] for r in ref])
    assert (conn >= 0).all()
    return Mesh(3, "hexs" if serendipity else "hex", 2, _soa(coords, np.float64), _soa(conn, np.int32))


def tet_box(nx: int, ny: int, nz: int, lx=1.0, ly=1.0, lz=1.0, order: int = 1) -> Mesh:
    """Kuhn triangulation: 6 tets per cube, tet p = (c, c+e_p0, c+e_p0+e_p1, c+(1,1,1)) for the
    axis permutations p in itertools order; two vertices swapped where needed so det J > 0.
    P1 nodes: lattice id = i + (nx+1)(j + (ny+1)k).  P2 nodes: the doubled lattice
    (id = I + (2nx+1)(J + (2ny+1)K)) = vertices, edge midpoints, face and cube centres."""
    s = 2 if order == 2 else 1
    mx, my, mz = s * nx, s * ny, s * nz
    I, J, K = np.meshgrid(np.arange(mx + 1), np.arange(my + 1), np.arange(mz + 1), indexing="ij")
    I, J, K = (a.transpose(2, 1, 0).ravel() for a in (I, J, K))
    coords = np.stack([I * (lx / mx), J * (ly / my), K * (lz / mz)])
    ei, ej, ek = np.meshgrid(np.arange(nx), np.arange(ny), np.arange(nz), indexing="ij")
    ei, ej, ek = (a.transpose(2, 1, 0).ravel() for a in (ei, ej, ek))
    base = np.stack([ei, ej, ek])  # (3, C)
    tets = []
    for p in itertools.permutations(range(3)):
        e0 = np.zeros(3, int)
        e1 = np.zeros(3, int)
        e1[p[0]] = 1
        e2 = e1.copy()
        e2[p[1]] = 1
        e3 = np.ones(3, int)
        verts = [e0, e1, e2, e3]
        d = np.linalg.det(np.stack([e1 - e0, e2 - e0, e3 - e0]).astype(float))
        if d < 0:
            verts[1], verts[2] = verts[2], verts[1]
        tets.append(verts)
    n_c = base.shape[1]
    n_loc = 4 if order == 1 else 10
    conn = np.empty((n_loc, 6 * n_c), dtype=np.int64)

    def lid(pt):  # pt: (3, C) doubled-lattice coordinates
        return pt[0] + (mx + 1) * (pt[1] + (my + 1) * pt[2])

    for t, verts in enumerate(tets):
        vpts = [s * base + s * np.asarray(v)[:, None] for v in verts]
        for a in range(4):
            conn[a, t::6] = lid(vpts[a])
        if order == 2:
            for k, (a, b) in enumerate(_P2_EDGES):
                conn[4 + k, t::6] = lid((vpts[a] + vpts[b]) // 2)
    return Mesh(3, "tet", order, _soa(coords, np.float64), _soa(conn, np.int32))


def facets_on_plane(mesh: Mesh, axis: int, value: float, tol: float = 1e-12):
    """(elem int32[], facet int8[]) of all element facets whose vertices lie on x_axis == value."""
    verts = FACET_VERTS[mesh.etype]
    x = mesh.coords[axis]
    elems, facs = [], []
    for k, fv in enumerate(verts):
        on = np.ones(mesh.n_elems, dtype=bool)
        for a in fv:
            on &= np.abs(x[mesh.conn[a]] - value) <= tol
        e = np.nonzero(on)[0]
        elems.append(e)
        facs.append(np.full(e.shape, k))
    e = np.concatenate(elems)
    f = np.concatenate(facs)
    order = np.lexsort((f, e))
    return _soa(e[order], np.int32), _soa(f[order], np.int8)


def _boundary_node_mask(mesh: Mesh, lo, hi):
    m = np.zeros(mesh.n_nodes, dtype=bool)
    for d in range(mesh.dim):
        m |= np.abs(mesh.coords[d] - lo[d]) <= 1e-12
        m |= np.abs(mesh.coords[d] - hi[d]) <= 1e-12
    return m


def perturb_and_permute(mesh: Mesh, rng: np.random.Generator, h, amp: float = 0.2) -> Mesh:
    """Perturbed-unstructured variant: interior *vertices* get a uniform jitter of
    +-amp*h per coordinate (boundary nodes fixed so boundary planes/normals are exact); P2 edge
    nodes are re-placed at the midpoint of their (perturbed) edge vertices; then a seeded random
    permutation of the node numbering and of the element order; boundary sets are remapped."""
    coords = mesh.coords.copy()
    lo, hi = coords.min(axis=1), coords.max(axis=1)
    h = np.broadcast_to(np.asarray(h, dtype=np.float64), (mesh.dim,))
    bnd = _boundary_node_mask(mesh, lo, hi)
    nv = 3 if mesh.etype == "tri" else (4 if mesh.etype == "tet" else 8)
    quad_cube = mesh.etype in ("hex", "hexs") and mesh.order == 2
    vert_ids = np.unique(mesh.conn[:nv])
    interior = vert_ids[~bnd[vert_ids]]
    jit = rng.uniform(-1.0, 1.0, size=(mesh.dim, interior.size)) * (amp * h)[:, None]
    coords[:, interior] += jit
    if mesh.etype == "tet" and mesh.order == 2:
        for k, (a, b) in enumerate(_P2_EDGES):
            mid = mesh.conn[4 + k]
            coords[:, mid] = 0.5 * (coords[:, mesh.conn[a]] + coords[:, mesh.conn[b]])
    if quad_cube:  # non-vertex nodes on the trilinear map of the (perturbed) corners
        ref = quad_cube_ref_nodes(mesh.n_loc)
        for a in range(8, mesh.n_loc):
            w = [np.prod([(1 + ref[a][d] * _HEX_CORNERS[c][d]) / 2 for d in range(3)]) for c in range(8)]
            coords[:, mesh.conn[a]] = sum(w[c] * coords[:, mesh.conn[c]] for c in range(8))
    N, E = mesh.n_nodes, mesh.n_elems
    new_of_old = rng.permutation(N)
    c2 = np.empty_like(coords)
    c2[:, new_of_old] = coords
    conn = new_of_old[mesh.conn]
    old_of_new_e = rng.permutation(E)
    conn = conn[:, old_of_new_e]
    new_of_old_e = np.empty(E, dtype=np.int64)
    new_of_old_e[old_of_new_e] = np.arange(E)
    bsets = []
    for (be, bf) in mesh.bsets:
        ne = new_of_old_e[be]
        order = np.lexsort((bf, ne))
        bsets.append((_soa(ne[order], np.int32), _soa(bf[order], np.int8)))
    return Mesh(mesh.dim, mesh.etype, mesh.order, _soa(c2, np.float64), _soa(conn, np.int32),
                bsets, list(mesh.bset_names))
