"""Shared test helpers (no method arithmetic: meshes/problems/tolerance metrics only)."""
from __future__ import annotations

import json
import os
from fractions import Fraction

import numpy as np

from fem_inputs.configs import Problem, Term, TimeScheme
from fem_inputs.meshgen import Mesh

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def golden(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


def frac(x):
    return float(Fraction(x))


REF_TRI = np.array([[0.0, 1.0, 0.0], [0.0, 0.0, 1.0]])
REF_TET = np.array([[0.0, 1.0, 0.0, 0.0], [0.0, 0.0, 1.0, 0.0], [0.0, 0.0, 0.0, 1.0]])
HEX_CORNERS = np.array([(0, 0, 0), (1, 0, 0), (1, 1, 0), (0, 1, 0), (0, 0, 1), (1, 0, 1), (1, 1, 1),
                        (0, 1, 1)], dtype=float).T
P2_EDGES = [(0, 1), (1, 2), (0, 2), (0, 3), (1, 3), (2, 3)]


def p2_tet_coords(v):
    """10 nodes of a straight-sided P2 tet from its 4 vertices (3,4)."""
    mids = [(v[:, a] + v[:, b]) / 2 for a, b in P2_EDGES]
    return np.concatenate([v, np.stack(mids, axis=1)], axis=1)


def one_element(etype, order, coords, bsets=()):
    coords = np.ascontiguousarray(np.asarray(coords, dtype=float))
    n = coords.shape[1]
    conn = np.arange(n, dtype=np.int32).reshape(n, 1)
    m = Mesh(coords.shape[0], etype, order, coords, conn)
    m.bsets = [(np.asarray(e, np.int32), np.asarray(f, np.int8)) for e, f in bsets]
    return m


def problem(physics, etype, order, terms, quad_order=2, time=None):
    return Problem(physics, etype, order, quad_order, [Term(*t) for t in terms], time or TimeScheme())


def row_scaled_err(K_test, K_ref):
    """Reading L20: max_ij |K^test_ij - K^ref_ij| / max_j |K^ref_ij| (row-scaled)."""
    num = np.abs(K_test - K_ref).max(axis=1)
    den = np.abs(K_ref).max(axis=1)
    den = np.where(den > 0, den, 1.0)
    return float((num / den).max()) if len(num) else 0.0


def csr_row_scaled_err(rowptr, values_test, values_ref):
    """Reading L20 on CSR arrays with identical patterns."""
    diff = np.abs(values_test - values_ref)
    ref = np.abs(values_ref)
    nr = len(rowptr) - 1
    lens = np.diff(rowptr)
    rid = np.repeat(np.arange(nr), lens)
    rmax = np.zeros(nr)
    np.maximum.at(rmax, rid, ref)
    dmax = np.zeros(nr)
    np.maximum.at(dmax, rid, diff)
    ok = rmax > 0
    out = np.where(ok, dmax / np.where(ok, rmax, 1.0), dmax)
    return float(out.max()) if nr else 0.0


def rhs_err(d_test, d_ref, abs_d):
    """Reading L20: max_i |d^test_i - d^ref_i| / max(|d^ref_i|, A_d[i])."""
    den = np.maximum(np.abs(d_ref), abs_d)
    den = np.where(den > 0, den, 1.0)
    return float((np.abs(d_test - d_ref) / den).max()) if len(d_ref) else 0.0


def part_csr_to_global(part, rowptr, colidx, values, kh, n_global):
    """A partitioned rank's CSR (local relabelling, paper.partition) as global rows: returns
    (global row ids, rowptr, global colidx sorted within each row, values permuted alike).  Index
    bookkeeping only (the relabelling of paper_2111_03541_b200/partition.py)."""
    rows = part.global_rows(kh, n_global)
    cols = part.global_cols(colidx, n_global)
    out_c = np.empty_like(cols)
    out_v = np.empty_like(values)
    for r in range(len(rows)):
        a, b = rowptr[r], rowptr[r + 1]
        o = np.argsort(cols[a:b], kind="stable")
        out_c[a:b] = cols[a:b][o]
        out_v[a:b] = values[a:b][o]
    return rows, rowptr, out_c, out_v


def scatter_rows_into(full_rowptr, full_colidx, rows, rowptr, cols, vals, dst):
    """Place a part's global-row CSR into a full-size values array after checking that every row's global
    columns equal the full pattern's row (pattern bit-exact)."""
    for r, g in enumerate(rows):
        a, b = full_rowptr[g], full_rowptr[g + 1]
        np.testing.assert_array_equal(cols[rowptr[r]:rowptr[r + 1]], full_colidx[a:b])
        dst[a:b] = vals[rowptr[r]:rowptr[r + 1]]


def poisoned_system(mesh, problem, own=None):
    """A FemSystem whose outputs are filled with NaN before every non-accumulating assembly call, so a
    kernel that skips entries (or a call that silently does nothing) cannot pass on the values an earlier
    call left in the reused buffers."""
    from paper_2111_03541_b200 import FemSystem

    class _Poisoned(FemSystem):
        def _poison(self, matrix, residual, accumulate):
            self.alloc(matrix, residual)
            if not accumulate:
                if matrix:
                    self.values.fill_(float("nan"))
                if residual:
                    self.rhs.fill_(float("nan"))

        def system(self, state, scatter="atomic", accumulate=False):
            self._poison(True, True, accumulate)
            return super().system(state, scatter=scatter, accumulate=accumulate)

        def matrix(self, state, scatter="atomic", accumulate=False):
            self._poison(True, False, accumulate)
            return super().matrix(state, scatter=scatter, accumulate=accumulate)

        def residual(self, state, scatter="atomic", accumulate=False):
            self._poison(False, True, accumulate)
            return super().residual(state, scatter=scatter, accumulate=accumulate)

    return _Poisoned(mesh, problem, own=own)
