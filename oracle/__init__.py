"""oracle — TEST INFRASTRUCTURE ONLY.

Plain serial fp64 CPU oracle of the MetaFEM assembly (arXiv:2111.03541 Blocks B/D), written
from PAPER.md in C (fem_oracle.c) and loaded with ctypes.  Only tests/, __graft_entry__.smoke()
and bench.py's cpu_baseline / --impl reference legs may import this package; the product path
(paper_2111_03541_b200) never does.  Parity pins: see tests/test_oracle_*.py and DESIGN.md §5.
Residual families are pinned by closed-form weak-form moments (tests/test_oracle_pins_flux.py); the
inflow profile term (degree 4 under a degree-2 facet rule) is pinned by convergence to its exact integral.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "fem_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

ETYPE = {"tri": 1, "tet": 2, "hex": 4, "hexs": 5}
PHYSICS = {"thermal": 1, "elasticity": 2, "ns": 3}
FORM = {
    "THERMAL_DOMAIN": 0, "THERMAL_CONV_RAD": 1, "THERMAL_FIX": 2,
    "ELAST_DOMAIN": 3, "ELAST_FIX_ALL": 4, "ELAST_FIX_D1": 5, "ELAST_LOAD": 6,
    "NS_DOMAIN": 7, "NS_BND_INFLOW": 8, "NS_BND_OUTFLOW": 9, "NS_BND_FIX": 10,
}


def _params(form: str, p: dict):
    """Positional parameter layout of fem_oracle.c for each weak form."""
    if form == "THERMAL_DOMAIN":
        return [p["C"], p["k"], p["s"], 1.0 if p.get("source", "const") == "sine" else 0.0]
    if form == "THERMAL_CONV_RAD":
        return [p["h"], p["T_env"], p["e_m"], p["sigma_b"]]
    if form == "THERMAL_FIX":
        return [p["h_p"], p["T_fix"], p["k"]]
    if form == "ELAST_DOMAIN":
        return [p["E"], p["nu"]]
    if form == "ELAST_FIX_ALL":
        return [p["tau"], *p.get("dw", (0.0, 0.0, 0.0))]
    if form == "ELAST_FIX_D1":
        return [p["tau"], p.get("dw", (0.0,))[0]]
    if form == "ELAST_LOAD":
        return list(p["sigma_l"])
    if form == "NS_DOMAIN":
        return [p["rho"], p["mu"], p["tau_m"], p["tau_c"]]
    if form == "NS_BND_INFLOW":
        return [p["rho"], p["mu"], p["tau_b"], p["U"], p["H"]]
    if form == "NS_BND_OUTFLOW":
        return [p["rho"], p["mu"]]
    if form == "NS_BND_FIX":
        return [p["rho"], p["mu"], p["tau_b"]]
    raise KeyError(form)


class _Term(C.Structure):
    _fields_ = [("form", C.c_int), ("region", C.c_int), ("p", C.c_double * 16)]


class _Problem(C.Structure):
    _fields_ = [("physics", C.c_int), ("etype", C.c_int), ("order", C.c_int), ("quad_order", C.c_int),
                ("dim", C.c_int), ("nu_hat", C.c_int), ("dt", C.c_double), ("b1", C.c_double),
                ("b2", C.c_double), ("c1", C.c_double), ("c2", C.c_double), ("c3", C.c_double),
                ("n_terms", C.c_int), ("terms", _Term * 16)]


def build(force: bool = False) -> str:
    """Compile fem_oracle.c with gcc (plain -O2, no fast-math) into oracle/liboracle.so."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < max(
            os.path.getmtime(_SRC), os.path.getmtime(os.path.join(_HERE, "fem_oracle.h"))):
        tmp = _LIB + f".{os.getpid()}.tmp"
        subprocess.check_call(["gcc", "-O2", "-fno-fast-math", "-ffp-contract=off", "-shared",
                               "-fPIC", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        L = C.CDLL(build())
        P, I64, PI32, PF64 = C.c_void_p, C.c_int64, C.POINTER(C.c_int32), C.POINTER(C.c_double)
        L.or_assemble.restype = P
        L.or_assemble.argtypes = [C.POINTER(_Problem), I64, P, I64, P, C.c_int, P, P, P, P, P,
                                  C.c_int, C.c_int]
        L.or_status.argtypes = [P, C.POINTER(C.c_int64)]
        for f in ("or_n_sel_nodes", "or_n_rows", "or_nnz", "or_nnz_s"):
            getattr(L, f).restype = I64
            getattr(L, f).argtypes = [P]
        L.or_get.argtypes = [P] + [P] * 9
        L.or_get_slot.argtypes = [P, P, P]
        L.or_free.argtypes = [P]
        L.or_qp_data.argtypes = [C.POINTER(_Problem), I64, P, I64, P, I64, C.c_int, P, P, P, P, P, P]
        _lib = L
        del PI32, PF64
    return _lib


def make_problem(prob, dim: int) -> _Problem:
    P = _Problem()
    P.physics = PHYSICS[prob.physics]
    P.etype = ETYPE[prob.etype]
    P.order, P.quad_order, P.dim = prob.order, prob.quad_order, dim
    t = prob.time
    P.nu_hat = t.nu_hat if t.kind == "genalpha" else 0
    P.dt, P.b1, P.b2, P.c1, P.c2, P.c3 = t.dt, t.b1, t.b2, t.c1, t.c2, t.c3
    P.n_terms = len(prob.terms)
    for i, term in enumerate(prob.terms):
        P.terms[i].form = FORM[term.form]
        P.terms[i].region = term.region
        vals = _params(term.form, term.params)
        for j, v in enumerate(vals):
            P.terms[i].p[j] = float(v)
    return P


def _ptr(a):
    return a.ctypes.data_as(C.c_void_p) if a is not None else None


def assemble(mesh, prob, state, row_mask=None, matrix=True, residual=True, slot=False):
    """Run the oracle.  Returns a dict with the selected rows' CSR (rowptr, colidx, values),
    rhs, abs_d (Σ|qp contributions|, the d tolerance scale of reading L20), the scalar pattern
    (rowptr_s, colidx_s), sel_nodes, rows (global row ids) and optionally the slot map."""
    L = lib()
    P = make_problem(prob, mesh.dim)
    coords = np.ascontiguousarray(mesh.coords, dtype=np.float64)
    conn = np.ascontiguousarray(mesh.conn, dtype=np.int32)
    st = np.ascontiguousarray(state, dtype=np.float64)
    nb = len(mesh.bsets)
    blen = np.array([len(b[0]) for b in mesh.bsets] or [0], dtype=np.int64)
    be = [np.ascontiguousarray(b[0], dtype=np.int32) for b in mesh.bsets]
    bf = [np.ascontiguousarray(b[1], dtype=np.int8) for b in mesh.bsets]
    bep = (C.c_void_p * max(nb, 1))(*[_ptr(x).value for x in be])
    bfp = (C.c_void_p * max(nb, 1))(*[_ptr(x).value for x in bf])
    mask = None if row_mask is None else np.ascontiguousarray(row_mask, dtype=np.uint8)
    h = L.or_assemble(C.byref(P), mesh.n_nodes, _ptr(coords), mesh.n_elems, _ptr(conn), nb,
                      _ptr(blen), C.cast(bep, C.c_void_p), C.cast(bfp, C.c_void_p), _ptr(st),
                      _ptr(mask), int(matrix), int(residual))
    if not h:
        raise MemoryError("oracle allocation failed")
    try:
        bad = C.c_int64(-1)
        status = L.or_status(h, C.byref(bad))
        out = {"status": status, "bad_elem": bad.value}
        if status != 0:
            return out
        ns, nr, nnz, nnzs = L.or_n_sel_nodes(h), L.or_n_rows(h), L.or_nnz(h), L.or_nnz_s(h)
        out.update(sel_nodes=np.empty(ns, np.int64), rows=np.empty(nr, np.int64),
                   rowptr=np.empty(nr + 1, np.int64), colidx=np.empty(nnz, np.int32),
                   values=np.empty(nnz, np.float64), rhs=np.empty(nr, np.float64),
                   abs_d=np.empty(nr, np.float64), rowptr_s=np.empty(ns + 1, np.int64),
                   colidx_s=np.empty(nnzs, np.int32))
        L.or_get(h, *[_ptr(out[k]) for k in ("sel_nodes", "rows", "rowptr", "colidx", "values",
                                               "rhs", "abs_d", "rowptr_s", "colidx_s")])
        if slot:
            out["slot_s"] = np.empty((mesh.n_loc * mesh.n_loc, mesh.n_elems), np.int32)
            L.or_get_slot(h, _ptr(conn), _ptr(out["slot_s"]))
        return out
    finally:
        L.or_free(h)


def qp_data(mesh, prob, e: int, facet: int = -1):
    """Quadrature-point probe: dict(x, w, n, N, G, H) for element e (volume rule, or facet `facet`);
    H = physical second derivatives of the shape functions [nq][n_loc][3][3]."""
    L = lib()
    P = make_problem(prob, mesh.dim)
    coords = np.ascontiguousarray(mesh.coords, dtype=np.float64)
    conn = np.ascontiguousarray(mesh.conn, dtype=np.int32)
    nl = mesh.n_loc
    x, w, n = np.zeros((64, 3)), np.zeros(64), np.zeros((64, 3))
    N, G, H = np.zeros((64, nl)), np.zeros((64, nl, 3)), np.zeros((64, nl, 3, 3))
    nq = L.or_qp_data(C.byref(P), mesh.n_nodes, _ptr(coords), mesh.n_elems, _ptr(conn), e, facet,
                      _ptr(x), _ptr(w), _ptr(n), _ptr(N), _ptr(G), _ptr(H))
    if nq < 0:
        raise ValueError(f"oracle qp_data error {nq}")
    return dict(x=x[:nq], w=w[:nq], n=n[:nq], N=N[:nq], G=G[:nq], H=H[:nq])


def to_dense(out, n_cols):
    """Dense matrix of the selected rows (small problems only)."""
    nr = len(out["rows"])
    K = np.zeros((nr, n_cols))
    rp, ci, v = out["rowptr"], out["colidx"], out["values"]
    for r in range(nr):
        K[r, ci[rp[r]:rp[r + 1]]] = v[rp[r]:rp[r + 1]]
    return K


def coo_view(out, n_nodes: int, kappa_hat: int, row_offset: int = 0):
    """The paper's COO of one workpiece (NEXT-4): B-4 numbers the global entries by the
    sparse ID of Eq. `sparse_ID` — symbol pairs (κ₀, κ_λ) (A-3) times control-point
    pairs (α₁, α₂) (B-1 item 4), with I = (κ₀-1)α̂ + α₁, J = (κ_λ-1)α̂ + α₂ (P:398-401, 0-based
    here).  The paper hashes both pair sets; reading L4 fixes the order: symbol pairs lexicographic in
    (κ₀, κ_λ), control-point pairs lexicographic in (α₁, α₂).  Built by plain loops from the oracle's
    scalar pattern and CSR (small cases only).  row_offset = the workpiece's n^dense; a caller
    concatenating workpieces also offsets the sparse IDs by n^sp.
    Returns dict(I, J, values) in sparse-ID order."""
    rps, cis = out["rowptr_s"], out["colidx_s"]
    rp, ci, va = out["rowptr"], out["colidx"], out["values"]
    I, J, V = [], [], []
    for k0 in range(kappa_hat):
        for kl in range(kappa_hat):
            for a1 in range(n_nodes):
                for s in range(rps[a1], rps[a1 + 1]):
                    a2 = int(cis[s])
                    gi, gj = k0 * n_nodes + a1, kl * n_nodes + a2
                    row = list(ci[rp[gi]:rp[gi + 1]])
                    V.append(va[rp[gi] + row.index(gj)])
                    I.append(gi + row_offset)
                    J.append(gj + row_offset)
    return dict(I=np.array(I, np.int64), J=np.array(J, np.int64), values=np.array(V, np.float64))
