"""Thin ctypes binding of libfem.so (include/libfem.h) — argument marshalling only.

Every step of the assembly path runs inside libfem.so (hand-written CUDA for sm_100a).  There is
no CPU fallback: if the library is missing this module raises at import/first use.  PyTorch is
used by callers only for device memory and streams; tensors are passed as raw pointers.
Function names mirror the C ABI.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("FEM_LIB_PATH") or os.path.join(_HERE, "libfem.so")  # override: dev A/B builds

FEM_TRI, FEM_TET, FEM_HEX, FEM_HEX_SERENDIPITY = 1, 2, 4, 5
FEM_THERMAL, FEM_ELASTICITY, FEM_NS = 1, 2, 3
SCATTER = {"atomic": 0, "coloured": 1, "tiled": 2, "tiled_unordered": 3, "stored": 4}
ETYPE = {"tri": FEM_TRI, "tet": FEM_TET, "hex": FEM_HEX, "hexs": FEM_HEX_SERENDIPITY}
PHYSICS = {"thermal": FEM_THERMAL, "elasticity": FEM_ELASTICITY, "ns": FEM_NS}
FORM = {
    "THERMAL_DOMAIN": 0, "THERMAL_CONV_RAD": 1, "THERMAL_FIX": 2,
    "ELAST_DOMAIN": 3, "ELAST_FIX_ALL": 4, "ELAST_FIX_D1": 5, "ELAST_LOAD": 6,
    "NS_DOMAIN": 7, "NS_BND_INFLOW": 8, "NS_BND_OUTFLOW": 9, "NS_BND_FIX": 10,
}
ERRORS = {-1: "INVALID_ARG", -2: "UNSUPPORTED", -3: "INDEX_OVERFLOW", -4: "INVERTED_ELEMENT", -5: "NAN",
          -6: "CUDA", -8: "OOM"}


class FemError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"libfem error {code} ({ERRORS.get(code, '?')}): {msg}")
        self.code = code


class fem_time_scheme(C.Structure):
    _fields_ = [("kind", C.c_int), ("nu_hat", C.c_int), ("dt", C.c_double), ("b1", C.c_double),
                ("b2", C.c_double), ("c1", C.c_double), ("c2", C.c_double), ("c3", C.c_double)]


class fem_term(C.Structure):
    _fields_ = [("form", C.c_int), ("region", C.c_int), ("params", C.c_double * 16)]


class fem_problem(C.Structure):
    _fields_ = [("etype", C.c_int), ("order", C.c_int), ("quad_order", C.c_int), ("physics", C.c_int),
                ("time", fem_time_scheme), ("n_terms", C.c_int), ("terms", fem_term * 16)]


def form_params(form: str, p: dict):
    """Positional params[] layout of include/libfem.h for each weak form."""
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


def make_problem(prob) -> fem_problem:
    """Marshal a problem description (attributes physics/etype/order/quad_order/terms/time)."""
    P = fem_problem()
    P.etype = ETYPE[prob.etype]
    P.order = prob.order
    P.quad_order = prob.quad_order
    P.physics = PHYSICS[prob.physics]
    t = prob.time
    P.time.kind = 1 if t.kind == "genalpha" else 0
    P.time.nu_hat = t.nu_hat if t.kind == "genalpha" else 0
    P.time.dt, P.time.b1, P.time.b2 = t.dt, t.b1, t.b2
    P.time.c1, P.time.c2, P.time.c3 = t.c1, t.c2, t.c3
    P.n_terms = len(prob.terms)
    for i, term in enumerate(prob.terms):
        P.terms[i].form = FORM[term.form]
        P.terms[i].region = term.region
        for j, v in enumerate(form_params(term.form, term.params)):
            P.terms[i].params[j] = float(v)
    return P


_lib = None


def lib():
    """Load libfem.so (fails loudly if it has not been built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise FileNotFoundError(f"{LIB_PATH} is missing: run `python -m paper_2111_03541_b200.build`")
        L = C.CDLL(LIB_PATH)
        V, I, I64 = C.c_void_p, C.c_int, C.c_int64
        PP = C.POINTER(fem_problem)
        L.fem_mesh_create.argtypes = [PP, I, I64, V, I64, V, I, V, V, V, I64, I64, V, C.POINTER(V)]
        L.fem_pattern_build.argtypes = [V, V, C.POINTER(V), C.POINTER(I64), C.POINTER(I64)]
        L.fem_pattern_nnz_s.argtypes = [V]
        L.fem_pattern_nnz_s.restype = I64
        L.fem_pattern_export.argtypes = [V, V, V, V, V, V, V]
        L.fem_pattern_info.argtypes = [V, V]
        L.fem_pattern_stored_prepare.argtypes = [V, I, V]
        L.fem_assemble_matrix.argtypes = [V, V, PP, V, V, I, I, V]
        L.fem_assemble_residual.argtypes = [V, V, PP, V, V, I, I, V]
        L.fem_assemble_system.argtypes = [V, V, PP, V, V, V, I, I, V]
        L.fem_residual_norms.argtypes = [V, V, V, V]
        L.fem_linearize_host.argtypes = [V, V, PP, V, V, V, V, I, V]
        L.fem_linearize_host_async.argtypes = [V, V, PP, V, V, V, V, I, V]
        L.fem_pattern_export_coo.argtypes = [V, I64, V, V, V, V]
        L.fem_gather.argtypes = [I64, V, V, V, V]
        L.fem_get_status.argtypes = [V, V, C.POINTER(I64)]
        L.fem_mesh_info.argtypes = [V, C.POINTER(I), C.POINTER(I), C.POINTER(I), C.POINTER(I64)]
        L.fem_pattern_destroy.argtypes = [V]
        L.fem_pattern_destroy.restype = None
        L.fem_mesh_destroy.argtypes = [V]
        L.fem_mesh_destroy.restype = None
        L.fem_pattern_csr.argtypes = [V, C.POINTER(V), C.POINTER(V), C.POINTER(I64)]
        L.fem_spmv.argtypes = [I64, V, V, V, V, V, C.c_double, C.c_double, V]
        L.fem_vec_axpby.argtypes = [I64, C.c_double, V, C.c_double, V, V]
        L.fem_gmres_work_doubles.argtypes = [I64, I64, I, I]
        L.fem_gmres_work_doubles.restype = I64
        L.fem_gmres_solve.argtypes = [I64, V, V, V, I64, I, V, V, I, I, C.c_double, I64, V, C.POINTER(I),
                                      C.POINTER(C.c_double), V]
        L.fem_cg_work_doubles.argtypes = [I64]
        L.fem_cg_work_doubles.restype = I64
        L.fem_cg_solve.argtypes = [I64, V, V, V, V, V, C.c_double, I, C.c_double, I, V, C.POINTER(I),
                                   C.POINTER(C.c_double), V]
        L.fem_bicgstab_work_doubles.argtypes = [I64]
        L.fem_bicgstab_work_doubles.restype = I64
        L.fem_bicgstab_solve.argtypes = [I64, V, V, V, V, V, I, C.c_double, I, V, C.POINTER(I),
                                         C.POINTER(C.c_double), V]
        PT = C.POINTER(fem_time_scheme)
        L.fem_time_init.argtypes = [PT, I64, V, V, V, V]
        L.fem_time_effective.argtypes = [PT, I64, V, V, V, V]
        L.fem_time_increment.argtypes = [PT, I64, V, V, V, V, V]
        L.fem_last_error.restype = C.c_char_p
        L.fem_version.restype = I
        _lib = L
    return _lib


EXPORTED = ["fem_mesh_create", "fem_pattern_build", "fem_pattern_nnz_s", "fem_pattern_export", "fem_pattern_info",
            "fem_assemble_matrix", "fem_assemble_residual", "fem_assemble_system", "fem_residual_norms",
            "fem_linearize_host", "fem_linearize_host_async", "fem_pattern_export_coo", "fem_gather", "fem_get_status", "fem_mesh_info", "fem_pattern_destroy",
            "fem_mesh_destroy", "fem_last_error", "fem_version", "fem_pattern_csr", "fem_spmv",
            "fem_cg_work_doubles", "fem_cg_solve", "fem_bicgstab_work_doubles", "fem_bicgstab_solve",
            "fem_time_init", "fem_time_effective", "fem_time_increment", "fem_vec_axpby",
            "fem_gmres_work_doubles", "fem_gmres_solve", "fem_pattern_stored_prepare"]


def _check(rc):
    if rc != 0:
        raise FemError(rc, lib().fem_last_error().decode())


def _ptr(x):
    """Raw address of a torch tensor / numpy array / int / None."""
    if x is None:
        return None
    if isinstance(x, int):
        return x
    if hasattr(x, "data_ptr"):
        return x.data_ptr()
    if isinstance(x, np.ndarray):
        return x.ctypes.data
    raise TypeError(type(x))


def _stream(stream):
    if stream is None:
        try:
            import torch
            if torch.cuda.is_available():
                return torch.cuda.current_stream().cuda_stream
        except ImportError:
            pass
        return None
    return stream if isinstance(stream, int) else stream.cuda_stream


def fem_mesh_create(problem, mesh, own=None, stream=None):
    """mesh: object with dim, coords (dim,N) f64, conn (n_loc,E) i32, bsets [(elem i32, facet i8)]."""
    L = lib()
    P = make_problem(problem)
    coords = np.ascontiguousarray(mesh.coords, dtype=np.float64)
    conn = np.ascontiguousarray(mesh.conn, dtype=np.int32)
    be = [np.ascontiguousarray(b[0], dtype=np.int32) for b in mesh.bsets]
    bf = [np.ascontiguousarray(b[1], dtype=np.int8) for b in mesh.bsets]
    nb = len(be)
    blen = np.array([len(b) for b in be] or [0], dtype=np.int64)
    bep = (C.c_void_p * max(nb, 1))(*[b.ctypes.data for b in be])
    bfp = (C.c_void_p * max(nb, 1))(*[b.ctypes.data for b in bf])
    lo, hi = (0, coords.shape[1]) if own is None else own
    h = C.c_void_p()
    _check(L.fem_mesh_create(C.byref(P), mesh.dim, coords.shape[1], coords.ctypes.data, conn.shape[1],
                             conn.ctypes.data, nb, blen.ctypes.data, C.cast(bep, C.c_void_p),
                             C.cast(bfp, C.c_void_p), lo, hi, _stream(stream), C.byref(h)))
    return h.value


def fem_pattern_build(mesh_h, stream=None):
    L = lib()
    h, nr, nnz = C.c_void_p(), C.c_int64(), C.c_int64()
    _check(L.fem_pattern_build(mesh_h, _stream(stream), C.byref(h), C.byref(nr), C.byref(nnz)))
    return h.value, nr.value, nnz.value


def fem_pattern_nnz_s(pat_h):
    return lib().fem_pattern_nnz_s(pat_h)


def fem_pattern_info(pat_h):
    out = np.zeros(9, dtype=np.int64)
    _check(lib().fem_pattern_info(pat_h, out.ctypes.data))
    keys = ["tiles", "max_tile_points", "max_acc_doubles", "max_record_bytes", "max_halo_points", "visits",
            "max_tile_visits", "record_bytes", "schedule"]
    return dict(zip(keys, out.tolist()))


def fem_pattern_stored_prepare(pat_h, with_matrix=True, stream=None):
    _check(lib().fem_pattern_stored_prepare(pat_h, int(bool(with_matrix)), _stream(stream)))


def fem_pattern_export(pat_h, rowptr=None, colidx=None, slot_s=None, rowptr_s=None, colidx_s=None, stream=None):
    _check(lib().fem_pattern_export(pat_h, _ptr(rowptr), _ptr(colidx), _ptr(slot_s), _ptr(rowptr_s),
                                    _ptr(colidx_s), _stream(stream)))


def fem_assemble_matrix(mesh_h, pat_h, problem, state, values, accumulate=0, scatter="atomic", stream=None):
    P = make_problem(problem)
    _check(lib().fem_assemble_matrix(mesh_h, pat_h, C.byref(P), _ptr(state), _ptr(values), int(accumulate),
                                     SCATTER[scatter], _stream(stream)))


def fem_assemble_residual(mesh_h, pat_h, problem, state, rhs, accumulate=0, scatter="atomic", stream=None):
    P = make_problem(problem)
    _check(lib().fem_assemble_residual(mesh_h, pat_h, C.byref(P), _ptr(state), _ptr(rhs), int(accumulate),
                                       SCATTER[scatter], _stream(stream)))


def fem_assemble_system(mesh_h, pat_h, problem, state, values, rhs, accumulate=0, scatter="atomic",
                        stream=None, P=None):
    P = P if P is not None else make_problem(problem)
    _check(lib().fem_assemble_system(mesh_h, pat_h, C.byref(P), _ptr(state), _ptr(values), _ptr(rhs),
                                     int(accumulate), SCATTER[scatter], _stream(stream)))


def fem_residual_norms(mesh_h, rhs, norms, stream=None):
    _check(lib().fem_residual_norms(mesh_h, _ptr(rhs), _ptr(norms), _stream(stream)))


def fem_linearize_host(mesh_h, pat_h, problem, state_host, values, rhs, norms_host, scatter="atomic",
                       stream=None, P=None):
    P = P if P is not None else make_problem(problem)
    _check(lib().fem_linearize_host(mesh_h, pat_h, C.byref(P), _ptr(state_host), _ptr(values), _ptr(rhs),
                                    _ptr(norms_host), SCATTER[scatter], _stream(stream)))


def fem_pattern_csr(pat_h):
    """Library-owned device CSR of the pattern: (rowptr ptr, colidx ptr, column offset)."""
    rp, ci, off = C.c_void_p(), C.c_void_p(), C.c_int64()
    _check(lib().fem_pattern_csr(pat_h, C.byref(rp), C.byref(ci), C.byref(off)))
    return rp.value, ci.value, off.value


def fem_spmv(n_rows, rowptr, colidx, values, x, y, alpha=1.0, beta=0.0, stream=None):
    _check(lib().fem_spmv(int(n_rows), _ptr(rowptr), _ptr(colidx), _ptr(values), _ptr(x), _ptr(y), float(alpha),
                          float(beta), _stream(stream)))


def fem_vec_axpby(n, alpha, x, beta, y, stream=None):
    """y = alpha x + beta y on the device (fem_vec_axpby)."""
    _check(lib().fem_vec_axpby(int(n), float(alpha), _ptr(x), float(beta), _ptr(y), _stream(stream)))


def fem_gmres_work_doubles(n_rows, n_points, kappa_hat, restart=30):
    return int(lib().fem_gmres_work_doubles(int(n_rows), int(n_points), int(kappa_hat), int(restart)))


def fem_gmres_solve(n_rows, rowptr, colidx, values, n_points, kappa_hat, b, x, work, restart=30, max_iter=2000,
                    rtol=1e-10, pin_row=-1, stream=None):
    """Point-block-Jacobi GMRES(restart) for K x = b (row/column pin_row pinned to the identity when >= 0);
    returns (Arnoldi steps, ||b - K x|| / ||b|| of the pinned system)."""
    it, rel = C.c_int(0), C.c_double(0.0)
    _check(lib().fem_gmres_solve(int(n_rows), _ptr(rowptr), _ptr(colidx), _ptr(values), int(n_points),
                                 int(kappa_hat), _ptr(b), _ptr(x), int(restart), int(max_iter), float(rtol),
                                 int(pin_row), _ptr(work), C.byref(it), C.byref(rel), _stream(stream)))
    return it.value, rel.value


def fem_cg_work_doubles(n_rows):
    return int(lib().fem_cg_work_doubles(int(n_rows)))


def fem_cg_solve(n_rows, rowptr, colidx, values, b, x, work, spd_sign=-1.0, max_iter=10000, rtol=1e-12,
                 check_every=16, stream=None):
    """Jacobi-PCG for K x = b on (spd_sign K) x = spd_sign b; returns (iterations, ||r||/||r0||)."""
    it, rel = C.c_int(0), C.c_double(0.0)
    _check(lib().fem_cg_solve(int(n_rows), _ptr(rowptr), _ptr(colidx), _ptr(values), _ptr(b), _ptr(x),
                              float(spd_sign), int(max_iter), float(rtol), int(check_every), _ptr(work),
                              C.byref(it), C.byref(rel), _stream(stream)))
    return it.value, rel.value


def fem_bicgstab_work_doubles(n_rows):
    return int(lib().fem_bicgstab_work_doubles(int(n_rows)))


def fem_bicgstab_solve(n_rows, rowptr, colidx, values, b, x, work, max_iter=10000, rtol=1e-12, check_every=16,
                       stream=None):
    """Jacobi-BiCGStab for K x = b (non-symmetric K); returns (iterations, ||r||/||r0||)."""
    it, rel = C.c_int(0), C.c_double(0.0)
    _check(lib().fem_bicgstab_solve(int(n_rows), _ptr(rowptr), _ptr(colidx), _ptr(values), _ptr(b), _ptr(x),
                                    int(max_iter), float(rtol), int(check_every), _ptr(work), C.byref(it),
                                    C.byref(rel), _stream(stream)))
    return it.value, rel.value


def fem_linearize_host_async(mesh_h, pat_h, problem, state_host, values, rhs, norms_host, scatter="atomic",
                             stream=None, P=None):
    """Pipelined host-buffer linearisation (no sync): the H2D of this call overlaps the previous assembly."""
    P = P if P is not None else make_problem(problem)
    _check(lib().fem_linearize_host_async(mesh_h, pat_h, C.byref(P), _ptr(state_host), _ptr(values), _ptr(rhs),
                                          _ptr(norms_host), SCATTER[scatter], _stream(stream)))


def fem_pattern_export_coo(pat_h, row_offset, I, J, csr_index, stream=None):
    _check(lib().fem_pattern_export_coo(pat_h, int(row_offset), _ptr(I), _ptr(J), _ptr(csr_index), _stream(stream)))


def fem_gather(n, index, src, dst, stream=None):
    _check(lib().fem_gather(int(n), _ptr(index), _ptr(src), _ptr(dst), _stream(stream)))


def make_time_scheme(t) -> fem_time_scheme:
    """Marshal a TimeScheme (kind/nu_hat/dt/b1/b2/c1/c2/c3) for the NEXT-3 time-stepping calls."""
    T = fem_time_scheme()
    T.kind = 1 if t.kind == "genalpha" else 0
    T.nu_hat = t.nu_hat
    T.dt, T.b1, T.b2, T.c1, T.c2, T.c3 = t.dt, t.b1, t.b2, t.c1, t.c2, t.c3
    return T


def fem_time_init(ts, n, phi0, incr, eff=None, stream=None):
    _check(lib().fem_time_init(C.byref(ts), int(n), _ptr(phi0), _ptr(incr), _ptr(eff), _stream(stream)))


def fem_time_effective(ts, n, phi0, incr, eff, stream=None):
    _check(lib().fem_time_effective(C.byref(ts), int(n), _ptr(phi0), _ptr(incr), _ptr(eff), _stream(stream)))


def fem_time_increment(ts, n, delta_sub, incr, phi0=None, eff=None, stream=None):
    _check(lib().fem_time_increment(C.byref(ts), int(n), _ptr(delta_sub), _ptr(incr), _ptr(phi0), _ptr(eff),
                                    _stream(stream)))


def fem_get_status(mesh_h, stream=None):
    bad = C.c_int64(-1)
    rc = lib().fem_get_status(mesh_h, _stream(stream), C.byref(bad))
    return rc, bad.value


def fem_mesh_info(mesh_h):
    a, b, c, d = C.c_int(), C.c_int(), C.c_int(), C.c_int64()
    _check(lib().fem_mesh_info(mesh_h, C.byref(a), C.byref(b), C.byref(c), C.byref(d)))
    return dict(n_loc=a.value, kappa_hat=b.value, n_colours=c.value, n_tiles=d.value)


def fem_pattern_destroy(pat_h):
    lib().fem_pattern_destroy(pat_h)


def fem_mesh_destroy(mesh_h):
    lib().fem_mesh_destroy(mesh_h)


def fem_version():
    return lib().fem_version()
