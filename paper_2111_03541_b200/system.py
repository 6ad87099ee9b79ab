"""FemSystem — torch-tensor convenience wrapper over the libfem C ABI (no compute here: every step of
the method, including the Newton update and the convergence norms, runs in libfem.so)."""
from __future__ import annotations

import math

import torch

from . import fem


class FemSystem:
    """Owns one libfem mesh + pattern and the caller-side device buffers (values, rhs).

    mesh: fem_inputs.Mesh-like (dim, coords, conn, bsets); problem: fem_inputs.Problem-like.
    own:  (lo, hi) owned control-point range (multi-GPU partition), default all points.
    """

    def __init__(self, mesh, problem, own=None, device="cuda", build_pattern=True, stream=None):
        self.problem = problem
        self.P = fem.make_problem(problem)
        self.dim = mesh.dim
        self.N = mesh.coords.shape[1]
        self.E = mesh.conn.shape[1]
        self.n_loc = mesh.conn.shape[0]
        self.own = (0, self.N) if own is None else tuple(own)
        self.n_own = self.own[1] - self.own[0]
        self.device = torch.device(device)
        self.kh = problem.kappa_hat(mesh.dim)
        self.mesh_h = fem.fem_mesh_create(problem, mesh, own=self.own, stream=stream)
        self.pat_h = None
        self.n_rows = self.kh * self.n_own
        self.nnz = None
        if build_pattern:
            self.pat_h, self.n_rows, self.nnz = fem.fem_pattern_build(self.mesh_h, stream=stream)
            self.nnz_s = fem.fem_pattern_nnz_s(self.pat_h)
        self.values = None
        self.rhs = None
        self._stored = 0  # FEM_SCATTER_STORED setup: 0 none, 1 residual scratch, 2 with the element blocks

    def info(self):
        d = fem.fem_mesh_info(self.mesh_h)
        if self.pat_h:
            d.update(fem.fem_pattern_info(self.pat_h))
        return d

    def alloc(self, matrix=True, residual=True):
        if matrix and self.values is None:
            self.values = torch.empty(self.nnz, dtype=torch.float64, device=self.device)
        if residual and self.rhs is None:
            self.rhs = torch.empty(self.n_rows, dtype=torch.float64, device=self.device)

    def export_pattern(self, slot=True):
        dev = self.device
        out = dict(rowptr=torch.empty(self.n_rows + 1, dtype=torch.int64, device=dev),
                   colidx=torch.empty(self.nnz, dtype=torch.int32, device=dev),
                   rowptr_s=torch.empty(self.n_own + 1, dtype=torch.int64, device=dev),
                   colidx_s=torch.empty(self.nnz_s, dtype=torch.int32, device=dev))
        if slot:
            out["slot_s"] = torch.empty((self.n_loc * self.n_loc, self.E), dtype=torch.int32, device=dev)
        fem.fem_pattern_export(self.pat_h, out["rowptr"], out["colidx"], out.get("slot_s"), out["rowptr_s"],
                               out["colidx_s"])
        return out

    def export_coo(self, row_offset=0, values=True):
        """NEXT-4: the paper's COO view (B-4) in sparse-ID order: dict(I, J, csr_index[, values])
        with I, J offset by the workpiece's n^dense (row_offset)."""
        dev = self.device
        out = {k: torch.empty(self.nnz, dtype=torch.int64, device=dev) for k in ("I", "J", "csr_index")}
        fem.fem_pattern_export_coo(self.pat_h, row_offset, out["I"], out["J"], out["csr_index"])
        if values and self.values is not None:
            out["values"] = torch.empty(self.nnz, dtype=torch.float64, device=dev)
            fem.fem_gather(self.nnz, out["csr_index"], self.values, out["values"])
        return out

    def _prepare(self, scatter, matrix):
        """FEM_SCATTER_STORED needs its one-time setup (contribution lists, element scratch) first."""
        if scatter == "stored" and self._stored < (2 if matrix else 1):
            fem.fem_pattern_stored_prepare(self.pat_h, with_matrix=matrix)
            self._stored = 2 if matrix else 1

    def matrix(self, state, scatter="atomic", accumulate=False):
        self._prepare(scatter, True)
        self.alloc(True, False)
        fem.fem_assemble_matrix(self.mesh_h, self.pat_h, self.problem, state, self.values, int(accumulate),
                                scatter)
        return self.values

    def residual(self, state, scatter="atomic", accumulate=False):
        self._prepare(scatter, False)
        self.alloc(False, True)
        fem.fem_assemble_residual(self.mesh_h, self.pat_h, self.problem, state, self.rhs, int(accumulate),
                                  scatter)
        return self.rhs

    def system(self, state, scatter="atomic", accumulate=False):
        self._prepare(scatter, True)
        self.alloc(True, True)
        fem.fem_assemble_system(self.mesh_h, self.pat_h, self.problem, state, self.values, self.rhs,
                                int(accumulate), scatter, P=self.P)
        return self.values, self.rhs

    # ---- NEXT-1: the Newton sub-step's linear solve (D-4) on the GPU
    def solve(self, b, x=None, spd_sign=-1.0, rtol=1e-12, max_iter=20000, check_every=16, method="cg", restart=30):
        """Solve K x = b for the last assembled K (self.values).  method "cg": Jacobi-PCG on (spd_sign K)
        — the elasticity K is symmetric negative definite in the paper's sign convention (reading L17);
        "bicgstab": Jacobi-BiCGStab for non-symmetric K (thermal FIX); "gmres": point-block-Jacobi GMRES(restart)
        for the NS saddle point.  Returns (x, iterations,
        ||r|| / ||r0||).  Single-GPU patterns only."""
        if self.own != (0, self.N):
            raise ValueError("solve: the iterative solvers take a single-GPU (unpartitioned) pattern")
        if x is None:
            x = torch.zeros(self.n_rows, dtype=torch.float64, device=self.device)
        rp, ci, _ = fem.fem_pattern_csr(self.pat_h)
        if method == "cg":
            if getattr(self, "_cg_work", None) is None:
                self._cg_work = torch.empty(fem.fem_cg_work_doubles(self.n_rows), dtype=torch.float64,
                                            device=self.device)
            it, rel = fem.fem_cg_solve(self.n_rows, rp, ci, self.values, b, x, self._cg_work, spd_sign, max_iter,
                                       rtol, check_every)
        elif method == "gmres":
            need = fem.fem_gmres_work_doubles(self.n_rows, self.N, self.kh, restart)
            if getattr(self, "_gm_work", None) is None or self._gm_work.numel() < need:
                self._gm_work = torch.empty(need, dtype=torch.float64, device=self.device)
            # NS: pin the pressure of point 0 (the paper's forms fix the pressure only up to a constant, L29)
            pin = self.dim * self.N if self.problem.physics == "ns" else -1
            it, rel = fem.fem_gmres_solve(self.n_rows, rp, ci, self.values, self.N, self.kh, b, x, self._gm_work,
                                          restart, max_iter, rtol, pin)
        elif method == "bicgstab":
            if getattr(self, "_bi_work", None) is None:
                self._bi_work = torch.empty(fem.fem_bicgstab_work_doubles(self.n_rows), dtype=torch.float64,
                                            device=self.device)
            it, rel = fem.fem_bicgstab_solve(self.n_rows, rp, ci, self.values, b, x, self._bi_work, max_iter, rtol,
                                             check_every)
        else:
            raise ValueError(method)
        return x, it, rel

    def spmv(self, x, y=None, alpha=1.0, beta=0.0):
        """y = alpha K x + beta y with the last assembled K (single-GPU pattern)."""
        if y is None:
            y = torch.zeros(self.n_rows, dtype=torch.float64, device=self.device)
        rp, ci, _ = fem.fem_pattern_csr(self.pat_h)
        fem.fem_spmv(self.n_rows, rp, ci, self.values, x, y, alpha, beta)
        return y

    def _solve_checked(self, d, method, spd_sign, rtol, max_iter, restart=200):
        """Solve K y = d (y = -Δφ of D-4) and reject a NaN / non-converged solve (returns y, it, rel)."""
        y, it, rel = self.solve(d, spd_sign=spd_sign, rtol=rtol, max_iter=max_iter, method=method, restart=restart)
        if not math.isfinite(rel):
            raise fem.FemError(-5, f"linear solve broke down (relative residual {rel})")
        return y, it, rel

    def newton_step(self, state, scatter="tiled", spd_sign=-1.0, rtol=1e-12, max_iter=20000, method="cg", restart=200):
        """One Newton sub-step (D-1..D-4) for a static problem: assemble K and d at φ, solve
        K Δφ = -d as K y = d, φ ← φ - y (fem_vec_axpby).  Returns the new state (level 0
        updated), the solver iterations and the relative residual ||r||/||r0|| (compare with rtol: hitting
        max_iter is reported, not raised; a NaN raises FemError)."""
        K, d = self.system(state, scatter=scatter)
        y, it, rel = self._solve_checked(d, method, spd_sign, rtol, max_iter, restart)
        new = state.clone()
        fem.fem_vec_axpby(self.kh * self.N, -1.0, y, 1.0, new[0])
        return new, it, rel

    # ---- NEXT-3: one generalized-alpha timestep (Blocks C and D) on the GPU
    def time_step(self, phi0, incr, n_sub=1, scatter="tiled", method="bicgstab", spd_sign=-1.0, rtol=1e-12,
                  max_iter=20000, tol=0.0):
        """Advance one timestep with the problem's generalized-alpha scheme, in place on the DEVICE arrays
        phi0 (committed ∂^ν φ) and incr (Δ∂^ν φ), both float64 [ν̂+1][κ̂][N].  Block C (fem_time_init,
        fused with the first D-1), then up to n_sub sub-steps: assemble K, d at the effective values (D-2,
        D-3), the D-2 test ||d||_2 <= tol (fem_residual_norms), solve K y = d (D-4, CG/BiCGStab), Δ_sub = -y
        (fem_vec_axpby), fem_time_increment (fused with the next D-1).  Returns the list of
        (||d||_2 before the solve, iterations, relative solver residual)."""
        t = self.problem.time
        if t.kind != "genalpha":
            raise ValueError("time_step needs a genalpha problem")
        ts = fem.make_time_scheme(t)
        n = self.kh * self.N
        eff = getattr(self, "_eff", None)
        if eff is None or eff.shape != phi0.shape:
            eff = self._eff = torch.empty_like(phi0)
        fem.fem_time_init(ts, n, phi0, incr, eff)
        hist = []
        for _ in range(n_sub):
            K, d = self.system(eff, scatter=scatter)
            dn = math.sqrt(float(self.norms(d)[0]))
            if dn <= tol:
                hist.append((dn, 0, 0.0))
                break
            y, it, rel = self._solve_checked(d, method, spd_sign, rtol, max_iter)
            fem.fem_vec_axpby(n, 0.0, y, -1.0, y)   # Δ_sub = -y
            fem.fem_time_increment(ts, n, y, incr, phi0, eff)
            hist.append((dn, it, rel))
        return hist

    def norms(self, rhs=None):
        out = torch.empty(2, dtype=torch.float64, device=self.device)
        fem.fem_residual_norms(self.mesh_h, self.rhs if rhs is None else rhs, out)
        return out

    def status(self):
        return fem.fem_get_status(self.mesh_h)

    def close(self):
        if getattr(self, "pat_h", None):
            fem.fem_pattern_destroy(self.pat_h)
            self.pat_h = None
        if getattr(self, "mesh_h", None):
            fem.fem_mesh_destroy(self.mesh_h)
            self.mesh_h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
