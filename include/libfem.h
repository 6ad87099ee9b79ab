/* libfem.h — C ABI of the B200-native MetaFEM assembly path (arXiv:2111.03541).
 *
 * The paper states that the linear system K x = d "is uniquely described by":
 *   1. PDE weak forms (domain, boundary, stabilization)     -> fem_problem.terms[] (form ids below)
 *   2. linearization, complete gradient of nonlinear terms   -> fixed device integrands per form
 *   3. element type and order                                 -> fem_problem.etype / order
 *   4. quadrature order or scheme                             -> fem_problem.quad_order
 *   5. temporal discretization scheme                         -> fem_problem.time
 *   6. the numbering of variables                             -> fixed: κ-major, g(κ,α) = κ·N + α
 *      (Block B-3: α'(κ,α) = (κ-1)α̂ + α, 0-based here; readings L2/L3 in DESIGN.md)
 * "which the kernel 'simply' assembles".  The four calls of the hot path are
 * fem_mesh_create (Block B-1 input), fem_pattern_build (B-1 item 4 + B-4 as CSR + slot map),
 * fem_assemble_matrix (D-3) and fem_assemble_residual (D-2).
 *
 * Conventions
 *  - 0-based indices.  Arrays are plain pointers; which side (host/device) is stated per argument.
 *  - Stream arguments are a cudaStream_t passed as void* (NULL = legacy default stream).
 *    Assembly calls are stream-ordered and never synchronize the host.
 *  - Every function returns 0 on success or a negative FEM_E* code; fem_last_error() returns a
 *    thread-local message for the last failure.  No C++ exception crosses the ABI; nothing aborts.
 *  - Device-detected errors (det J <= 0 at a quadrature point) set a per-mesh device error
 *    word read by fem_get_status (which synchronizes the stream).
 */
#ifndef LIBFEM_H
#define LIBFEM_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- error codes */
#define FEM_OK 0
#define FEM_E_INVALID_ARG (-1)
#define FEM_E_UNSUPPORTED (-2)      /* element/order/quadrature/form combination not built      */
#define FEM_E_INDEX_OVERFLOW (-3)   /* a count exceeds the index width (int32 columns/slots)      */
#define FEM_E_INVERTED_ELEMENT (-4) /* det J <= 0 at some quadrature point                */
#define FEM_E_NAN (-5)              /* a NaN / breakdown in an iterative solve             */
#define FEM_E_CUDA (-6)
#define FEM_E_OOM (-8)

/* ---- element types (reading L7: VTK node orders; reference simplex / [-1,1]^3 cube) */
#define FEM_TRI 1 /* order 1: 3 nodes                                   */
#define FEM_TET 2 /* order 1: 4 nodes; order 2: 10 nodes (VTK edge order) */
#define FEM_HEX 4 /* order 1: 8 nodes; order 2: 27-node Lagrange cube (NEXT-2)          */
#define FEM_HEX_SERENDIPITY 5 /* order 2: 20-node serendipity cube (NEXT-2)            */
/* Quadratic cube node order (reading L28): 8 corners as the Q1 hex, the 12 edge midpoints of VTK's
 * quadratic hexahedron (0,1),(1,2),(2,3),(3,0),(4,5),(5,6),(6,7),(7,4),(0,4),(1,5),(2,6),(3,7), then for
 * the 27-node cube the 6 face centres in facet order x-,x+,y-,y+,z-,z+ and the centre.  Quadrature:
 * quad_order 2 or 3 Gauss-Legendre points per axis.  Facets are integrated over all element nodes (L18). */

/* ---- physics (κ̂ = number of scalar basic variables, reading L2/L3) */
#define FEM_THERMAL 1    /* κ̂ = 1: T  */
#define FEM_ELASTICITY 2 /* κ̂ = dim: d_1..d_dim  */
#define FEM_NS 3         /* κ̂ = dim+1: u_1..u_dim, p (3D; Rm carries −μ u_i,kk) */

/* ---- weak forms: the paper's named groups; params[] layout per form */
#define FEM_WF_THERMAL_DOMAIN 0   /* -C(T,T_t) - k(T_,i,T_,i) + (T,s)    P:821,832 params {C, k, s, source_kind(0 const, 1 s·Π sin(π x_d))} */
#define FEM_WF_THERMAL_CONV_RAD 1 /* h(T,T_env-T) + e_m σ^b(T,T_env^4-T^4) P:822,834 params {h, T_env, e_m, σ^b} */
#define FEM_WF_THERMAL_FIX 2      /* h_p(T,T_fix-T) + k(T, n_i T_,i)     P:823,835 params {h_p, T_fix, k} */
#define FEM_WF_ELAST_DOMAIN 3     /* -(ε_ij, σ_ij)                       P:904,920 params {E, ν} */
#define FEM_WF_ELAST_FIX_ALL 4    /* τ(d_i, d^w_i - d_i)                 P:906,921 params {τ, d^w_1, d^w_2, d^w_3} */
#define FEM_WF_ELAST_FIX_D1 5     /* τ(d_1, d^w_1 - d_1)                 P:922     params {τ, d^w_1} */
#define FEM_WF_ELAST_LOAD 6       /* (d_i, σ^l_ij n_j)                   P:905,923 params {σ^l_11..σ^l_33 row-major} */
#define FEM_WF_NS_DOMAIN 7        /* NS_domain = BASE + SUPG             P:982-983,1003-1008,1022 params {ρ, μ, τ^m, τ^c} */
#define FEM_WF_NS_BND_INFLOW 8    /* BASE + INFLOW, u^w of P:1050        P:988-990,1009-1013,1023 params {ρ, μ, τ^b, U, H} */
#define FEM_WF_NS_BND_OUTFLOW 9   /* BASE + OUTFLOW                      P:991,1015,1024 params {ρ, μ} */
#define FEM_WF_NS_BND_FIX 10      /* BASE + FIX                          P:992,1017-1018,1025 params {ρ, μ, τ^b} */

/* ---- scatter modes ("(atomic) increment") — determinism is part of the mode, not a setting:
 * FEM_SCATTER_ATOMIC     element-parallel, fp64 atomicAdd into values/rhs; summation order varies run to run.
 * FEM_SCATTER_COLOURED   element colours (no two elements of a colour share a point) in fixed order, plain
 *                        read-modify-write: bit-identical run to run.
 * FEM_SCATTER_TILED      owner gather: each CTA owns a set of points and sums every contribution to their rows
 *                        in shared memory in a FIXED order (per-row turns in record order, or colour runs), then
 *                        writes every owned row once (no clear pass; accumulate must be 0): bit-identical run to
 *                        run.  Q1-hex elasticity on lattice meshes takes the z-sweep schedule, other meshes
 *                        node tiles.  Residual-only calls on tetrahedra use the coloured element pass (cheaper
 *                        than the tiles for rows alone; still deterministic).  FEM_E_UNSUPPORTED (never a silent
 *                        fallback) for elements without a tile kernel (quadratic cubes) or a tile point touched
 *                        by more than 255 visits.  Calls on one pattern use its schedule's scratch (ring
 *                        records; on renumbered lattice meshes a lattice-ordered state copy): issue them on
 *                        one stream (or otherwise in order).
 * FEM_SCATTER_TILED_UNORDERED  owner gather with shared-memory fp64 atomics where a kernel has them (P2 and
 *                        NS tets, generic tiles; hex as TILED): faster, summation order varies run to run.
 *                        Residual-only calls on tetrahedra use the atomic element pass.
 * FEM_SCATTER_STORED     element-stored gather (D-2/D-3 split over HBM): every element writes its whole local
 *                        block and residual into a scratch owned by the pattern, then every CSR entry sums the
 *                        blocks of the elements that contain its two points in ELEMENT ORDER and every row its
 *                        elements' residual rows: no atomics, bit-identical run to run, complete rows written
 *                        (accumulate must be 0).  Needs fem_pattern_stored_prepare first (FEM_E_INVALID_ARG
 *                        otherwise).  Every element type and physics.  The element scratch belongs to the
 *                        pattern: issue the calls on one pattern on one stream. */
#define FEM_SCATTER_ATOMIC 0
#define FEM_SCATTER_COLOURED 1
#define FEM_SCATTER_TILED 2
#define FEM_SCATTER_TILED_UNORDERED 3
#define FEM_SCATTER_STORED 4

#define FEM_TIME_STATIC 0
#define FEM_TIME_GENALPHA 1

typedef struct {
  int kind;   /* FEM_TIME_STATIC (ν̂ = 0, c1 := 1, reading L12) or FEM_TIME_GENALPHA            */
  int nu_hat; /* highest time-derivative order carried by the state (0..2)                      */
  double dt, b1, b2, c1, c2, c3; /* Eq. time_constraints/time_effective               */
} fem_time_scheme;

#define FEM_MAX_TERMS 16
#define FEM_MAX_PARAMS 16
typedef struct {
  int form;   /* FEM_WF_*                                     */
  int region; /* -1 = domain Ω, k >= 0 = boundary facet set k */
  double params[FEM_MAX_PARAMS];
} fem_term;

typedef struct {
  int etype, order;
  int quad_order; /* hex: Gauss-Legendre points per axis (1..3); tri/tet: exactness degree (1..2) */
  int physics;    /* FEM_THERMAL | FEM_ELASTICITY | FEM_NS                                        */
  fem_time_scheme time;
  int n_terms;
  fem_term terms[FEM_MAX_TERMS];
} fem_problem;

typedef struct fem_mesh_s* fem_mesh_t;
typedef struct fem_pattern_s* fem_pattern_t;

/* fem_mesh_create — Block B-1 input: the element→control-point map α(β^el, β^el_cp).
 *  prob        host; element type/order/physics/quadrature (validated here).
 *  dim         2 (FEM_TRI) or 3.
 *  n_nodes     N, number of control points (global numbering).
 *  coords      HOST, float64 SoA [dim][N].
 *  n_elems     E; conn HOST int32 SoA [n_loc][E] (VTK local order), values in [0, N).
 *  bsets       n_bsets boundary facet sets; set k = (bset_elem[k][m], bset_facet[k][m]) HOST arrays of
 *              length bset_len[k]: element id and local facet (reading L8).
 *  own_lo/hi   rows assembled by this mesh: control points [own_lo, own_hi) (multi-GPU partition;
 *              [0, N) on one GPU).  Elements must include every element touching an owned point.
 *  stream      used for the host→device copies; the call synchronizes it before returning.
 * The library copies everything into its own device memory (freed by fem_mesh_destroy), builds the
 * deterministic element colouring and the node-tile schedule.  Errors: INVALID_ARG (sizes/ids out of
 * range), UNSUPPORTED (combination), OOM, CUDA. */
int fem_mesh_create(const fem_problem* prob, int dim, int64_t n_nodes, const double* coords,
                    int64_t n_elems, const int32_t* conn, int n_bsets, const int64_t* bset_len,
                    const int32_t* const* bset_elem, const int8_t* const* bset_facet,
                    int64_t own_lo, int64_t own_hi, void* stream, fem_mesh_t* out);

/* fem_pattern_build — Block B-1 item 4 ("each unique pair is only kept once"), A-3 symbol
 * pairs (all (κ0,κλ), reading L6) and B-4 realised as a CSR matrix with ascending columns:
 * row r = κ0·n_own + (α1 - own_lo) holds columns κλ·N + α2 for κλ ascending, α2 ascending.  Also
 * builds the element→slot map slot_s[(a·n_loc+b)·E + e] = position of (α(e,a), α(e,b)) in the
 * scalar-graph CSR (rowptr_s over owned points, colidx_s), -1 if α(e,a) is not owned.
 * Synchronizes `stream` once (to read nnz).  Outputs (host): *n_rows = κ̂·n_own, *nnz.
 * Errors: INDEX_OVERFLOW (scalar nnz >= 2^31 or κ̂·N >= 2^31), OOM, CUDA. */
int fem_pattern_build(fem_mesh_t mesh, void* stream, fem_pattern_t* out, int64_t* n_rows,
                      int64_t* nnz);
int64_t fem_pattern_nnz_s(fem_pattern_t pat);

/* fem_pattern_export — copy the library-owned pattern into caller DEVICE buffers (any may be NULL):
 * rowptr int64[n_rows+1], colidx int32[nnz], slot_s int32[n_loc²·E], rowptr_s int64[n_own+1],
 * colidx_s int32[nnz_s].  Stream-ordered. */
int fem_pattern_export(fem_pattern_t pat, int64_t* rowptr, int32_t* colidx, int32_t* slot_s,
                       int64_t* rowptr_s, int32_t* colidx_s, void* stream);

/* fem_assemble_matrix — D-3: values[β^sp] (+)= Σ_γ w_γ f_ν (D0 N̄_a D_λ N_b) ∂L^a/∂λ,
 * f_ν = c_{ν+1}/Π_{β'≤ν}(b_β' Δt) (Eq. gen_alpha; reading L13).
 *  state   DEVICE float64 [ν̂+1][κ̂][N]: effective values ∂_t^ν φ̃ (D-1 output).
 *  values  DEVICE float64 [nnz] (caller-owned).  accumulate = 0: cleared first ("cleared first",
 *          P:441); 1: added to the existing contents (not allowed with FEM_SCATTER_TILED).
 *  scatter FEM_SCATTER_*.  prob must match the mesh's element/physics.  No host sync, no allocation. */
int fem_assemble_matrix(fem_mesh_t mesh, fem_pattern_t pat, const fem_problem* prob,
                        const double* state, double* values, int accumulate, int scatter,
                        void* stream);

/* fem_assemble_residual — D-2: rhs[g(κ0,α(e,a)) local] (+)= Σ_γ w_γ (D0 N̄_a) L^a(...).
 *  rhs DEVICE float64 [κ̂·n_own]; other arguments as fem_assemble_matrix.  `pat` may be NULL for the
 *  atomic and coloured modes (the residual needs no sparsity pattern). */
int fem_assemble_residual(fem_mesh_t mesh, fem_pattern_t pat, const fem_problem* prob,
                          const double* state, double* rhs, int accumulate, int scatter,
                          void* stream);

/* fem_assemble_system — D-2 and D-3 in one pass over the elements (one Newton linearisation). */
int fem_assemble_system(fem_mesh_t mesh, fem_pattern_t pat, const fem_problem* prob,
                        const double* state, double* values, double* rhs, int accumulate,
                        int scatter, void* stream);

/* fem_residual_norms — norms_dev[0] = Σ_i d_i², norms_dev[1] = max_i |d_i| over the κ̂·n_own owned rows
 * (the D-2 convergence test).  DEVICE output, stream-ordered, no host sync.  Fixed grid (4 × SM
 * count) and fixed summation order: bit-identical run to run on a given device.  NaN propagates into both
 * norms (a NaN residual never passes a ‖d‖ < tol test).  Uses per-mesh scratch: calls on one mesh must
 * not run concurrently on different streams.  Multi-GPU: all-reduce [0] with SUM and [1] with MAX. */
int fem_residual_norms(fem_mesh_t mesh, const double* rhs, double* norms_dev, void* stream);

/* fem_linearize_host — end-to-end call with HOST buffers: copies the state from (pinned) host memory
 * into library scratch, runs fem_assemble_system into the DEVICE values/rhs, computes the residual
 * norms and copies them to norms_host[2]; synchronizes the stream before returning. */
int fem_linearize_host(fem_mesh_t mesh, fem_pattern_t pat, const fem_problem* prob,
                       const double* state_host, double* values, double* rhs, double* norms_host,
                       int scatter, void* stream);

/* fem_linearize_host_async — fem_linearize_host without the final synchronization, pipelined: the state
 * is staged through two library-owned device buffers on a library-owned copy stream, so the host->device
 * copy of this call overlaps the assembly of the previous call on `stream`.  norms_host (pinned) is
 * valid, and state_host may be modified, once `stream` has completed this call's work (the caller syncs).
 * values / rhs are overwritten by every call in stream order. */
int fem_linearize_host_async(fem_mesh_t mesh, fem_pattern_t pat, const fem_problem* prob,
                             const double* state_host, double* values, double* rhs, double* norms_host,
                             int scatter, void* stream);

/* ---- NEXT-4: the paper's COO view (B-4) and workpiece offsets ------------
 * fem_pattern_export_coo — for every entry in sparse-ID order (symbol pairs (κ₀, κ_λ) then control-point
 *   pairs (α₁, α₂), both lexicographic, reading L4): I[id] = row_offset + κ₀ N + α₁, J[id] = row_offset +
 *   κ_λ N + α₂ (the workpiece's n^dense, as row_offset) and csr_index[id] = the entry's position in
 *   the CSR values.  DEVICE int64 outputs of nnz entries (any may be NULL, not all); a multi-workpiece
 *   system passes each workpiece's arrays at its n^sp.  Stream-ordered, no sync.
 * fem_gather — dst[i] = src[index[i]] (DEVICE), e.g. the CSR values in sparse-ID order. */
int fem_pattern_export_coo(fem_pattern_t pat, int64_t row_offset, int64_t* I, int64_t* J, int64_t* csr_index,
                           void* stream);
int fem_gather(int64_t n, const int64_t* index, const double* src, double* dst, void* stream);

/* ---- NEXT-3: generalized-α time stepping around the assembly (Block C P:404-417, D-1 P:421-424,
 * D-4 P:459-465; Eqs. time_constraints/time_effective P:226-236).  All arrays DEVICE float64, layout
 * [ν][n] (ν = 0..ts->nu_hat, n = rows of the system = κ̂N, κ-major), caller-owned, stream-ordered, no
 * host sync.  phi0 = committed values ∂_t^ν φ, incr = increments Δ∂_t^ν φ, eff = effective values
 * ∂_t^ν φ̃ (the `state` input of the assembly calls).  Values are the correctly rounded left-to-right
 * evaluation of the expressions below (no FMA contraction).  Errors: INVALID_ARG (ts NULL, kind not
 * FEM_TIME_GENALPHA, nu_hat outside 0..2, dt <= 0, b_ν = 0 for a ν <= nu_hat that divides, n < 0,
 * NULL arrays), CUDA.
 *
 * fem_time_init — Block C.  C-1: phi0[ν] += incr[ν]; C-2: incr[ν̂] = 0; C-3 (reading L14, Eq.
 *   time_constraints): incr[ν] = dt·(phi0[ν+1] + b_{ν+1}·incr[ν+1]) for ν = ν̂-1 … 0.  If eff != NULL
 *   also writes D-1 of the first sub-step (fused, same pass).
 * fem_time_effective — D-1: eff[ν] = c_{ν+1}·incr[ν] + phi0[ν].
 * fem_time_increment — D-4 (reading L13): incr[ν] += delta_sub / Π_{β'=1}^{ν}(b_β'·dt), delta_sub [n]
 *   the solve's sub-step increment Δ_sub φ; if eff != NULL (then phi0 is required) also writes D-1 of the
 *   next sub-step in the same pass. */
int fem_time_init(const fem_time_scheme* ts, int64_t n, double* phi0, double* incr, double* eff, void* stream);
int fem_time_effective(const fem_time_scheme* ts, int64_t n, const double* phi0, const double* incr, double* eff,
                       void* stream);
int fem_time_increment(const fem_time_scheme* ts, int64_t n, const double* delta_sub, double* incr,
                       const double* phi0, double* eff, void* stream);

/* fem_get_status — synchronizes `stream`; returns 0 or FEM_E_INVERTED_ELEMENT (bad_elem = an
 * offending element id, else -1).  Resets the device error word. */
int fem_get_status(fem_mesh_t mesh, void* stream, int64_t* bad_elem);

/* fem_mesh_info — host query: n_loc, kappa_hat, number of colours, number of node tiles. */
int fem_mesh_info(fem_mesh_t mesh, int* n_loc, int* kappa_hat, int* n_colours, int64_t* n_tiles);

/* fem_pattern_info — host query of the node-tile schedule built with the pattern:
 * out[0] tiles (sweep: steps), [1] largest tile (points; sweep: ring rows), [2] largest accumulator
 * (doubles), [3] largest packed record (bytes), [4] largest halo (points), [5] element visits in total,
 * [6] largest per-tile visit count, [7] total packed record bytes, [8] schedule: 0 node tiles, 1 z-sweep,
 * -1 none (tiled calls return FEM_E_UNSUPPORTED).  out has 9 entries. */
int fem_pattern_info(fem_pattern_t pat, int64_t* out9);

/* ---- NEXT-1: the linear solve of the Newton sub-step, D-4 ----------------
 * The linearisation K Δφ = -d of d(φ) = 0 is solved on the CSR of fem_pattern_build.
 *
 * fem_spmv — y = alpha·K·x + beta·y for the CSR K (rowptr int64 [n_rows+1], colidx int32 [nnz], values
 *   fp64 [nnz], all DEVICE; x, y DEVICE fp64, x indexed by column).  Stream-ordered, no sync.  A warp owns
 *   32 consecutive rows; the per-row sum order is fixed (bit-identical run to run).
 *   Single-GPU pattern (columns index the same vector as rows).  FEM_E_INVALID_ARG on NULL / n_rows < 0.
 *
 * fem_cg_work_doubles — size of the caller-owned DEVICE work buffer of fem_cg_solve, in doubles.
 *
 * fem_cg_solve — Jacobi-preconditioned conjugate gradients for K x = b, run on (s K) x = s b with
 *   s = spd_sign = ±1 chosen by the caller so that s K is symmetric positive definite (thermal and
 *   elasticity with penalty boundary terms: s = -1, reading L17).  x (DEVICE) holds the initial guess on
 *   entry and the solution on exit; b DEVICE.  Stops when ||r||_2 <= rtol ||r_0||_2 or after max_iter
 *   iterations; the convergence test is read back every check_every iterations (<= 0: 16), so the call
 *   synchronizes `stream` (the only host syncs).  iters_out / relres_out (host, may be NULL) receive the
 *   iteration count and ||r||/||r_0||.  Every reduction sums in fixed order: bit-identical run to run.
 *   A zero p·Kp or r·z freezes the iterate instead of dividing by zero.  Not converging within max_iter
 *   is NOT an error: check relres_out against rtol.  Errors: FEM_E_INVALID_ARG for bad arguments or a
 *   non-positive diagonal of s K (not SPD); FEM_E_NAN when the residual becomes NaN. */
/* fem_pattern_stored_prepare — one-time setup of FEM_SCATTER_STORED for this pattern: the per-slot
 *   contribution lists (a stable device radix sort of the slot map: 4 B per (element, a, b) with an owned
 *   row), the diagonal slot of every owned row, and the element scratch — residual rows E·n_loc·κ̂ doubles,
 *   and with with_matrix != 0 the element blocks E·n_loc²·κ̂² doubles (c3: 5.3 GB).  Library-owned, freed by
 *   fem_pattern_destroy; a second call only adds what is missing.  Synchronizes `stream`.  Errors:
 *   FEM_E_INDEX_OVERFLOW when E·n_loc² >= 2^32, FEM_E_OOM, FEM_E_CUDA. */
int fem_pattern_stored_prepare(fem_pattern_t pat, int with_matrix, void* stream);
/* fem_pattern_csr — the pattern's own DEVICE CSR arrays (library-owned, valid until fem_pattern_destroy,
 *   read-only): rowptr int64 [n_rows+1], colidx int32 [nnz] (global column ids; *col_offset = own_lo, 0
 *   on a single GPU).  No copy, no sync. */
int fem_pattern_csr(fem_pattern_t pat, const int64_t** rowptr, const int32_t** colidx, int64_t* col_offset);
/* fem_bicgstab_solve — Jacobi-preconditioned BiCGStab for K x = b with a non-symmetric K (the thermal FIX
 *   term k N_a n·∇T, and the NS forms make K non-symmetric).  Same conventions as
 *   fem_cg_solve (DEVICE vectors, caller-owned work of fem_bicgstab_work_doubles(n_rows) doubles, host
 *   syncs every check_every iterations, fixed-order reductions).  FEM_E_INVALID_ARG for a zero diagonal;
 *   FEM_E_NAN on breakdown. */
int64_t fem_bicgstab_work_doubles(int64_t n_rows);
int fem_bicgstab_solve(int64_t n_rows, const int64_t* rowptr, const int32_t* colidx, const double* values,
                       const double* b, double* x, int max_iter, double rtol, int check_every, double* work,
                       int* iters_out, double* relres_out, void* stream);
/* fem_vec_axpby — y = alpha·x + beta·y over n DEVICE doubles, each product and the sum correctly rounded
 *   (no FMA contraction).  The Newton update φ ← φ − Δφ of D-4 and sign flips around the
 *   solves run here, not in the binding.  Stream-ordered, no sync.  INVALID_ARG on n < 0 / NULL. */
int fem_vec_axpby(int64_t n, double alpha, const double* x, double beta, double* y, void* stream);
/* fem_gmres_solve — restarted GMRES(restart) with right point-block-Jacobi preconditioning for K x = b with
 *   a non-symmetric, indefinite K: the stabilised NS saddle point, where Jacobi-BiCGStab diverges.
 *   The κ̂ x κ̂ diagonal block of every control point (rows κ·n_points + α of the κ-major numbering, B-3
 *   P:368-375) is inverted once (Gauss-Jordan, partial pivoting); n_rows must equal n_points·kappa_hat
 *   (single-GPU pattern, kappa_hat 1..4).  Arnoldi by classical Gram-Schmidt with re-orthogonalisation;
 *   every inner product is a fixed-order reduction (bit-identical run to run); the host solves the small
 *   Hessenberg problem and syncs once per Arnoldi step.  Stops when the true ||b - K x|| <= rtol·||b||
 *   (within 10x of the recurrence's estimate) or after max_iter Arnoldi steps; x holds the initial guess on
 *   entry.  pin_row >= 0: solve with that row and column replaced by the identity and the pinned unknown held
 *   at its initial value (the gauge of a singular K: the paper's NS forms determine the pressure only up to a
 *   constant, reading L29 — pin one pressure row, e.g. dim·n_points); -1: no pin.  work: caller-owned DEVICE
 *   buffer of fem_gmres_work_doubles(n_rows, n_points, kappa_hat, restart) doubles.  Errors: INVALID_ARG (bad
 *   sizes, singular point block), NAN (breakdown). */
int64_t fem_gmres_work_doubles(int64_t n_rows, int64_t n_points, int kappa_hat, int restart);
int fem_gmres_solve(int64_t n_rows, const int64_t* rowptr, const int32_t* colidx, const double* values,
                    int64_t n_points, int kappa_hat, const double* b, double* x, int restart, int max_iter,
                    double rtol, int64_t pin_row, double* work, int* iters_out, double* relres_out, void* stream);
int fem_spmv(int64_t n_rows, const int64_t* rowptr, const int32_t* colidx, const double* values,
             const double* x, double* y, double alpha, double beta, void* stream);
int64_t fem_cg_work_doubles(int64_t n_rows);
int fem_cg_solve(int64_t n_rows, const int64_t* rowptr, const int32_t* colidx, const double* values,
                 const double* b, double* x, double spd_sign, int max_iter, double rtol, int check_every,
                 double* work, int* iters_out, double* relres_out, void* stream);

void fem_pattern_destroy(fem_pattern_t pat);
void fem_mesh_destroy(fem_mesh_t mesh);
const char* fem_last_error(void);
int fem_version(void);

#ifdef __cplusplus
}
#endif
#endif
