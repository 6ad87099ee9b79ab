/* oracle/fem_oracle.h — TEST INFRASTRUCTURE ONLY (not part of the product path).
 *
 * A plain, slow, serial fp64 CPU assembler of the MetaFEM linear system K x = d
 * (arXiv:2111.03541, §2.2 Blocks B and D).  Only tests/, the
 * __graft_entry__.smoke() check and bench.py's cpu_baseline / --impl reference legs may load it.
 * It shares no code, header, table or constant with paper_2111_03541_b200/ (the CUDA path).
 *
 * Conventions: 0-based indices; κ-major global numbering g(κ,α) = κ·N + α (B-3, reading L2/L3);
 * CSR with ascending columns (reading L4); SoA coords [dim][N], conn [n_loc][E].
 */
#ifndef FEM_ORACLE_H
#define FEM_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { OR_TRI = 1, OR_TET = 2, OR_HEX = 4, OR_HEXS = 5 }; /* HEXS: 20-node serendipity cube (order 2) */
enum { OR_THERMAL = 1, OR_ELASTICITY = 2, OR_NS = 3 };
enum {
  OR_THERMAL_DOMAIN = 0, OR_THERMAL_CONV_RAD = 1, OR_THERMAL_FIX = 2,
  OR_ELAST_DOMAIN = 3, OR_ELAST_FIX_ALL = 4, OR_ELAST_FIX_D1 = 5, OR_ELAST_LOAD = 6,
  OR_NS_DOMAIN = 7, OR_NS_BND_INFLOW = 8, OR_NS_BND_OUTFLOW = 9, OR_NS_BND_FIX = 10
};

#define OR_MAX_TERMS 16
typedef struct { int form; int region; double p[16]; } or_term;

typedef struct {
  int physics, etype, order, quad_order, dim;
  int nu_hat;                       /* 0 static, >=1 generalized-alpha operands present      */
  double dt, b1, b2, c1, c2, c3;    /* P:226-236; static: c1 = 1                              */
  int n_terms;
  or_term terms[OR_MAX_TERMS];
} or_problem;

typedef struct or_system or_system;

/* Assemble the rows of K and d whose control point is selected by row_mask (NULL = all nodes).
 * state: [nu_hat+1][kappa_hat][N].  Returns NULL only on allocation failure. */
or_system* or_assemble(const or_problem* prob, int64_t n_nodes, const double* coords,
                       int64_t n_elems, const int32_t* conn, int n_bsets, const int64_t* bset_len,
                       const int32_t* const* bset_elem, const int8_t* const* bset_facet,
                       const double* state, const uint8_t* row_mask, int want_matrix,
                       int want_residual);
int     or_status(const or_system* s, int64_t* bad_elem); /* 0 ok, -4 inverted element, -2 unsupported */
int64_t or_n_sel_nodes(const or_system* s);
int64_t or_n_rows(const or_system* s);
int64_t or_nnz(const or_system* s);
int64_t or_nnz_s(const or_system* s);
/* rows: global row id of each selected row (κ0-major over selected nodes). */
void or_get(const or_system* s, int64_t* sel_nodes, int64_t* rows, int64_t* rowptr, int32_t* colidx,
            double* values, double* rhs, double* abs_d, int64_t* rowptr_s, int32_t* colidx_s);
/* slot_s[(a*n_loc+b)*E + e] = scalar-CSR position of (α(e,a), α(e,b)), -1 if α(e,a) not selected */
void or_get_slot(const or_system* s, const int32_t* conn, int32_t* slot_s);
void or_free(or_system* s);

/* Probe: quadrature-point data of element e (facet < 0: volume rule; else facet `facet`).
 * Outputs (capacity 64 points): x [nq][3], w [nq], n [nq][3], N [nq][n_loc], G [nq][n_loc][3],
 * H [nq][n_loc][3][3] (physical second derivatives ∂²N_a/∂x_i∂x_j; may be NULL).
 * Returns nq, or a negative error. */
int or_qp_data(const or_problem* prob, int64_t n_nodes, const double* coords, int64_t n_elems,
               const int32_t* conn, int64_t e, int facet, double* x, double* w, double* n,
               double* N, double* G, double* H);

#ifdef __cplusplus
}
#endif
#endif
