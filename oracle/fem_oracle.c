/* oracle/fem_oracle.c — TEST INFRASTRUCTURE ONLY.  Not part of the product path.
 *
 * Plain, slow, serial fp64 reference assembler for the MetaFEM system K x = d
 * (arXiv:2111.03541).  Written from PAPER.md, independently of paper_2111_03541_b200/:
 * its own shape functions, quadrature tables, geometry, integrands and sparsity code.
 * Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline / --impl reference)
 * may load it.  Every function names the passage it follows:
 *   P:n = /root/reference/PAPER.md line n;  Lxx = reading xx in DESIGN.md §4.
 *
 * What is computed (the plain definition, no blocking/fusion/reordering):
 *   d_{g(κ0,α(e,a))} += Σ_γ w_γ  r(a,κ0; fields at x_γ)                       (D-2)
 *   K_{g(κ0,α(e,a)), g(κλ,α(e,b))} += Σ_γ w_γ f_ν ∂r(a,κ0)/∂(operand)·D N_b   (D-3)
 * with w_γ the physical weight (L1), f_ν = c_{ν+1}/Π_{β'≤ν}(b_β' Δt) (Eq. gen_alpha, P:256-258,
 * P:452; L13), and the tangent evaluated as the directional derivative of the residual along the
 * trial function ("complete gradient"): every operand is replaced by its derivative
 * w.r.t. the control value (value → f_ν N_b, gradient → f_ν G_b), product rule by hand.
 */
#include "fem_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#ifndef M_PI
#define M_PI 3.14159265358979323846
#endif

#define MAXN 27 /* nodes per element (Q2 hex)                     */
#define MAXK 4  /* basic-variable components κ̂ (NS: u1,u2,u3,p) */
#define MAXQ 64

/* ------------------------------------------------------------------ reference elements (L7) */
static int n_loc_of(int etype, int order) {
  if (etype == OR_TRI && order == 1) return 3;
  if (etype == OR_TET && order == 1) return 4;
  if (etype == OR_TET && order == 2) return 10;
  if (etype == OR_HEX && order == 1) return 8;
  if (etype == OR_HEX && order == 2) return 27; /* Lagrange cube of order 2      */
  if (etype == OR_HEXS && order == 2) return 20; /* serendipity cube of order 2   */
  return -1;
}
static int n_vert_of(int etype) { return etype == OR_TRI ? 3 : (etype == OR_TET ? 4 : 8); }

static const double HEX_SIGN[8][3] = {{-1, -1, -1}, {1, -1, -1}, {1, 1, -1}, {-1, 1, -1},
                                      {-1, -1, 1},  {1, -1, 1},  {1, 1, 1},  {-1, 1, 1}};
static const int TET_EDGE[6][2] = {{0, 1}, {1, 2}, {0, 2}, {0, 3}, {1, 3}, {2, 3}};

/* Quadratic cubes (NEXT-2; reading L28): reference coordinates r_a ∈ {-1,0,1}³ of the nodes — corners in
 * VTK order (L7), the 12 edge midpoints of VTK's quadratic hexahedron ((0,1),(1,2),(2,3),(3,0),(4,5),(5,6),
 * (6,7),(7,4),(0,4),(1,5),(2,6),(3,7)), then (27-node only) the face centres in facet order x-,x+,y-,y+,z-,z+
 * (L8) and the centre. */
static const int HEX_EDGE[12][2] = {{0, 1}, {1, 2}, {2, 3}, {3, 0}, {4, 5}, {5, 6},
                                    {6, 7}, {7, 4}, {0, 4}, {1, 5}, {2, 6}, {3, 7}};
static void quad_cube_node(int a, double* r) {
  if (a < 8) { for (int d = 0; d < 3; d++) r[d] = HEX_SIGN[a][d]; return; }
  if (a < 20) {
    for (int d = 0; d < 3; d++) r[d] = 0.5 * (HEX_SIGN[HEX_EDGE[a - 8][0]][d] + HEX_SIGN[HEX_EDGE[a - 8][1]][d]);
    return;
  }
  r[0] = r[1] = r[2] = 0.0;
  if (a < 26) r[(a - 20) / 2] = ((a - 20) & 1) ? 1.0 : -1.0;
}
/* 1D quadratic Lagrange factor on the nodes {-1, 0, 1}: value, first and second derivative at t */
static void lag1d(double r, double t, double* v, double* d1, double* d2) {
  if (r < -0.5) { *v = 0.5 * t * (t - 1.0); *d1 = t - 0.5; *d2 = 1.0; }
  else if (r > 0.5) { *v = 0.5 * t * (t + 1.0); *d1 = t + 0.5; *d2 = 1.0; }
  else { *v = 1.0 - t * t; *d1 = -2.0 * t; *d2 = -2.0; }
}
/* N = c Π_d f_d(ξ_d) with per-axis factors (value v, derivatives d1, d2): gradient and Hessian. */
static void product3(double c, const double* v, const double* d1, const double* d2, double* N, double* g,
                     double h[3][3]) {
  *N = c * v[0] * v[1] * v[2];
  for (int d = 0; d < 3; d++) {
    int e1 = (d + 1) % 3, e2 = (d + 2) % 3;
    g[d] = c * d1[d] * v[e1] * v[e2];
    if (h) h[d][d] = c * d2[d] * v[e1] * v[e2];
  }
  if (h)
    for (int d = 0; d < 3; d++)
      for (int e = 0; e < 3; e++)
        if (d != e) h[d][e] = c * d1[d] * d1[e] * v[3 - d - e];
}
/* 27-node Lagrange cube: tensor product of the 1D quadratics. */
static void shape_q2(const double* xi, double* N, double dN[][3], double (*d2N)[3][3]) {
  for (int a = 0; a < 27; a++) {
    double r[3], v[3], d1[3], d2[3];
    quad_cube_node(a, r);
    for (int d = 0; d < 3; d++) lag1d(r[d], xi[d], &v[d], &d1[d], &d2[d]);
    product3(1.0, v, d1, d2, &N[a], dN[a], d2N ? d2N[a] : NULL);
  }
}
/* 20-node serendipity cube, the textbook basis:
 *   corner (r ∈ {±1}³): N = 1/8 Π_d (1 + r_d ξ_d) · (Σ_d r_d ξ_d − 2);
 *   edge midpoint with r_m = 0: N = 1/4 (1 − ξ_m²) Π_{d≠m} (1 + r_d ξ_d). */
static void shape_s2(const double* xi, double* N, double dN[][3], double (*d2N)[3][3]) {
  for (int a = 0; a < 20; a++) {
    double r[3], v[3], d1[3], d2[3];
    quad_cube_node(a, r);
    if (a < 8) {
      double f, fg[3], fh[3][3];
      for (int d = 0; d < 3; d++) { v[d] = 1.0 + r[d] * xi[d]; d1[d] = r[d]; d2[d] = 0.0; }
      product3(0.125, v, d1, d2, &f, fg, fh);
      double sv = r[0] * xi[0] + r[1] * xi[1] + r[2] * xi[2] - 2.0;
      N[a] = f * sv;
      for (int d = 0; d < 3; d++) dN[a][d] = fg[d] * sv + f * r[d];
      if (d2N)
        for (int d = 0; d < 3; d++)
          for (int e = 0; e < 3; e++) d2N[a][d][e] = fh[d][e] * sv + fg[d] * r[e] + fg[e] * r[d];
    } else {
      for (int d = 0; d < 3; d++) {
        if (r[d] == 0.0) { v[d] = 1.0 - xi[d] * xi[d]; d1[d] = -2.0 * xi[d]; d2[d] = -2.0; }
        else { v[d] = 1.0 + r[d] * xi[d]; d1[d] = r[d]; d2[d] = 0.0; }
      }
      product3(0.25, v, d1, d2, &N[a], dN[a], d2N ? d2N[a] : NULL);
    }
  }
}

/* Lagrange shape functions N_a(ξ), reference gradients ∂N_a/∂ξ_j and (d2N != NULL) reference second
 * derivatives ∂²N_a/∂ξ_j∂ξ_l (φ^h = Σ N_α φ_α; the second derivatives feed μ u_i,kk). */
static void shape(int etype, int order, const double* xi, double* N, double dN[][3], double (*d2N)[3][3]) {
  memset(dN, 0, sizeof(double) * 3 * MAXN);
  if (d2N) memset(d2N, 0, sizeof(double) * 9 * MAXN);
  if (etype == OR_HEX && order == 2) { shape_q2(xi, N, dN, d2N); return; }
  if (etype == OR_HEXS) { shape_s2(xi, N, dN, d2N); return; }
  if (etype == OR_TRI) { /* P1 triangle, vertices (0,0),(1,0),(0,1) */
    N[0] = 1.0 - xi[0] - xi[1]; N[1] = xi[0]; N[2] = xi[1];
    dN[0][0] = -1; dN[0][1] = -1; dN[1][0] = 1; dN[2][1] = 1;
    return;
  }
  if (etype == OR_TET) {
    double L[4] = {1.0 - xi[0] - xi[1] - xi[2], xi[0], xi[1], xi[2]};
    double dL[4][3] = {{-1, -1, -1}, {1, 0, 0}, {0, 1, 0}, {0, 0, 1}};
    if (order == 1) {
      for (int a = 0; a < 4; a++) { N[a] = L[a]; for (int j = 0; j < 3; j++) dN[a][j] = dL[a][j]; }
      return;
    }
    for (int a = 0; a < 4; a++) { /* vertex: L(2L-1) */
      N[a] = L[a] * (2.0 * L[a] - 1.0);
      for (int j = 0; j < 3; j++) dN[a][j] = (4.0 * L[a] - 1.0) * dL[a][j];
      if (d2N)
        for (int j = 0; j < 3; j++)
          for (int l = 0; l < 3; l++) d2N[a][j][l] = 4.0 * dL[a][j] * dL[a][l];
    }
    for (int k = 0; k < 6; k++) { /* edge (p,q): 4 L_p L_q */
      int p = TET_EDGE[k][0], q = TET_EDGE[k][1];
      N[4 + k] = 4.0 * L[p] * L[q];
      for (int j = 0; j < 3; j++) dN[4 + k][j] = 4.0 * (L[p] * dL[q][j] + L[q] * dL[p][j]);
      if (d2N)
        for (int j = 0; j < 3; j++)
          for (int l = 0; l < 3; l++) d2N[4 + k][j][l] = 4.0 * (dL[p][j] * dL[q][l] + dL[q][j] * dL[p][l]);
    }
    return;
  }
  /* Q1 hexahedron on [-1,1]^3: N_a = 1/8 Π_d (1 + s_ad ξ_d) */
  for (int a = 0; a < 8; a++) {
    double f[3];
    for (int d = 0; d < 3; d++) f[d] = 1.0 + HEX_SIGN[a][d] * xi[d];
    N[a] = 0.125 * f[0] * f[1] * f[2];
    dN[a][0] = 0.125 * HEX_SIGN[a][0] * f[1] * f[2];
    dN[a][1] = 0.125 * HEX_SIGN[a][1] * f[0] * f[2];
    dN[a][2] = 0.125 * HEX_SIGN[a][2] * f[0] * f[1];
    if (d2N)
      for (int d = 0; d < 3; d++)
        for (int e = 0; e < 3; e++)
          if (d != e) d2N[a][d][e] = 0.125 * HEX_SIGN[a][d] * HEX_SIGN[a][e] * f[3 - d - e];
  }
}

/* Reference vertex coordinates (for facet parameterisations). */
static void ref_vertex(int etype, int v, double* out) {
  out[0] = out[1] = out[2] = 0.0;
  if (etype == OR_HEX || etype == OR_HEXS) { for (int d = 0; d < 3; d++) out[d] = HEX_SIGN[v][d]; return; }
  if (v >= 1) out[v - 1] = 1.0; /* simplex: v0 = origin, v_k = e_k */
}

/* ------------------------------------------------------------------ quadrature (L9) */
static int gauss1d(int n, double* x, double* w) { /* Gauss-Legendre on [-1,1] */
  if (n == 1) { x[0] = 0.0; w[0] = 2.0; return 1; }
  if (n == 2) { x[0] = -1.0 / sqrt(3.0); x[1] = 1.0 / sqrt(3.0); w[0] = w[1] = 1.0; return 2; }
  if (n == 3) {
    x[0] = -sqrt(0.6); x[1] = 0.0; x[2] = sqrt(0.6);
    w[0] = 5.0 / 9.0; w[1] = 8.0 / 9.0; w[2] = 5.0 / 9.0; return 3;
  }
  return -1;
}
/* triangle rule on the reference triangle {s,t >= 0, s+t <= 1}, exact to `deg` */
static int tri_rule(int deg, double p[][2], double* w) {
  if (deg <= 1) { p[0][0] = p[0][1] = 1.0 / 3.0; w[0] = 0.5; return 1; }
  if (deg == 2) {
    p[0][0] = 1.0 / 6.0; p[0][1] = 1.0 / 6.0;
    p[1][0] = 2.0 / 3.0; p[1][1] = 1.0 / 6.0;
    p[2][0] = 1.0 / 6.0; p[2][1] = 2.0 / 3.0;
    w[0] = w[1] = w[2] = 1.0 / 6.0; return 3;
  }
  return -1;
}
static int vol_rule(int etype, int q, double pts[][3], double* w) {
  memset(pts, 0, sizeof(double) * 3 * MAXQ);
  if (etype == OR_TRI) {
    double p[8][2];
    int n = tri_rule(q, p, w);
    for (int i = 0; i < n; i++) { pts[i][0] = p[i][0]; pts[i][1] = p[i][1]; }
    return n;
  }
  if (etype == OR_TET) {
    if (q <= 1) { pts[0][0] = pts[0][1] = pts[0][2] = 0.25; w[0] = 1.0 / 6.0; return 1; }
    if (q == 2) {
      double a = (5.0 - sqrt(5.0)) / 20.0, b = (5.0 + 3.0 * sqrt(5.0)) / 20.0;
      double P[4][3] = {{a, a, a}, {b, a, a}, {a, b, a}, {a, a, b}};
      for (int i = 0; i < 4; i++) { for (int d = 0; d < 3; d++) pts[i][d] = P[i][d]; w[i] = 1.0 / 24.0; }
      return 4;
    }
    return -1;
  }
  double x[4], ww[4];
  int n = gauss1d(q, x, ww);
  if (n < 0) return -1;
  int m = 0;
  for (int k = 0; k < n; k++)
    for (int j = 0; j < n; j++)
      for (int i = 0; i < n; i++) {
        pts[m][0] = x[i]; pts[m][1] = x[j]; pts[m][2] = x[k];
        w[m] = ww[i] * ww[j] * ww[k]; m++;
      }
  return m;
}

static const int HEX_FACE[6][4] = {{0, 4, 7, 3}, {1, 2, 6, 5}, {0, 1, 5, 4},
                                   {3, 7, 6, 2}, {0, 3, 2, 1}, {4, 5, 6, 7}}; /* L8 */

/* Facet rule: points in element reference coordinates with reference tangents dξ/ds, dξ/dt.
 * "boundary conditions are just the domain physics one dimension lower"; L8. */
static int facet_rule(int etype, int q, int facet, double pts[][3], double* w, double t1[][3],
                      double t2[][3]) {
  memset(pts, 0, sizeof(double) * 3 * MAXQ);
  memset(t1, 0, sizeof(double) * 3 * MAXQ);
  memset(t2, 0, sizeof(double) * 3 * MAXQ);
  if (etype == OR_TRI) { /* edge k = (k, k+1 mod 3), Gauss-Legendre on s in [0,1] */
    if (facet < 0 || facet > 2) return -1;
    double A[3], B[3], x[4], ww[4];
    ref_vertex(etype, facet, A);
    ref_vertex(etype, (facet + 1) % 3, B);
    int n = gauss1d((q + 2) / 2, x, ww);
    for (int i = 0; i < n; i++) {
      double s = 0.5 * (1.0 + x[i]);
      for (int d = 0; d < 3; d++) { pts[i][d] = A[d] + s * (B[d] - A[d]); t1[i][d] = B[d] - A[d]; }
      w[i] = 0.5 * ww[i];
    }
    return n;
  }
  if (etype == OR_TET) { /* face k = the face opposite vertex k; triangle rule in (s,t) */
    if (facet < 0 || facet > 3) return -1;
    int v[3], m = 0;
    for (int k = 0; k < 4; k++) if (k != facet) v[m++] = k;
    double P0[3], P1[3], P2[3], p[8][2];
    ref_vertex(etype, v[0], P0); ref_vertex(etype, v[1], P1); ref_vertex(etype, v[2], P2);
    int n = tri_rule(q, p, w);
    for (int i = 0; i < n; i++)
      for (int d = 0; d < 3; d++) {
        pts[i][d] = P0[d] + p[i][0] * (P1[d] - P0[d]) + p[i][1] * (P2[d] - P0[d]);
        t1[i][d] = P1[d] - P0[d];
        t2[i][d] = P2[d] - P0[d];
      }
    return n;
  }
  /* hex face: bilinear map of its 4 reference corners, Gauss-Legendre n x n on [-1,1]^2 */
  if (facet < 0 || facet > 5) return -1;
  double c[4][3], x[4], ww[4];
  for (int k = 0; k < 4; k++) ref_vertex(etype, HEX_FACE[facet][k], c[k]);
  int n = gauss1d(q, x, ww), m = 0;
  if (n < 0) return -1;
  for (int j = 0; j < n; j++)
    for (int i = 0; i < n; i++) {
      double s = x[i], t = x[j];
      for (int d = 0; d < 3; d++) {
        pts[m][d] = 0.25 * ((1 - s) * (1 - t) * c[0][d] + (1 + s) * (1 - t) * c[1][d] +
                            (1 + s) * (1 + t) * c[2][d] + (1 - s) * (1 + t) * c[3][d]);
        t1[m][d] = 0.25 * (-(1 - t) * c[0][d] + (1 - t) * c[1][d] + (1 + t) * c[2][d] - (1 + t) * c[3][d]);
        t2[m][d] = 0.25 * (-(1 - s) * c[0][d] - (1 + s) * c[1][d] + (1 + s) * c[2][d] + (1 - s) * c[3][d]);
      }
      w[m] = ww[i] * ww[j];
      m++;
    }
  return m;
}

/* ------------------------------------------------------------------ geometry at a point (A5) */
typedef struct {
  double x[3], w, n[3];
  double N[MAXN], G[MAXN][3];
  double H[MAXN][3][3]; /* ∂²N_a/∂x_i∂x_j (physical)                 */
  double lap[MAXN];     /* Σ_k ∂²N_a/∂x_k∂x_k: feeds μ u_i,kk */
} qpt;

typedef struct {
  const or_problem* P;
  int64_t N, E;
  const double* coords;
  const int32_t* conn;
  int nloc, dim, kh;
} ctx;

static double det3(double J[3][3]) {
  return J[0][0] * (J[1][1] * J[2][2] - J[1][2] * J[2][1]) -
         J[0][1] * (J[1][0] * J[2][2] - J[1][2] * J[2][0]) +
         J[0][2] * (J[1][0] * J[2][1] - J[1][1] * J[2][0]);
}

/* x = Σ N_a x_a; J_ij = ∂x_i/∂ξ_j = Σ_a x_{a,i} ∂N_a/∂ξ_j; J^{-1} by cofactors;
 * G_{a,i} = ∂N_a/∂x_i = Σ_j (J^{-1})_{ji} ∂N_a/∂ξ_j.  Volume: w = ŵ|det J| (L1).
 * Facet: w = ŵ |J t1 × J t2| (3D) or ŵ |J t1| (2D); n = unit normal, oriented away from the
 * element's vertex centroid (outward, L8).  Returns 0, or -4 if det J <= 0. */
static int eval_point(const ctx* c, int64_t e, const double* xi, double wref, const double* t1,
                      const double* t2, int is_facet, qpt* q) {
  int dim = c->dim, nl = c->nloc;
  double dN[MAXN][3], X[MAXN][3], d2N[MAXN][3][3];
  shape(c->P->etype, c->P->order, xi, q->N, dN, d2N);
  for (int a = 0; a < nl; a++) {
    int64_t node = c->conn[(int64_t)a * c->E + e];
    for (int d = 0; d < dim; d++) X[a][d] = c->coords[(int64_t)d * c->N + node];
  }
  double J[3][3] = {{0}}, inv[3][3] = {{0}}, det;
  for (int i = 0; i < dim; i++)
    for (int j = 0; j < dim; j++)
      for (int a = 0; a < nl; a++) J[i][j] += X[a][i] * dN[a][j];
  if (dim == 2) {
    det = J[0][0] * J[1][1] - J[0][1] * J[1][0];
    inv[0][0] = J[1][1] / det; inv[0][1] = -J[0][1] / det;
    inv[1][0] = -J[1][0] / det; inv[1][1] = J[0][0] / det;
  } else {
    det = det3(J);
    inv[0][0] = (J[1][1] * J[2][2] - J[1][2] * J[2][1]) / det;
    inv[0][1] = (J[0][2] * J[2][1] - J[0][1] * J[2][2]) / det;
    inv[0][2] = (J[0][1] * J[1][2] - J[0][2] * J[1][1]) / det;
    inv[1][0] = (J[1][2] * J[2][0] - J[1][0] * J[2][2]) / det;
    inv[1][1] = (J[0][0] * J[2][2] - J[0][2] * J[2][0]) / det;
    inv[1][2] = (J[0][2] * J[1][0] - J[0][0] * J[1][2]) / det;
    inv[2][0] = (J[1][0] * J[2][1] - J[1][1] * J[2][0]) / det;
    inv[2][1] = (J[0][1] * J[2][0] - J[0][0] * J[2][1]) / det;
    inv[2][2] = (J[0][0] * J[1][1] - J[0][1] * J[1][0]) / det;
  }
  if (!(det > 0.0)) return -4;
  for (int a = 0; a < nl; a++)
    for (int i = 0; i < 3; i++) {
      q->G[a][i] = 0.0;
      if (i < dim)
        for (int j = 0; j < dim; j++) q->G[a][i] += inv[j][i] * dN[a][j];
    }
  for (int i = 0; i < 3; i++) {
    q->x[i] = 0.0;
    q->n[i] = 0.0;
    if (i < dim)
      for (int a = 0; a < nl; a++) q->x[i] += q->N[a] * X[a][i];
  }
  /* Second derivatives (chain rule twice): ∂²N/∂ξ_j∂ξ_l = Σ_im H_im J_ij J_ml + Σ_i G_i ∂²x_i/∂ξ_j∂ξ_l, so
   * H = J^{-T} (∂²N/∂ξ² − Σ_i G_i ∂²x_i/∂ξ²) J^{-1}, with ∂²x_i/∂ξ_j∂ξ_l = Σ_a x_{a,i} ∂²N_a/∂ξ_j∂ξ_l. */
  double Xh[3][3][3] = {{{0}}}; /* Xh[i][j][l] = ∂²x_i/∂ξ_j∂ξ_l */
  for (int i = 0; i < dim; i++)
    for (int j = 0; j < dim; j++)
      for (int l = 0; l < dim; l++)
        for (int a = 0; a < nl; a++) Xh[i][j][l] += X[a][i] * d2N[a][j][l];
  for (int a = 0; a < nl; a++) {
    double A[3][3] = {{0}}; /* reference-space Hessian minus the geometric term */
    for (int j = 0; j < dim; j++)
      for (int l = 0; l < dim; l++) {
        A[j][l] = d2N[a][j][l];
        for (int i = 0; i < dim; i++) A[j][l] -= q->G[a][i] * Xh[i][j][l];
      }
    q->lap[a] = 0.0;
    for (int i = 0; i < 3; i++)
      for (int m = 0; m < 3; m++) {
        double h = 0.0;
        if (i < dim && m < dim)
          for (int j = 0; j < dim; j++)
            for (int l = 0; l < dim; l++) h += inv[j][i] * A[j][l] * inv[l][m];
        q->H[a][i][m] = h;
      }
    for (int i = 0; i < dim; i++) q->lap[a] += q->H[a][i][i];
  }
  if (!is_facet) { q->w = wref * fabs(det); return 0; }
  double T1[3] = {0, 0, 0}, T2[3] = {0, 0, 0}, dA;
  for (int i = 0; i < dim; i++)
    for (int j = 0; j < dim; j++) { T1[i] += J[i][j] * t1[j]; T2[i] += J[i][j] * t2[j]; }
  if (dim == 2) {
    q->n[0] = T1[1]; q->n[1] = -T1[0];
    dA = sqrt(T1[0] * T1[0] + T1[1] * T1[1]);
  } else {
    q->n[0] = T1[1] * T2[2] - T1[2] * T2[1];
    q->n[1] = T1[2] * T2[0] - T1[0] * T2[2];
    q->n[2] = T1[0] * T2[1] - T1[1] * T2[0];
    dA = sqrt(q->n[0] * q->n[0] + q->n[1] * q->n[1] + q->n[2] * q->n[2]);
  }
  double cen[3] = {0, 0, 0}, dot = 0.0;
  int nv = n_vert_of(c->P->etype);
  for (int a = 0; a < nv; a++)
    for (int i = 0; i < dim; i++) cen[i] += X[a][i] / nv;
  for (int i = 0; i < dim; i++) { q->n[i] /= dA; dot += q->n[i] * (q->x[i] - cen[i]); }
  if (dot < 0.0)
    for (int i = 0; i < dim; i++) q->n[i] = -q->n[i];
  q->w = wref * dA;
  return 0;
}

/* ------------------------------------------------------------------ fields at a point (A6) */
/* Operand values Σ_b (D_λ N_b) ∂_t^ν φ̃_{α'(κ,b)} (D-2); ν = time level. */
typedef struct {
  double v[3][MAXK]; /* v[ν][κ]: value of ∂_t^ν φ̃^κ  */
  double g[MAXK][3]; /* g[κ][i]: ∂φ̃^κ/∂x_i (level 0) */
  double l[MAXK];    /* l[κ]: Σ_k ∂²φ̃^κ/∂x_k² (level 0), the u_i,kk of Rm */
} fld;

static void eval_fields(const ctx* c, int64_t e, const qpt* q, const double* state, fld* f) {
  memset(f, 0, sizeof(*f));
  int levels = c->P->nu_hat + 1;
  for (int b = 0; b < c->nloc; b++) {
    int64_t node = c->conn[(int64_t)b * c->E + e];
    for (int nu = 0; nu < levels && nu < 3; nu++)
      for (int k = 0; k < c->kh; k++)
        f->v[nu][k] += q->N[b] * state[((int64_t)nu * c->kh + k) * c->N + node];
    for (int k = 0; k < c->kh; k++) {
      for (int i = 0; i < c->dim; i++) f->g[k][i] += q->G[b][i] * state[(int64_t)k * c->N + node];
      f->l[k] += q->lap[b] * state[(int64_t)k * c->N + node];
    }
  }
}

/* ------------------------------------------------------------------ weak forms (A7) */
/* res(): the base term of each bilinear form times its dual word D0 N̄_a, for row (a, κ0).
 * dres(): the same expression differentiated along the trial direction `df` (product rule).
 * Forms: thermal P:821-823 / P:832-835; elasticity P:900-906 / P:913-923;
 * Navier-Stokes P:979-992 / P:998-1025. */
static double uw_inflow(const double* p, const double* x) {
  double U = p[3], H = p[4], y = x[1], z = x[2];
  return 16.0 * U * (H - y) * (H - z) * y * z / (H * H * H * H);
}

/* elasticity helpers: ε(a,i)_kl = ∂ε_kl/∂(δd_{a,i}) = ½(δ_ki G_al + δ_li G_ak) */
static void deps(const qpt* q, int a, int i, double out[3][3]) {
  for (int k = 0; k < 3; k++)
    for (int l = 0; l < 3; l++) out[k][l] = 0.5 * ((k == i ? q->G[a][l] : 0.0) + (l == i ? q->G[a][k] : 0.0));
}
static void stress(const double* p, int dim, const double g[][3], double sig[3][3]) {
  double E = p[0], nu = p[1];
  double lam = E * nu / ((1.0 + nu) * (1.0 - 2.0 * nu)), mu = E / (2.0 * (1.0 + nu));
  double eps[3][3], tr = 0.0;
  for (int k = 0; k < 3; k++)
    for (int l = 0; l < 3; l++) eps[k][l] = (k < dim && l < dim) ? 0.5 * (g[k][l] + g[l][k]) : 0.0;
  for (int k = 0; k < dim; k++) tr += eps[k][k];
  for (int k = 0; k < 3; k++)
    for (int l = 0; l < 3; l++) sig[k][l] = lam * (k == l ? tr : 0.0) + 2.0 * mu * eps[k][l];
}

static double res(const ctx* c, const or_term* t, const qpt* q, const fld* f, int a, int k0) {
  const double* p = t->p;
  int dim = c->dim;
  double Na = q->N[a];
  switch (t->form) {
    case OR_THERMAL_DOMAIN: { /* -C(T,T_t) - k(T_,i, T_,i) + (T, s) */
      double s = p[2];
      if (p[3] != 0.0) /* manufactured source s0 Π sin(π x_d) */
        for (int d = 0; d < dim; d++) s *= sin(M_PI * q->x[d]);
      double r = Na * s;
      for (int i = 0; i < dim; i++) r -= p[1] * q->G[a][i] * f->g[0][i];
      if (c->P->nu_hat >= 1) r -= p[0] * Na * f->v[1][0];
      return r;
    }
    case OR_THERMAL_CONV_RAD: { /* h(T, T_env - T) + e_m σ^b (T, T_env^4 - T^4) */
      double T = f->v[0][0], Te = p[1];
      return Na * (p[0] * (Te - T) + p[2] * p[3] * (Te * Te * Te * Te - T * T * T * T));
    }
    case OR_THERMAL_FIX: { /* h_p(T, T_fix - T) + k(T, n_i T_,i) */
      double T = f->v[0][0], nt = 0.0;
      for (int i = 0; i < dim; i++) nt += q->n[i] * f->g[0][i];
      return p[0] * Na * (p[1] - T) + p[2] * Na * nt;
    }
    case OR_ELAST_DOMAIN: { /* -(ε_ij, σ_ij) */
      double de[3][3], sig[3][3], r = 0.0;
      deps(q, a, k0, de);
      stress(p, dim, f->g, sig);
      for (int k = 0; k < dim; k++)
        for (int l = 0; l < dim; l++) r -= de[k][l] * sig[k][l];
      return r;
    }
    case OR_ELAST_FIX_ALL: /* τ(d_i, d^w_i - d_i) */
      return p[0] * Na * (p[1 + k0] - f->v[0][k0]);
    case OR_ELAST_FIX_D1: /* τ(d_1, d^w_1 - d_1) — component 1 only */
      return k0 == 0 ? p[0] * Na * (p[1] - f->v[0][0]) : 0.0;
    case OR_ELAST_LOAD: { /* (d_i, σ^l_ij n_j) */
      double r = 0.0;
      for (int j = 0; j < dim; j++) r += p[3 * k0 + j] * q->n[j];
      return Na * r;
    }
    default: break;
  }
  /* ---- Navier-Stokes: κ = 0..dim-1 velocity u_i, κ = dim pressure p (L3) */
  double rho = p[0], mu = p[1];
  const double* u = f->v[0];
  double pr = f->v[0][dim];
  double Rc = 0.0, Rm[3] = {0, 0, 0}; /* Rm_i = ρ u_k u_i,k + p_,i − μ u_i,kk (0 for P1, L10) */
  for (int k = 0; k < dim; k++) Rc += f->g[k][k];
  for (int i = 0; i < dim; i++) {
    Rm[i] = f->g[dim][i];
    for (int k = 0; k < dim; k++) Rm[i] += rho * u[k] * f->g[i][k];
    Rm[i] -= mu * f->l[i];
  }
  double Gn = 0.0, un = 0.0;
  for (int j = 0; j < dim; j++) { Gn += q->G[a][j] * q->n[j]; un += u[j] * q->n[j]; }
  int is_p = (k0 == dim), i = k0;
  double r = 0.0;
  if (t->form == OR_NS_DOMAIN) {
    double tm = p[2], tc = p[3];
    if (!is_p) {
      for (int j = 0; j < dim; j++) r += -rho * q->G[a][j] * u[i] * u[j]; /* -ρ(u_i,j, u_i u_j) */
      r += -q->G[a][i] * pr;                                              /* -(u_i,i, p)       */
      for (int j = 0; j < dim; j++) r += mu * q->G[a][j] * f->g[i][j];    /* μ(u_i,j, u_i,j)   */
      for (int j = 0; j < dim; j++) r += tm * rho * q->G[a][j] * Rm[i] * u[j]; /* SUPG */
      r += tc * q->G[a][i] * Rc;                                          /* τc(u_i,i, Rc)     */
    } else {
      r += Na * Rc;                                                       /* (p, u_i,i)        */
      for (int ii = 0; ii < dim; ii++) r += tm * q->G[a][ii] * Rm[ii];   /* τm(p_,i, Rm_i)    */
    }
    return r;
  }
  /* boundary: every NS boundary group = BASE + its own part */
  if (!is_p) { /* BASE: (u_i, p n_i) - μ(u_i, u_i,j n_j) */
    r += Na * pr * q->n[i];
    for (int j = 0; j < dim; j++) r -= mu * Na * f->g[i][j] * q->n[j];
  }
  if (t->form == OR_NS_BND_INFLOW) {
    double uw[3] = {uw_inflow(p, q->x), 0.0, 0.0}, uwn = 0.0;
    for (int j = 0; j < dim; j++) uwn += uw[j] * q->n[j];
    if (!is_p) {
      r += rho * Na * uw[i] * uwn;             /* ρ(u_i, u^w_i u^w_j n_j)     */
      r += mu * Gn * (uw[i] - u[i]);           /* μ(u_i,j, (u^w_i - u_i) n_j) */
      r += p[2] * rho * Na * (u[i] - uw[i]);   /* τb ρ(u_i, u_i - u^w_i)      */
    } else {
      double s = 0.0;
      for (int ii = 0; ii < dim; ii++) s += (uw[ii] - u[ii]) * q->n[ii];
      r += Na * s;                              /* (p, (u^w_i - u_i) n_i)      */
    }
  } else if (t->form == OR_NS_BND_OUTFLOW) {
    if (!is_p) r += rho * Na * u[i] * un;      /* ρ(u_i, u_i u_j n_j)         */
  } else if (t->form == OR_NS_BND_FIX) {
    if (!is_p) {
      r += -mu * Gn * u[i];                     /* μ(u_i,j, -u_i n_j)          */
      r += p[2] * rho * Na * u[i];              /* τb ρ(u_i, u_i)              */
    } else {
      r += -Na * un;                            /* (p, -u_i n_i)               */
    }
  }
  return r;
}

/* Directional derivative of res() along df (df = trial-function operand values × f_ν). */
static double dres(const ctx* c, const or_term* t, const qpt* q, const fld* f, const fld* df, int a,
                   int k0) {
  const double* p = t->p;
  int dim = c->dim;
  double Na = q->N[a];
  switch (t->form) {
    case OR_THERMAL_DOMAIN: {
      double r = 0.0;
      for (int i = 0; i < dim; i++) r -= p[1] * q->G[a][i] * df->g[0][i];
      if (c->P->nu_hat >= 1) r -= p[0] * Na * df->v[1][0];
      return r;
    }
    case OR_THERMAL_CONV_RAD: {
      double T = f->v[0][0];
      return Na * (-p[0] * df->v[0][0] - 4.0 * p[2] * p[3] * T * T * T * df->v[0][0]);
    }
    case OR_THERMAL_FIX: {
      double nt = 0.0;
      for (int i = 0; i < dim; i++) nt += q->n[i] * df->g[0][i];
      return -p[0] * Na * df->v[0][0] + p[2] * Na * nt;
    }
    case OR_ELAST_DOMAIN: {
      double de[3][3], dsig[3][3], r = 0.0;
      deps(q, a, k0, de);
      stress(p, dim, df->g, dsig); /* σ is linear in ∇d */
      for (int k = 0; k < dim; k++)
        for (int l = 0; l < dim; l++) r -= de[k][l] * dsig[k][l];
      return r;
    }
    case OR_ELAST_FIX_ALL: return -p[0] * Na * df->v[0][k0];
    case OR_ELAST_FIX_D1: return k0 == 0 ? -p[0] * Na * df->v[0][0] : 0.0;
    case OR_ELAST_LOAD: return 0.0;
    default: break;
  }
  double rho = p[0], mu = p[1];
  const double* u = f->v[0];
  const double* du = df->v[0];
  double dpr = df->v[0][dim];
  double Rm[3] = {0, 0, 0}, dRm[3] = {0, 0, 0}, dRc = 0.0;
  for (int k = 0; k < dim; k++) dRc += df->g[k][k];
  for (int i = 0; i < dim; i++) {
    Rm[i] = f->g[dim][i];
    dRm[i] = df->g[dim][i];
    for (int k = 0; k < dim; k++) {
      Rm[i] += rho * u[k] * f->g[i][k];
      dRm[i] += rho * (du[k] * f->g[i][k] + u[k] * df->g[i][k]);
    }
    Rm[i] -= mu * f->l[i];   /* − μ u_i,kk */
    dRm[i] -= mu * df->l[i];
  }
  double Gn = 0.0, un = 0.0, dun = 0.0;
  for (int j = 0; j < dim; j++) {
    Gn += q->G[a][j] * q->n[j];
    un += u[j] * q->n[j];
    dun += du[j] * q->n[j];
  }
  int is_p = (k0 == dim), i = k0;
  double r = 0.0;
  if (t->form == OR_NS_DOMAIN) {
    double tm = p[2], tc = p[3];
    if (!is_p) {
      for (int j = 0; j < dim; j++) r += -rho * q->G[a][j] * (du[i] * u[j] + u[i] * du[j]);
      r += -q->G[a][i] * dpr;
      for (int j = 0; j < dim; j++) r += mu * q->G[a][j] * df->g[i][j];
      for (int j = 0; j < dim; j++) r += tm * rho * q->G[a][j] * (dRm[i] * u[j] + Rm[i] * du[j]);
      r += tc * q->G[a][i] * dRc;
    } else {
      r += Na * dRc;
      for (int ii = 0; ii < dim; ii++) r += tm * q->G[a][ii] * dRm[ii];
    }
    return r;
  }
  if (!is_p) {
    r += Na * dpr * q->n[i];
    for (int j = 0; j < dim; j++) r -= mu * Na * df->g[i][j] * q->n[j];
  }
  if (t->form == OR_NS_BND_INFLOW) {
    if (!is_p) {
      r += -mu * Gn * du[i];
      r += p[2] * rho * Na * du[i];
    } else {
      r += -Na * dun;
    }
  } else if (t->form == OR_NS_BND_OUTFLOW) {
    if (!is_p) r += rho * Na * (du[i] * un + u[i] * dun);
  } else if (t->form == OR_NS_BND_FIX) {
    if (!is_p) {
      r += -mu * Gn * du[i];
      r += p[2] * rho * Na * du[i];
    } else {
      r += -Na * dun;
    }
  }
  return r;
}

static int form_ok(int physics, int form) {
  if (physics == OR_THERMAL) return form >= OR_THERMAL_DOMAIN && form <= OR_THERMAL_FIX;
  if (physics == OR_ELASTICITY) return form >= OR_ELAST_DOMAIN && form <= OR_ELAST_LOAD;
  if (physics == OR_NS) return form >= OR_NS_DOMAIN && form <= OR_NS_BND_FIX;
  return 0;
}

/* ------------------------------------------------------------------ the system */
struct or_system {
  int status;
  int64_t bad_elem;
  int64_t N, E, n_sel, n_rows, nnz, nnz_s;
  int nloc, kh;
  int64_t* sel;      /* selected nodes, ascending                       */
  int64_t* loc;      /* node -> local selected index or -1              */
  int64_t* rowptr_s; /* scalar CSR over selected rows                   */
  int32_t* colidx_s;
  int64_t* rowptr;   /* block CSR, rows κ0-major over selected nodes    */
  int32_t* colidx;
  double* values;
  double* rhs;
  double* absd;
};

static int cmp_i64(const void* x, const void* y) {
  int64_t a = *(const int64_t*)x, b = *(const int64_t*)y;
  return (a > b) - (a < b);
}

/* Block B: control-point pairs "by variating the last input ... each unique pair is only
 * kept once" (B-1 item 4), symbol pairs (A-3) = all (κ0,κλ) (L6), I = g(κ0,α1), J = g(κλ,α2) (B-4). */
static int build_pattern(or_system* s, const ctx* c) {
  int64_t N = c->N, E = c->E;
  int nl = c->nloc, kh = c->kh;
  int64_t npairs = 0;
  for (int64_t e = 0; e < E; e++)
    for (int a = 0; a < nl; a++)
      if (s->loc[c->conn[(int64_t)a * E + e]] >= 0) npairs += nl;
  int64_t* keys = (int64_t*)malloc(sizeof(int64_t) * (npairs > 0 ? npairs : 1));
  if (!keys) return -1;
  int64_t m = 0;
  for (int64_t e = 0; e < E; e++)
    for (int a = 0; a < nl; a++) {
      int64_t r = c->conn[(int64_t)a * E + e];
      if (s->loc[r] < 0) continue;
      for (int b = 0; b < nl; b++) keys[m++] = r * N + c->conn[(int64_t)b * E + e];
    }
  qsort(keys, (size_t)npairs, sizeof(int64_t), cmp_i64);
  int64_t u = 0;
  for (int64_t i = 0; i < npairs; i++)
    if (i == 0 || keys[i] != keys[i - 1]) keys[u++] = keys[i];
  s->nnz_s = u;
  s->rowptr_s = (int64_t*)calloc((size_t)s->n_sel + 1, sizeof(int64_t));
  s->colidx_s = (int32_t*)malloc(sizeof(int32_t) * (u > 0 ? u : 1));
  if (!s->rowptr_s || !s->colidx_s) { free(keys); return -1; }
  for (int64_t i = 0; i < u; i++) {
    int64_t r = keys[i] / N;
    s->rowptr_s[s->loc[r] + 1]++;
    s->colidx_s[i] = (int32_t)(keys[i] % N);
  }
  for (int64_t i = 0; i < s->n_sel; i++) s->rowptr_s[i + 1] += s->rowptr_s[i];
  free(keys);
  /* block rows: row (κ0, node) has columns g(κλ, α2) for κλ ascending, α2 ascending */
  s->n_rows = (int64_t)kh * s->n_sel;
  s->nnz = (int64_t)kh * kh * u;
  s->rowptr = (int64_t*)malloc(sizeof(int64_t) * (size_t)(s->n_rows + 1));
  s->colidx = (int32_t*)malloc(sizeof(int32_t) * (size_t)(s->nnz > 0 ? s->nnz : 1));
  if (!s->rowptr || !s->colidx) return -1;
  int64_t pos = 0;
  for (int k0 = 0; k0 < kh; k0++)
    for (int64_t i = 0; i < s->n_sel; i++) {
      s->rowptr[(int64_t)k0 * s->n_sel + i] = pos;
      for (int kl = 0; kl < kh; kl++)
        for (int64_t t = s->rowptr_s[i]; t < s->rowptr_s[i + 1]; t++)
          s->colidx[pos++] = (int32_t)((int64_t)kl * N + s->colidx_s[t]);
    }
  s->rowptr[s->n_rows] = pos;
  return 0;
}


/* position of column `col` in the scalar row of selected node li (binary search), -1 if absent */
static int64_t find_pos(const or_system* s, int64_t li, int64_t col) {
  int64_t lo = s->rowptr_s[li], hi = s->rowptr_s[li + 1] - 1;
  while (lo <= hi) {
    int64_t mid = (lo + hi) / 2;
    if (s->colidx_s[mid] == col) return mid;
    if (s->colidx_s[mid] < col) lo = mid + 1; else hi = mid - 1;
  }
  return -1;
}

static double time_factor(const or_problem* P, int nu) { /* Eq. gen_alpha, L12/L13 */
  if (nu == 0) return P->nu_hat == 0 ? 1.0 : P->c1;
  if (nu == 1) return P->c2 / (P->b1 * P->dt);
  return P->c3 / (P->b1 * P->b2 * P->dt * P->dt);
}

/* Accumulate one quadrature point of one term of element e (the D-2 / D-3 updates). */
static void add_point(or_system* s, const ctx* c, const or_term* t, int64_t e, const qpt* q,
                      const double* state, int want_m, int want_r) {
  int nl = c->nloc, kh = c->kh, dim = c->dim;
  fld f;
  eval_fields(c, e, q, state, &f);
  int64_t node[MAXN], li[MAXN];
  for (int a = 0; a < nl; a++) {
    node[a] = c->conn[(int64_t)a * c->E + e];
    li[a] = s->loc[node[a]];
  }
  if (want_r)
    for (int a = 0; a < nl; a++) {
      if (li[a] < 0) continue;
      for (int k0 = 0; k0 < kh; k0++) {
        double v = q->w * res(c, t, q, &f, a, k0);
        int64_t r = (int64_t)k0 * s->n_sel + li[a];
        s->rhs[r] += v;
        s->absd[r] += fabs(v);
      }
    }
  if (!want_m || t->form == OR_ELAST_LOAD) return;
  int levels = c->P->nu_hat + 1;
  for (int b = 0; b < nl; b++)
    for (int kl = 0; kl < kh; kl++) {
      fld df; /* trial direction: ∂(operand)/∂φ_{b,κλ} times f_ν */
      memset(&df, 0, sizeof(df));
      for (int nu = 0; nu < levels && nu < 3; nu++) df.v[nu][kl] = time_factor(c->P, nu) * q->N[b];
      for (int i = 0; i < dim; i++) df.g[kl][i] = time_factor(c->P, 0) * q->G[b][i];
      df.l[kl] = time_factor(c->P, 0) * q->lap[b];
      for (int a = 0; a < nl; a++) {
        if (li[a] < 0) continue;
        int64_t deg = s->rowptr_s[li[a] + 1] - s->rowptr_s[li[a]];
        int64_t sl = find_pos(s, li[a], node[b]); /* slot of (α(e,a), α(e,b)) */
        for (int k0 = 0; k0 < kh; k0++) {
          int64_t r = (int64_t)k0 * s->n_sel + li[a];
          int64_t idx = s->rowptr[r] + (int64_t)kl * deg + (sl - s->rowptr_s[li[a]]);
          s->values[idx] += q->w * dres(c, t, q, &f, &df, a, k0);
        }
      }
    }
}

or_system* or_assemble(const or_problem* P, int64_t n_nodes, const double* coords, int64_t n_elems,
                       const int32_t* conn, int n_bsets, const int64_t* bset_len,
                       const int32_t* const* bset_elem, const int8_t* const* bset_facet,
                       const double* state, const uint8_t* row_mask, int want_matrix,
                       int want_residual) {
  or_system* s = (or_system*)calloc(1, sizeof(or_system));
  if (!s) return NULL;
  s->bad_elem = -1;
  ctx c = {P, n_nodes, n_elems, coords, conn, n_loc_of(P->etype, P->order), P->dim, 0};
  c.kh = P->physics == OR_THERMAL ? 1 : (P->physics == OR_ELASTICITY ? P->dim : P->dim + 1);
  s->N = n_nodes; s->E = n_elems; s->nloc = c.nloc; s->kh = c.kh;
  if (c.nloc < 0 || (P->etype == OR_TRI) != (P->dim == 2)) {
    s->status = -2;
    return s;
  }
  for (int t = 0; t < P->n_terms; t++)
    if (!form_ok(P->physics, P->terms[t].form) ||
        (P->terms[t].region >= n_bsets) || (P->terms[t].region < -1)) { s->status = -2; return s; }
  s->loc = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n_nodes > 0 ? n_nodes : 1));
  s->sel = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n_nodes > 0 ? n_nodes : 1));
  for (int64_t i = 0; i < n_nodes; i++) {
    if (!row_mask || row_mask[i]) { s->loc[i] = s->n_sel; s->sel[s->n_sel++] = i; }
    else s->loc[i] = -1;
  }
  if (build_pattern(s, &c) != 0) { s->status = -1; return s; }
  s->values = (double*)calloc((size_t)(s->nnz > 0 ? s->nnz : 1), sizeof(double));
  s->rhs = (double*)calloc((size_t)(s->n_rows > 0 ? s->n_rows : 1), sizeof(double));
  s->absd = (double*)calloc((size_t)(s->n_rows > 0 ? s->n_rows : 1), sizeof(double));
  double pts[MAXQ][3], w[MAXQ], t1[MAXQ][3], t2[MAXQ][3];
  qpt q;
  for (int t = 0; t < P->n_terms; t++) { /* "each bilinear form" (D-2/D-3) */
    const or_term* term = &P->terms[t];
    if (term->region < 0) { /* domain: each element, each quadrature point */
      int nq = vol_rule(P->etype, P->quad_order, pts, w);
      if (nq < 0) { s->status = -2; return s; }
      for (int64_t e = 0; e < n_elems; e++) {
        int touch = 0;
        for (int a = 0; a < c.nloc; a++) touch |= s->loc[conn[(int64_t)a * n_elems + e]] >= 0;
        if (!touch) continue;
        for (int g = 0; g < nq; g++) {
          if (eval_point(&c, e, pts[g], w[g], NULL, NULL, 0, &q) != 0) {
            if (s->status == 0) { s->status = -4; s->bad_elem = e; }
            break;
          }
          add_point(s, &c, term, e, &q, state, want_matrix, want_residual);
        }
      }
    } else { /* boundary: each (element, facet) of the set, each facet point */
      int k = term->region;
      for (int64_t m = 0; m < bset_len[k]; m++) {
        int64_t e = bset_elem[k][m];
        int touch = 0;
        for (int a = 0; a < c.nloc; a++) touch |= s->loc[conn[(int64_t)a * n_elems + e]] >= 0;
        if (!touch) continue;
        int nq = facet_rule(P->etype, P->quad_order, bset_facet[k][m], pts, w, t1, t2);
        if (nq < 0) { s->status = -2; return s; }
        for (int g = 0; g < nq; g++) {
          if (eval_point(&c, e, pts[g], w[g], t1[g], t2[g], 1, &q) != 0) {
            if (s->status == 0) { s->status = -4; s->bad_elem = e; }
            break;
          }
          add_point(s, &c, term, e, &q, state, want_matrix, want_residual);
        }
      }
    }
  }
  return s;
}

int or_status(const or_system* s, int64_t* bad_elem) {
  if (bad_elem) *bad_elem = s->bad_elem;
  return s->status;
}
int64_t or_n_sel_nodes(const or_system* s) { return s->n_sel; }
int64_t or_n_rows(const or_system* s) { return s->n_rows; }
int64_t or_nnz(const or_system* s) { return s->nnz; }
int64_t or_nnz_s(const or_system* s) { return s->nnz_s; }

void or_get(const or_system* s, int64_t* sel_nodes, int64_t* rows, int64_t* rowptr, int32_t* colidx,
            double* values, double* rhs, double* abs_d, int64_t* rowptr_s, int32_t* colidx_s) {
  if (sel_nodes) memcpy(sel_nodes, s->sel, sizeof(int64_t) * (size_t)s->n_sel);
  if (rows)
    for (int k0 = 0; k0 < s->kh; k0++)
      for (int64_t i = 0; i < s->n_sel; i++) rows[(int64_t)k0 * s->n_sel + i] = (int64_t)k0 * s->N + s->sel[i];
  if (rowptr) memcpy(rowptr, s->rowptr, sizeof(int64_t) * (size_t)(s->n_rows + 1));
  if (colidx) memcpy(colidx, s->colidx, sizeof(int32_t) * (size_t)s->nnz);
  if (values) memcpy(values, s->values, sizeof(double) * (size_t)s->nnz);
  if (rhs) memcpy(rhs, s->rhs, sizeof(double) * (size_t)s->n_rows);
  if (abs_d) memcpy(abs_d, s->absd, sizeof(double) * (size_t)s->n_rows);
  if (rowptr_s) memcpy(rowptr_s, s->rowptr_s, sizeof(int64_t) * (size_t)(s->n_sel + 1));
  if (colidx_s) memcpy(colidx_s, s->colidx_s, sizeof(int32_t) * (size_t)s->nnz_s);
}

void or_get_slot(const or_system* s, const int32_t* conn, int32_t* slot_s) {
  int nl = s->nloc;
  for (int a = 0; a < nl; a++)
    for (int b = 0; b < nl; b++)
      for (int64_t e = 0; e < s->E; e++) {
        int64_t r = conn[(int64_t)a * s->E + e], col = conn[(int64_t)b * s->E + e];
        slot_s[((int64_t)a * nl + b) * s->E + e] = s->loc[r] >= 0 ? (int32_t)find_pos(s, s->loc[r], col) : -1;
      }
}

void or_free(or_system* s) {
  if (!s) return;
  free(s->sel); free(s->loc); free(s->rowptr_s); free(s->colidx_s); free(s->rowptr);
  free(s->colidx); free(s->values); free(s->rhs); free(s->absd);
  free(s);
}

int or_qp_data(const or_problem* P, int64_t n_nodes, const double* coords, int64_t n_elems,
               const int32_t* conn, int64_t e, int facet, double* x, double* w, double* n,
               double* N, double* G, double* H) {
  ctx c = {P, n_nodes, n_elems, coords, conn, n_loc_of(P->etype, P->order), P->dim, 1};
  if (c.nloc < 0) return -2;
  double pts[MAXQ][3], wr[MAXQ], t1[MAXQ][3], t2[MAXQ][3];
  int nq = facet < 0 ? vol_rule(P->etype, P->quad_order, pts, wr)
                     : facet_rule(P->etype, P->quad_order, facet, pts, wr, t1, t2);
  if (nq < 0) return -2;
  for (int g = 0; g < nq; g++) {
    qpt q;
    int rc = facet < 0 ? eval_point(&c, e, pts[g], wr[g], NULL, NULL, 0, &q)
                       : eval_point(&c, e, pts[g], wr[g], t1[g], t2[g], 1, &q);
    if (rc != 0) return rc;
    for (int d = 0; d < 3; d++) { x[3 * g + d] = q.x[d]; n[3 * g + d] = q.n[d]; }
    w[g] = q.w;
    for (int a = 0; a < c.nloc; a++) {
      N[g * c.nloc + a] = q.N[a];
      for (int d = 0; d < 3; d++) G[(g * c.nloc + a) * 3 + d] = q.G[a][d];
      if (H)
        for (int d = 0; d < 3; d++)
          for (int d2 = 0; d2 < 3; d2++) H[((g * c.nloc + a) * 3 + d) * 3 + d2] = q.H[a][d][d2];
    }
  }
  return nq;
}
