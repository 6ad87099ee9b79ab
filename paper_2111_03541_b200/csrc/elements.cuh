// elements.cuh — reference elements, quadrature rules and facet rules for the device path.
//
// PAPER.md: "φ^h = Σ_α N_α φ_α", numerical integration Σ_γ w_γ (...) at x_γ,
// Lagrange simplex/cube elements.  Readings: L7 VTK node orders,
// L8 facet numbering with outward normals, L9 quadrature (hex: Gauss-Legendre points per axis;
// simplices: exactness degree).
//
// Facet geometry uses Nanson's relation n dA = det(J) J^{-T} m̂ dÂ, with m̂ the outward reference
// normal of the facet scaled by (reference facet measure / parameter measure).  Since det J > 0 is
// enforced, the physical normal is outward by construction (no orientation test needed).
#pragma once
#include <cstdint>

namespace fem {

enum { ET_TRI = 1, ET_TET = 2, ET_HEX = 4, ET_HEXS = 5 };  // ET_HEXS: 20-node serendipity cube

// ---------------------------------------------------------------- 1D Gauss-Legendre on [-1,1]
__host__ __device__ inline void gauss_legendre(int n, int i, double& x, double& w) {
  if (n == 1) { x = 0.0; w = 2.0; return; }
  if (n == 2) { x = (i == 0 ? -1.0 : 1.0) * 0.57735026918962576451; w = 1.0; return; }
  // n == 3
  const double r = 0.77459666924148337704;
  x = (i == 0) ? -r : (i == 1 ? 0.0 : r);
  w = (i == 1) ? 8.0 / 9.0 : 5.0 / 9.0;
}

// ---------------------------------------------------------------- element traits
template <int ET, int ORD> struct Elem;

// P1 triangle: λ = (1-ξ-η, ξ, η)
template <> struct Elem<ET_TRI, 1> {
  static constexpr int DIM = 2, NL = 3, NV = 3, NF = 3;
  __host__ __device__ static void shape(const double* xi, double* N, double (*dN)[2]) {
    N[0] = 1.0 - xi[0] - xi[1];
    N[1] = xi[0];
    N[2] = xi[1];
    dN[0][0] = -1.0; dN[0][1] = -1.0;
    dN[1][0] = 1.0;  dN[1][1] = 0.0;
    dN[2][0] = 0.0;  dN[2][1] = 1.0;
  }
  __host__ __device__ static constexpr int vol_nq(int q) { return q <= 1 ? 1 : 3; }
  __host__ __device__ static void vol_qp(int q, int i, double* xi, double& w) {
    if (q <= 1) { xi[0] = xi[1] = 1.0 / 3.0; w = 0.5; return; }
    const double s = 1.0 / 6.0, t = 2.0 / 3.0;
    xi[0] = (i == 1) ? t : s;
    xi[1] = (i == 2) ? t : s;
    w = 1.0 / 6.0;
  }
  __host__ __device__ static constexpr int fac_nq(int q) { return (q + 2) / 2; }
  // edge f joins vertex f and vertex f+1 (mod 3); parameter s in [0,1]
  __host__ __device__ static void fac_qp(int q, int f, int i, double* xi, double& w, double* mref) {
    const double V[3][2] = {{0, 0}, {1, 0}, {0, 1}};
    double x, wg;
    gauss_legendre(fac_nq(q), i, x, wg);
    const double s = 0.5 * (1.0 + x);
    const int p = f, r = (f + 1) % 3;
    xi[0] = V[p][0] + s * (V[r][0] - V[p][0]);
    xi[1] = V[p][1] + s * (V[r][1] - V[p][1]);
    w = 0.5 * wg;
    // outward reference normal scaled by edge length: rotate the edge vector clockwise
    mref[0] = V[r][1] - V[p][1];
    mref[1] = -(V[r][0] - V[p][0]);
  }
};

// P1 / P2 tetrahedra: λ = (1-ξ-η-ζ, ξ, η, ζ); P2 edge nodes (0,1),(1,2),(0,2),(0,3),(1,3),(2,3)
__host__ __device__ inline void tet_bary(const double* xi, double* L) {
  L[0] = 1.0 - xi[0] - xi[1] - xi[2];
  L[1] = xi[0];
  L[2] = xi[1];
  L[3] = xi[2];
}
__host__ __device__ inline double dbary(int k, int j) { return k == 0 ? -1.0 : (k == j + 1 ? 1.0 : 0.0); }

struct TetRules {
  __host__ __device__ static constexpr int vol_nq(int q) { return q <= 1 ? 1 : 4; }
  __host__ __device__ static void vol_qp(int q, int i, double* xi, double& w) {
    if (q <= 1) { xi[0] = xi[1] = xi[2] = 0.25; w = 1.0 / 6.0; return; }
    const double a = 0.13819660112501051518, b = 0.58541019662496845446;  // (5∓√5)/20, (5+3√5)/20
    xi[0] = (i == 1) ? b : a;
    xi[1] = (i == 2) ? b : a;
    xi[2] = (i == 3) ? b : a;
    w = 1.0 / 24.0;
  }
  __host__ __device__ static constexpr int fac_nq(int q) { return q <= 1 ? 1 : 3; }
  // face f = the face opposite vertex f; points = barycentric combinations of its three vertices
  __host__ __device__ static void fac_qp(int q, int f, int i, double* xi, double& w, double* mref) {
    const double V[4][3] = {{0, 0, 0}, {1, 0, 0}, {0, 1, 0}, {0, 0, 1}};
    int v[3], m = 0;
    for (int k = 0; k < 4; k++)
      if (k != f) v[m++] = k;
    double lam[3];
    if (q <= 1) { lam[0] = lam[1] = lam[2] = 1.0 / 3.0; w = 0.5; }
    else {
      for (int k = 0; k < 3; k++) lam[k] = (k == i) ? 2.0 / 3.0 : 1.0 / 6.0;
      w = 1.0 / 6.0;
    }
    for (int d = 0; d < 3; d++) xi[d] = lam[0] * V[v[0]][d] + lam[1] * V[v[1]][d] + lam[2] * V[v[2]][d];
    // outward normals of the reference tet, scaled by 2·face area
    if (f == 0) { mref[0] = mref[1] = mref[2] = 1.0; }
    else { mref[0] = mref[1] = mref[2] = 0.0; mref[f - 1] = -1.0; }
  }
};

template <> struct Elem<ET_TET, 1> : TetRules {
  static constexpr int DIM = 3, NL = 4, NV = 4, NF = 4;
  static constexpr bool CURVED2 = false;  // reference second derivatives vanish
  __host__ __device__ static void node_hess(int, const double*, double (*h)[3]) {
    for (int j = 0; j < 3; j++)
      for (int l = 0; l < 3; l++) h[j][l] = 0.0;
  }
  __host__ __device__ static void shape(const double* xi, double* N, double (*dN)[3]) {
    double L[4];
    tet_bary(xi, L);
    for (int k = 0; k < 4; k++) {
      N[k] = L[k];
      for (int j = 0; j < 3; j++) dN[k][j] = dbary(k, j);
    }
  }
};

template <> struct Elem<ET_TET, 2> : TetRules {
  static constexpr int DIM = 3, NL = 10, NV = 4, NF = 4;
  static constexpr bool CURVED2 = true;
  // ∂²N_a/∂ξ_j∂ξ_l: vertex L(2L-1) -> 4 ∂L_j ∂L_l; edge 4 L_p L_q -> 4(∂L_p,j ∂L_q,l + ∂L_q,j ∂L_p,l)
  __host__ __device__ static void node_hess(int a, const double*, double (*h)[3]) {
    const int EP[6] = {0, 1, 0, 0, 1, 2}, EQ[6] = {1, 2, 2, 3, 3, 3};
    for (int j = 0; j < 3; j++)
      for (int l = 0; l < 3; l++)
        h[j][l] = a < 4 ? 4.0 * dbary(a, j) * dbary(a, l)
                        : 4.0 * (dbary(EP[a - 4], j) * dbary(EQ[a - 4], l) + dbary(EQ[a - 4], j) * dbary(EP[a - 4], l));
  }
  __host__ __device__ static void shape(const double* xi, double* N, double (*dN)[3]) {
    const int EP[6] = {0, 1, 0, 0, 1, 2}, EQ[6] = {1, 2, 2, 3, 3, 3};
    double L[4];
    tet_bary(xi, L);
    for (int k = 0; k < 4; k++) {
      N[k] = L[k] * (2.0 * L[k] - 1.0);
      for (int j = 0; j < 3; j++) dN[k][j] = (4.0 * L[k] - 1.0) * dbary(k, j);
    }
    for (int e = 0; e < 6; e++) {
      const int p = EP[e], q = EQ[e];
      N[4 + e] = 4.0 * L[p] * L[q];
      for (int j = 0; j < 3; j++) dN[4 + e][j] = 4.0 * (dbary(p, j) * L[q] + L[p] * dbary(q, j));
    }
  }
};

// Q1 hexahedron on [-1,1]^3, VTK order
__host__ __device__ inline double hex_sign(int a, int d) {
  // x: - + + - - + + - ; y: - - + + - - + + ; z: - - - - + + + +
  if (d == 0) return ((a & 3) == 1 || (a & 3) == 2) ? 1.0 : -1.0;
  if (d == 1) return ((a & 3) >= 2) ? 1.0 : -1.0;
  return a >= 4 ? 1.0 : -1.0;
}

template <> struct Elem<ET_HEX, 1> {
  static constexpr int DIM = 3, NL = 8, NV = 8, NF = 6;
  static constexpr bool CURVED2 = true;  // trilinear: mixed second derivatives
  __host__ __device__ static void node_hess(int a, const double* xi, double (*h)[3]) {
    double f[3];
    for (int d = 0; d < 3; d++) f[d] = 0.5 * (1.0 + hex_sign(a, d) * xi[d]);
    for (int j = 0; j < 3; j++)
      for (int l = 0; l < 3; l++)
        h[j][l] = (j == l) ? 0.0 : 0.25 * hex_sign(a, j) * hex_sign(a, l) * f[3 - j - l];
  }
  __host__ __device__ static void shape(const double* xi, double* N, double (*dN)[3]) {
    for (int a = 0; a < 8; a++) {
      const double fx = 0.5 * (1.0 + hex_sign(a, 0) * xi[0]);
      const double fy = 0.5 * (1.0 + hex_sign(a, 1) * xi[1]);
      const double fz = 0.5 * (1.0 + hex_sign(a, 2) * xi[2]);
      N[a] = fx * fy * fz;
      dN[a][0] = 0.5 * hex_sign(a, 0) * fy * fz;
      dN[a][1] = 0.5 * hex_sign(a, 1) * fx * fz;
      dN[a][2] = 0.5 * hex_sign(a, 2) * fx * fy;
    }
  }
  __host__ __device__ static constexpr int vol_nq(int q) { return q * q * q; }
  __host__ __device__ static void vol_qp(int q, int i, double* xi, double& w) {
    double w0, w1, w2;
    gauss_legendre(q, i % q, xi[0], w0);
    gauss_legendre(q, (i / q) % q, xi[1], w1);
    gauss_legendre(q, i / (q * q), xi[2], w2);
    w = w0 * w1 * w2;
  }
  __host__ __device__ static constexpr int fac_nq(int q) { return q * q; }
  // faces: 0 x-, 1 x+, 2 y-, 3 y+, 4 z-, 5 z+  (reading L8)
  __host__ __device__ static void fac_qp(int q, int f, int i, double* xi, double& w, double* mref) {
    const int axis = f >> 1;
    const double side = (f & 1) ? 1.0 : -1.0;
    double s, t, ws, wt;
    gauss_legendre(q, i % q, s, ws);
    gauss_legendre(q, i / q, t, wt);
    const int a1 = (axis + 1) % 3, a2 = (axis + 2) % 3;
    xi[axis] = side;
    xi[a1] = s;
    xi[a2] = t;
    w = ws * wt;
    mref[0] = mref[1] = mref[2] = 0.0;
    mref[axis] = side;
  }
};

// ---------------------------------------------------------------- quadratic cubes (NEXT-2, reading L28)
// Node a sits at ξ = q_a ∈ {-1,0,1}³: corners in VTK order, the 12 edge midpoints of VTK's quadratic
// hexahedron, then (27-node) the face centres in facet order x-,x+,y-,y+,z-,z+ and the centre.
// Encoded as base-3 digits (q+1) per axis, x fastest: corners 0,2,8,6,18,20,26,24 etc.
constexpr int kQcCode[27] = {0, 2, 8, 6, 18, 20, 26, 24,                 // corners (---),(+--),(++-),(-+-),(--+)...
                             1, 5, 7, 3, 19, 23, 25, 21, 9, 11, 17, 15,  // edges (0,1),(1,2),(2,3),(3,0),(4,5)...(3,7)
                             12, 14, 10, 16, 4, 22, 13};                 // faces x-,x+,y-,y+,z-,z+; centre
// the digits (q+1 per axis, 2 bits each) of nodes 10w .. 10w+9 packed into one word at compile time, so a
// lookup is a shift and a mask (no per-call local array)
constexpr uint64_t qc_pack(int w) {
  uint64_t r = 0;
  for (int i = 0; i < 10 && 10 * w + i < 27; i++) {
    const int c = kQcCode[10 * w + i];
    r |= (uint64_t)((c % 3) | ((c / 3) % 3) << 2 | (c / 9) << 4) << (6 * i);
  }
  return r;
}
__host__ __device__ inline int qc_coord(int a, int d) {  // q_a,d ∈ {-1,0,1}
  constexpr uint64_t W0 = qc_pack(0), W1 = qc_pack(1), W2 = qc_pack(2);
  const uint64_t w = a < 10 ? W0 : a < 20 ? W1 : W2;
  return (int)((w >> (6 * (a % 10) + 2 * d)) & 3u) - 1;
}
// 1D quadratic Lagrange basis on {-1,0,1}: (value, first, second derivative) of node q at t
__host__ __device__ inline void lq1(int q, double t, double& v, double& d1, double& d2) {
  if (q == 0) { v = (1.0 - t) * (1.0 + t); d1 = -2.0 * t; d2 = -2.0; }
  else { v = 0.5 * t * (t + q); d1 = t + 0.5 * q; d2 = 1.0; }
}

// 27-node Lagrange cube: N_a = Π_d ℓ_{q_a,d}(ξ_d)
template <> struct Elem<ET_HEX, 2> {
  static constexpr int DIM = 3, NL = 27, NV = 8, NF = 6;
  static constexpr bool CURVED2 = true;
  __host__ __device__ static void shape(const double* xi, double* N, double (*dN)[3]) {
    double v[3][3], d1[3][3], d2[3][3];  // [axis][node coordinate + 1]
    for (int d = 0; d < 3; d++)
      for (int q = -1; q <= 1; q++) lq1(q, xi[d], v[d][q + 1], d1[d][q + 1], d2[d][q + 1]);
    for (int a = 0; a < 27; a++) {
      const int i = qc_coord(a, 0) + 1, j = qc_coord(a, 1) + 1, k = qc_coord(a, 2) + 1;
      N[a] = v[0][i] * v[1][j] * v[2][k];
      dN[a][0] = d1[0][i] * v[1][j] * v[2][k];
      dN[a][1] = v[0][i] * d1[1][j] * v[2][k];
      dN[a][2] = v[0][i] * v[1][j] * d1[2][k];
    }
  }
  __host__ __device__ static void node_hess(int a, const double* xi, double (*h)[3]) {
    double v[3], d1[3], d2[3];
    for (int d = 0; d < 3; d++) lq1(qc_coord(a, d), xi[d], v[d], d1[d], d2[d]);
    for (int j = 0; j < 3; j++)
      for (int l = 0; l < 3; l++) {
        const int m = 3 - j - l;
        h[j][l] = (j == l) ? d2[j] * v[(j + 1) % 3] * v[(j + 2) % 3] : d1[j] * d1[l] * v[m];
      }
  }
  __host__ __device__ static constexpr int vol_nq(int q) { return q * q * q; }
  __host__ __device__ static void vol_qp(int q, int i, double* xi, double& w) { Elem<ET_HEX, 1>::vol_qp(q, i, xi, w); }
  __host__ __device__ static constexpr int fac_nq(int q) { return q * q; }
  __host__ __device__ static void fac_qp(int q, int f, int i, double* xi, double& w, double* mref) {
    Elem<ET_HEX, 1>::fac_qp(q, f, i, xi, w, mref);
  }
};

// 20-node serendipity cube: corners N = ⅛ Π(1 + q_d ξ_d)(q·ξ - 2); edge midpoints (q_m = 0)
// N = ¼ (1 - ξ_m²) Π_{d≠m}(1 + q_d ξ_d).  Value / gradient / Hessian of one node from its three factors.
struct SerendipityNode {
  double N, g[3], h[3][3];
  __host__ __device__ SerendipityNode(int a, const double* xi) {
    double f[3], f1[3], f2[3];
    int q[3], zero = -1;
    for (int d = 0; d < 3; d++) {
      q[d] = qc_coord(a, d);
      if (q[d] == 0) { zero = d; f[d] = 1.0 - xi[d] * xi[d]; f1[d] = -2.0 * xi[d]; f2[d] = -2.0; }
      else { f[d] = 1.0 + q[d] * xi[d]; f1[d] = q[d]; f2[d] = 0.0; }
    }
    const double c = zero < 0 ? 0.125 : 0.25;
    double P = c * f[0] * f[1] * f[2], Pg[3], Ph[3][3];
    for (int j = 0; j < 3; j++)
      for (int l = 0; l < 3; l++) {
        const int m = 3 - j - l;
        Ph[j][l] = (j == l) ? c * f2[j] * f[(j + 1) % 3] * f[(j + 2) % 3] : c * f1[j] * f1[l] * f[m];
      }
    for (int j = 0; j < 3; j++) Pg[j] = c * f1[j] * f[(j + 1) % 3] * f[(j + 2) % 3];
    if (zero >= 0) {  // edge midpoint: the product itself
      N = P;
      for (int j = 0; j < 3; j++) {
        g[j] = Pg[j];
        for (int l = 0; l < 3; l++) h[j][l] = Ph[j][l];
      }
    } else {  // corner: product × (q·ξ - 2)
      const double s = q[0] * xi[0] + q[1] * xi[1] + q[2] * xi[2] - 2.0;
      N = P * s;
      for (int j = 0; j < 3; j++) {
        g[j] = Pg[j] * s + P * q[j];
        for (int l = 0; l < 3; l++) h[j][l] = Ph[j][l] * s + Pg[j] * q[l] + Pg[l] * q[j];
      }
    }
  }
};

template <> struct Elem<ET_HEXS, 2> {
  static constexpr int DIM = 3, NL = 20, NV = 8, NF = 6;
  static constexpr bool CURVED2 = true;
  __host__ __device__ static void shape(const double* xi, double* N, double (*dN)[3]) {
    for (int a = 0; a < 20; a++) {
      const SerendipityNode s(a, xi);
      N[a] = s.N;
      for (int d = 0; d < 3; d++) dN[a][d] = s.g[d];
    }
  }
  __host__ __device__ static void node_hess(int a, const double* xi, double (*h)[3]) {
    const SerendipityNode s(a, xi);
    for (int j = 0; j < 3; j++)
      for (int l = 0; l < 3; l++) h[j][l] = s.h[j][l];
  }
  __host__ __device__ static constexpr int vol_nq(int q) { return q * q * q; }
  __host__ __device__ static void vol_qp(int q, int i, double* xi, double& w) { Elem<ET_HEX, 1>::vol_qp(q, i, xi, w); }
  __host__ __device__ static constexpr int fac_nq(int q) { return q * q; }
  __host__ __device__ static void fac_qp(int q, int f, int i, double* xi, double& w, double* mref) {
    Elem<ET_HEX, 1>::fac_qp(q, f, i, xi, w, mref);
  }
};

}  // namespace fem
