// hex_tiled.cu — the c5/c2 hot path: Q1 hexahedra, 2x2x2 Gauss-Legendre points, node-tile owner
// gather (see tiled.cu) with a warp-synchronous element visit built around fp64 tensor-core MMA.
//
// PAPER.md D-3 for the elasticity form -(ε_ij, σ_ij) gives per element
//   K_(a,i),(b,m) = -f0 Σ_γ w [λ G_ai G_bm + μ G_am G_bi + μ δ_im G_a·G_b]
//                 = -f0 (λ M^im_ab + μ M^mi_ab + μ δ_im tr M_ab),   M^jk_ab = Σ_γ w_γ G_aj(γ) G_bk(γ),
// and for the thermal form -k(T_,i,T_,i) - C(T,T_t) K_ab = -k f0 Σ_j M^jj_ab - C f1 Σ_γ w N_a N_b.
// Lane l = 4a + c of a warp holds node a's gradient at Gauss points c and c+4, which is exactly the
// operand layout of mma.m8n8k4.f64 (A: row = l>>2, col = l&3; B: row = l&3, col = l>>2), so each 8x8
// tile M^jk (rows a, columns b) is two DMMA with the lane's own registers as A and B fragments; the
// accumulator fragment leaves lane l with M^jk_(a, 2c), M^jk_(a, 2c+1): the full 3x3 block of two pairs.
// The geometry (J, det J, J^-1 and the operand gradients) is computed with lane groups of
// 4 per Gauss point and shuffled to the fragment layout.  Visits are processed colour-synchronously
// (elements of one colour share no point), so the shared-memory accumulator takes plain adds and the
// result is bit-identical run to run.  Boundary terms reuse the generic warp path (tiled.cuh).
#include <algorithm>
#include <cstdlib>
#include <cuda/std/utility>
#include <string>
#include <type_traits>

#include "tiled.cuh"

namespace fem {

// acquire / release on a shared-memory turn counter (scope CTA)
__device__ __forceinline__ int ld_acquire_cta(const int* p) {
  int v;
  asm volatile("ld.acquire.cta.shared::cta.b32 %0, [%1];" : "=r"(v) : "r"((uint32_t)__cvta_generic_to_shared(p)) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_cta(int* p, int v) {
  asm volatile("st.release.cta.shared::cta.b32 [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(p)), "r"(v) : "memory");
}

__device__ __forceinline__ void dmma884(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

// Q1 shape value and reference gradient of node a at Gauss point q = ix + 2 iy + 4 iz (ξ = ±1/√3).
__device__ __forceinline__ void hex_ref(int a, int q, double (&g)[3], double& N) {
  const double r = 0.57735026918962576451;
  const double sx = hex_sign(a, 0), sy = hex_sign(a, 1), sz = hex_sign(a, 2);
  const double fx = 0.5 * (1.0 + sx * ((q & 1) ? r : -r));
  const double fy = 0.5 * (1.0 + sy * ((q & 2) ? r : -r));
  const double fz = 0.5 * (1.0 + sz * ((q & 4) ? r : -r));
  N = fx * fy * fz;
  g[0] = 0.5 * sx * fy * fz;
  g[1] = 0.5 * sy * fx * fz;
  g[2] = 0.5 * sz * fx * fy;
}

__device__ __forceinline__ double sum4(double v) {  // over the 4 lanes of a group (xor 1, 2)
  v += __shfl_xor_sync(0xffffffffu, v, 1);
  v += __shfl_xor_sync(0xffffffffu, v, 2);
  return v;
}

struct HexCoef {  // combined coefficients of the batch's domain forms
  double cl, cm;   // Σ f0 λ, Σ f0 μ            (elasticity matrix)
  double sl, sm;   // Σ λ, Σ μ                  (elasticity residual)
  double kf0, Cf1; // Σ k f0, Σ C f1            (thermal matrix)
};

// What one visit needs: its ownership / halo indices / local column offsets, the staged halo data
// and the tile accumulator (all in shared memory).
struct HexView {
  const int16_t* vown;   // [nv][8]
  const uint16_t* vhal;  // [nv][8]
  const int32_t* velem;  // [nv]
  const uint8_t* vloc;   // [nv][64] (shared) or nullptr -> global P.loc
  const double* hdat;    // [hcomp][H]
  int H;
  const int32_t* tdeg;
  const int32_t* toff;
  double* acc;
  double* racc;
  int T;
};

template <int KH, bool DET>
__device__ __forceinline__ void hex_visit(const TiledParams& P, const HexView& S, const HexCoef& H, int v) {
  const int lane = threadIdx.x & 31;
  const int16_t* own = S.vown + v * 8;
  const int e = S.velem[v];
  // ---- stage G: Gauss point q = lane >> 2, nodes sub and sub + 4
  const int q = lane >> 2, sub = lane & 3;
  double J[3][3], Dr[KH][3], xq[3] = {0, 0, 0}, Tt = 0.0;
#pragma unroll
  for (int i = 0; i < 3; i++)
#pragma unroll
    for (int j = 0; j < 3; j++) J[i][j] = 0.0;
#pragma unroll
  for (int k = 0; k < KH; k++)
#pragma unroll
    for (int j = 0; j < 3; j++) Dr[k][j] = 0.0;
  const uint16_t* hv = S.vhal + v * 8;
  const int HH = S.H;
#pragma unroll
  for (int t = 0; t < 2; t++) {
    const int a = sub + 4 * t, h = hv[a];
    double g[3], N;
    hex_ref(a, q, g, N);
    double X[3];
#pragma unroll
    for (int d = 0; d < 3; d++) X[d] = S.hdat[d * HH + h];
#pragma unroll
    for (int i = 0; i < 3; i++)
#pragma unroll
      for (int j = 0; j < 3; j++) J[i][j] = fma(X[i], g[j], J[i][j]);
#pragma unroll
    for (int k = 0; k < KH; k++) {
      const double D = S.hdat[(3 + k) * HH + h];
#pragma unroll
      for (int j = 0; j < 3; j++) Dr[k][j] = fma(D, g[j], Dr[k][j]);
    }
    if constexpr (KH == 1) {
#pragma unroll
      for (int d = 0; d < 3; d++) xq[d] = fma(N, X[d], xq[d]);
      if (P.nu_hat >= 1) Tt = fma(N, S.hdat[(3 + KH) * HH + h], Tt);
    }
  }
#pragma unroll
  for (int i = 0; i < 3; i++)
#pragma unroll
    for (int j = 0; j < 3; j++) J[i][j] = sum4(J[i][j]);
#pragma unroll
  for (int k = 0; k < KH; k++)
#pragma unroll
    for (int j = 0; j < 3; j++) Dr[k][j] = sum4(Dr[k][j]);
  if constexpr (KH == 1) {
#pragma unroll
    for (int d = 0; d < 3; d++) xq[d] = sum4(xq[d]);
    Tt = sum4(Tt);
  }
  const double c00 = J[1][1] * J[2][2] - J[1][2] * J[2][1];
  const double c01 = J[1][2] * J[2][0] - J[1][0] * J[2][2];
  const double c02 = J[1][0] * J[2][1] - J[1][1] * J[2][0];
  const double det = J[0][0] * c00 + J[0][1] * c01 + J[0][2] * c02;
  if (__any_sync(0xffffffffu, !(det > 0.0))) {
    if (lane == 0) atomicCAS((unsigned long long*)P.err, (unsigned long long)(-1LL), (unsigned long long)e);
    return;
  }
  const double rr = 1.0 / det;
  double Ji[3][3];
  Ji[0][0] = c00 * rr; Ji[1][0] = c01 * rr; Ji[2][0] = c02 * rr;
  Ji[0][1] = (J[0][2] * J[2][1] - J[0][1] * J[2][2]) * rr;
  Ji[1][1] = (J[0][0] * J[2][2] - J[0][2] * J[2][0]) * rr;
  Ji[2][1] = (J[0][1] * J[2][0] - J[0][0] * J[2][1]) * rr;
  Ji[0][2] = (J[0][1] * J[1][2] - J[0][2] * J[1][1]) * rr;
  Ji[1][2] = (J[0][2] * J[1][0] - J[0][0] * J[1][2]) * rr;
  Ji[2][2] = (J[0][0] * J[1][1] - J[0][1] * J[1][0]) * rr;
  const double w = det;  // Gauss-Legendre weight 1 per point
  // operand gradients ∇φ = Dr J^{-1}; point coefficients of the residual
  double Sq[3][3];  // elasticity: w σ_ij;  thermal: Sq[0][i] = w k ∇T_i, Sq[1][0] = w (s - C Ṫ)
#pragma unroll
  for (int k = 0; k < 3; k++)
#pragma unroll
    for (int i = 0; i < 3; i++) Sq[k][i] = 0.0;
  if constexpr (KH == 3) {
    double gu[3][3];
#pragma unroll
    for (int k = 0; k < 3; k++)
#pragma unroll
      for (int i = 0; i < 3; i++) gu[k][i] = Dr[k][0] * Ji[0][i] + Dr[k][1] * Ji[1][i] + Dr[k][2] * Ji[2][i];
    const double lw = H.sl * w * (gu[0][0] + gu[1][1] + gu[2][2]), mw = H.sm * w;
#pragma unroll
    for (int i = 0; i < 3; i++)
#pragma unroll
      for (int j = 0; j < 3; j++) Sq[i][j] = (i == j ? lw : 0.0) + mw * (gu[i][j] + gu[j][i]);
  } else {
    double gT[3];
#pragma unroll
    for (int i = 0; i < 3; i++) gT[i] = Dr[0][0] * Ji[0][i] + Dr[0][1] * Ji[1][i] + Dr[0][2] * Ji[2][i];
    double kk = 0.0, cn = 0.0;
    for (int f = 0; f < P.n_dom; f++) {
      const FormArgs& F = P.dom[f];
      double s = F.p[2];
      if (F.p[3] != 0.0) s *= sin(M_PI * xq[0]) * sin(M_PI * xq[1]) * sin(M_PI * xq[2]);
      kk += F.p[1];
      cn += s - (P.nu_hat >= 1 ? F.p[0] * Tt : 0.0);
    }
#pragma unroll
    for (int i = 0; i < 3; i++) Sq[0][i] = w * kk * gT[i];
    Sq[1][0] = w * cn;
  }
  // ---- fragment layout: node a = lane >> 2, Gauss points c and c + 4
  const int a = lane >> 2, c = lane & 3;
  const int s0 = 4 * c, s1 = 4 * c + 16;  // lanes holding points c and c+4 in the stage-G layout
  double G0[3], G1[3], N0, N1, g0[3], g1[3];
  hex_ref(a, c, g0, N0);
  hex_ref(a, c + 4, g1, N1);
  double w0 = __shfl_sync(0xffffffffu, w, s0), w1 = __shfl_sync(0xffffffffu, w, s1);
#pragma unroll
  for (int i = 0; i < 3; i++) { G0[i] = 0.0; G1[i] = 0.0; }
#pragma unroll
  for (int j = 0; j < 3; j++)
#pragma unroll
    for (int i = 0; i < 3; i++) {
      const double j0 = __shfl_sync(0xffffffffu, Ji[j][i], s0), j1 = __shfl_sync(0xffffffffu, Ji[j][i], s1);
      G0[i] = fma(j0, g0[j], G0[i]);
      G1[i] = fma(j1, g1[j], G1[i]);
    }
  const int li = own[a];
  // ---- residual rows (D-2): r_a = -Σ_γ w σ G_a (elasticity) | Σ_γ [N_a w(s - CṪ) - G_a·(w k ∇T)]
  if (P.rhs) {
    double r[KH];
    if constexpr (KH == 3) {
#pragma unroll
      for (int i = 0; i < 3; i++) {
        double t = 0.0;
#pragma unroll
        for (int j = 0; j < 3; j++) {
          t = fma(__shfl_sync(0xffffffffu, Sq[i][j], s0), G0[j], t);
          t = fma(__shfl_sync(0xffffffffu, Sq[i][j], s1), G1[j], t);
        }
        r[i] = -sum4(t);
      }
    } else {
      double t = N0 * __shfl_sync(0xffffffffu, Sq[1][0], s0) + N1 * __shfl_sync(0xffffffffu, Sq[1][0], s1);
#pragma unroll
      for (int j = 0; j < 3; j++) {
        t = fma(-G0[j], __shfl_sync(0xffffffffu, Sq[0][j], s0), t);
        t = fma(-G1[j], __shfl_sync(0xffffffffu, Sq[0][j], s1), t);
      }
      r[0] = sum4(t);
    }
    if (c == 0 && li >= 0) {
#pragma unroll
      for (int i = 0; i < KH; i++) {
        if constexpr (DET) S.racc[i * S.T + li] += r[i];
        else atomicAdd(S.racc + i * S.T + li, r[i]);
      }
    }
  }
  // ---- tangent (D-3): Gram tiles on the fp64 tensor cores
  if (P.values) {
    double Kb[2][KH][KH];
    if constexpr (KH == 3) {
      double M[3][3][2];
#pragma unroll
      for (int j = 0; j < 3; j++)
#pragma unroll
        for (int k = 0; k < 3; k++) {
          M[j][k][0] = 0.0;
          M[j][k][1] = 0.0;
          dmma884(M[j][k], w0 * G0[j], G0[k]);
          dmma884(M[j][k], w1 * G1[j], G1[k]);
        }
#pragma unroll
      for (int t = 0; t < 2; t++) {
        const double tr = M[0][0][t] + M[1][1][t] + M[2][2][t];
#pragma unroll
        for (int i = 0; i < 3; i++)
#pragma unroll
          for (int m = 0; m < 3; m++) Kb[t][i][m] = -(H.cl * M[i][m][t] + H.cm * M[m][i][t] + (i == m ? H.cm * tr : 0.0));
      }
    } else {
      double M[2] = {0.0, 0.0};
#pragma unroll
      for (int j = 0; j < 3; j++) {
        dmma884(M, w0 * G0[j], G0[j]);
        dmma884(M, w1 * G1[j], G1[j]);
      }
      double Mm[2] = {0.0, 0.0};
      if (H.Cf1 != 0.0) {
        dmma884(Mm, w0 * N0, N0);
        dmma884(Mm, w1 * N1, N1);
      }
#pragma unroll
      for (int t = 0; t < 2; t++) Kb[t][0][0] = -(H.kf0 * M[t] + H.Cf1 * Mm[t]);
    }
    if (li >= 0) {
      const int d = S.tdeg[li], sr = acc_row_stride(KH, d, P.nnz_s);
      double* base = S.acc + S.toff[li];
#pragma unroll
      for (int t = 0; t < 2; t++) {
        const int b = 2 * c + t;
        const int pos = S.vloc ? (int)S.vloc[v * 64 + a * 8 + b] : (int)__ldg(P.loc + (int64_t)e * 64 + a * 8 + b);
        double* rowb = base + pos;
#pragma unroll
        for (int i = 0; i < KH; i++)
#pragma unroll
          for (int m = 0; m < KH; m++) {
            if constexpr (DET) rowb[i * sr + m * d] += Kb[t][i][m];
            else atomicAdd(rowb + i * sr + m * d, Kb[t][i][m]);
          }
      }
    }
  }
}

constexpr int FACET_WARPS = 8;  // warps that take part in the (small) facet phase
constexpr int HEX_MAX_VISITS = 256;  // domain visits of one tile when boundary terms run inside the visits
constexpr int HEX_SCRATCH = 200;  // doubles of per-warp scratch of hex_visit_el2 (aliases the facet slots)
// exchanged gradient G_a,i(ξ_q) in the warp scratch: [i][q][a], a swizzled by bit 1 of q; w at 192 + q
__device__ __forceinline__ constexpr int hx_gx(int i, int q, int a) { return 64 * i + 8 * q + (a ^ (4 * ((q >> 1) & 1))); }
// Row r of the geometry GEMM output in the warp scratch: 24 r + (r >> 1), so the 4 x 4 lanes of a
// half-warp storing their accumulator fragments hit 16 distinct bank pairs.
__device__ __forceinline__ constexpr int hx_goff(int r) { return 24 * r + (r >> 1); }

// Reference-gradient B fragments of the geometry GEMM (constant per lane): for k-step s and n-tile t,
// lane l holds ∇̂N_a(ξ_q)_j with a = 4s + (l&3), (q, j) = divmod(8t + (l>>2), 3).
struct GeoFrag {
  double b[2][3];
};
__device__ __forceinline__ GeoFrag geo_frag() {
  GeoFrag F;
  const int l = threadIdx.x & 31;
#pragma unroll
  for (int s = 0; s < 2; s++)
#pragma unroll
    for (int t = 0; t < 3; t++) {
      const int a = 4 * s + (l & 3), n = 8 * t + (l >> 2), q = n / 3, j = n % 3;
      double g[3], N;
      hex_ref(a, q, g, N);
      F.b[s][t] = g[j];
    }
  return F;
}

// ---- persistent record-driven kernel: one CTA per SM walks the tiles; the next tile's packed record
// arrives by one TMA bulk copy and its halo points by LDGSTS while the current tile computes.
__device__ __forceinline__ void gather_halo(const TiledParams& P, const uint8_t* rec, double* hbuf) {
  const int32_t* hdr = reinterpret_cast<const int32_t*>(rec);
  const int H = hdr[1];
  const RecLayout L = rec_layout_hdr(8, hdr);
  const int32_t* hn = reinterpret_cast<const int32_t*>(rec + L.o_hnode);
  for (int c = 0; c < P.hcomp; c++) {  // component-major: no integer division per element
    const double* base = c < 3 ? P.coords + (int64_t)c * P.N : P.state + (int64_t)(c - 3) * P.N;
    for (int i = threadIdx.x; i < H; i += blockDim.x) cp_async8(hbuf + c * H + i, base + hn[i]);
  }
  cp_async_commit();
}

// Offsets (bytes from the dynamic shared-memory base) of the current tile's arrays: kept in shared
// memory so every visit addresses them with LDS and without rematerialising the record layout.
struct TileOffs {
  uint32_t vown, vhal, velem, vloc, hdat, tdeg, toff, acc, racc, vseq, turn, tnode, trps;
  int H, T;
};
// Per-lane constants of the fragment layout: B fragments of the geometry GEMM (6), ∇̂N_a at points c
// and c+4 (6) for lane l = 4a + c; ∇̂N_c and ∇̂N_(c+4) at point q (6) for l = 4q + c.
constexpr int LANE_TAB = 18;

// Boundary terms of the elasticity problem inside the owning element's visit ("boundary conditions are
// just the domain physics one dimension lower"; reading L18), for the forms of P:920-922:
// ELAST_FIX_ALL / ELAST_FIX_D1 (penalty τ, prescribed dʷ) add -f0 τ Σ_γ w N_a N_b δ_im to the lane's K
// entries and τ N_a (dʷ_i - d_i) to row (a, i) of the residual; ELAST_LOAD adds N_a σˡ_ij n_j.  Face
// points: Gauss-Legendre 2x2 on face f (axis f >> 1, side ±1; reading L8, L9); w = |det J J^-T m̂| and
// n = det J J^-T m̂ / w (Nanson).  fm holds bit 6 k + f for each face f of the element in boundary set k.
// Lane (a, c) receives K contributions in Kv (columns b = 2c + t) and fres[i] for its row a.
template <bool HAS_V, bool HAS_R>
__device__ __forceinline__ void hex_el_facets(const TiledParams& P, uint32_t fm, const double* hdat, int HH,
                                              const uint16_t* hv, double* sc, double (&Kv)[2][9], double (&fres)[3]) {
  const int lane = threadIdx.x & 31;
  const int a = lane >> 2, c = lane & 3;
  const double r = 0.57735026918962576451;
  for (int f = 0; f < P.n_fac; f++) {
    const FormArgs& F = P.fac[f];
    uint32_t faces = (fm >> (6 * P.fac_set[f])) & 63u;
    while (faces) {
      const int face = __ffs(faces) - 1;
      faces &= faces - 1;
      const int axis = face >> 1, a1 = (axis + 1) % 3, a2 = (axis + 2) % 3;
      const double side = (face & 1) ? 1.0 : -1.0;
      {  // geometry at face point q = lane >> 3 from node an = lane & 7 (reduced over the 8 lanes of q)
        const int q = lane >> 3, an = lane & 7;
        double xi[3];
        xi[axis] = side;
        xi[a1] = (q & 1) ? r : -r;
        xi[a2] = (q & 2) ? r : -r;
        const double sx = hex_sign(an, 0), sy = hex_sign(an, 1), sz = hex_sign(an, 2);
        const double fx = 0.5 * (1.0 + sx * xi[0]), fy = 0.5 * (1.0 + sy * xi[1]), fz = 0.5 * (1.0 + sz * xi[2]);
        const double Nn = fx * fy * fz, g[3] = {0.5 * sx * fy * fz, 0.5 * sy * fx * fz, 0.5 * sz * fx * fy};
        const int h = hv[an];
        double J[3][3], dq[3];
#pragma unroll
        for (int i = 0; i < 3; i++) {
          const double X = hdat[i * HH + h];
#pragma unroll
          for (int j = 0; j < 3; j++) J[i][j] = X * g[j];
          dq[i] = HAS_R ? Nn * hdat[(3 + i) * HH + h] : 0.0;
        }
#pragma unroll
        for (int o = 1; o < 8; o <<= 1) {
#pragma unroll
          for (int i = 0; i < 3; i++) {
#pragma unroll
            for (int j = 0; j < 3; j++) J[i][j] += __shfl_xor_sync(0xffffffffu, J[i][j], o);
            if (HAS_R) dq[i] += __shfl_xor_sync(0xffffffffu, dq[i], o);
          }
        }
        // Nanson: n dA = det J J^-T m̂, m̂ = side e_axis, so n_i dA = side (cofactor of J)_(i, axis)
        double cof[3];
        cof[0] = J[1][(axis + 1) % 3] * J[2][(axis + 2) % 3] - J[1][(axis + 2) % 3] * J[2][(axis + 1) % 3];
        cof[1] = J[2][(axis + 1) % 3] * J[0][(axis + 2) % 3] - J[2][(axis + 2) % 3] * J[0][(axis + 1) % 3];
        cof[2] = J[0][(axis + 1) % 3] * J[1][(axis + 2) % 3] - J[0][(axis + 2) % 3] * J[1][(axis + 1) % 3];
        const double nn = side * side * (cof[0] * cof[0] + cof[1] * cof[1] + cof[2] * cof[2]);
        const double dA = sqrt(nn);
        if (an == 0) {
          double* o = sc + q * 8;
          o[0] = dA;  // w: unit Gauss-Legendre weights
#pragma unroll
          for (int i = 0; i < 3; i++) { o[1 + i] = side * cof[i] / dA; o[4 + i] = dq[i]; }
        }
      }
      __syncwarp();
      const double tau = F.p[0];
#pragma unroll
      for (int q = 0; q < 4; q++) {
        const double* o = sc + q * 8;
        double xi[3];
        xi[axis] = side;
        xi[a1] = (q & 1) ? r : -r;
        xi[a2] = (q & 2) ? r : -r;
        auto Nf = [&](int n) {
          return 0.125 * (1.0 + hex_sign(n, 0) * xi[0]) * (1.0 + hex_sign(n, 1) * xi[1]) * (1.0 + hex_sign(n, 2) * xi[2]);
        };
        const double w = o[0], Na = Nf(a);
        if (F.form == FEM_WF_ELAST_FIX_ALL || F.form == FEM_WF_ELAST_FIX_D1) {
          if constexpr (HAS_V) {
#pragma unroll
            for (int t = 0; t < 2; t++) {
              const double kk = -F.f0 * tau * w * Na * Nf(2 * c + t);
              if (F.form == FEM_WF_ELAST_FIX_ALL) {
#pragma unroll
                for (int i = 0; i < 3; i++) Kv[t][i * 3 + i] += kk;
              } else {
                Kv[t][0] += kk;
              }
            }
          }
          if constexpr (HAS_R) {
            if (F.form == FEM_WF_ELAST_FIX_ALL) {
#pragma unroll
              for (int i = 0; i < 3; i++) fres[i] += w * tau * Na * (F.p[1 + i] - o[4 + i]);
            } else {
              fres[0] += w * tau * Na * (F.p[1] - o[4]);
            }
          }
        } else if (F.form == FEM_WF_ELAST_LOAD) {
          if constexpr (HAS_R) {
#pragma unroll
            for (int i = 0; i < 3; i++)
              fres[i] += w * Na * (F.p[3 * i] * o[1] + F.p[3 * i + 1] * o[2] + F.p[3 * i + 2] * o[3]);
          }
        }
      }
      __syncwarp();  // the face-point scratch is rewritten by the next face
    }
  }
}

// Call kinds, fixed per launch so each visit body is compiled lean: matrix only, residual only, system with
// the residual fused into the scatter (f0 = 1), system with the stress-GEMM residual (f0 != 1).
enum { HX_MAT = 0, HX_RES = 1, HX_SYS_FUSED = 2, HX_SYS = 3 };

// SW (sweep records, sweep.cu): the turn of each (visit, node) comes from the 16-bit vseq with the row's
// first-touch (bit 14) and last-touch (bit 15) flags; bit 7 of the local column offset marks the first
// contribution to a 3x3 block of the row's current life (stored, not added: no zeroing pass); the visit
// that makes the last touch of a row writes the completed row to HBM before passing the turn on (the
// ring slot's next occupant starts with the next turn), so no step needs a block-wide epilogue.
// SWSR > 0 (sweep rings): every row uses the fixed layout of a 27-column row — entry (i, m, col) at
// i·SWSR + 27·m + col, SWSR = 81 or 82 (the parity of 3·nnz_s) — so the 18 read-modify-writes of a lane
// address with immediates; rows with fewer columns (mesh boundary) are compacted when written out.
template <bool DET, int MODE, bool ORDERED = DET, bool SW = false, int SWSR = 0>
__device__ __forceinline__ void hex_visit_el2(const TiledParams& P, const TileOffs& to, const HexCoef& H,
                                              const double* __restrict__ lt, double* sc, int v,
                                              unsigned char* sm, const uint32_t* vfm) {
  const int lane = threadIdx.x & 31;
  const int16_t* own = reinterpret_cast<const int16_t*>(sm + to.vown) + v * 8;
  const uint16_t* hv = reinterpret_cast<const uint16_t*>(sm + to.vhal) + v * 8;
  const double* hdat = reinterpret_cast<const double*>(sm + to.hdat);
  const int HH = to.H;
  const int c = lane & 3, r = lane >> 2;
  const double* L = lt + lane;  // lane table, transposed: L[32 k] = constant k of this lane
  // The form is linear in d: r_(a,i) = Σ_(b,m) K'_(a,i),(b,m) d_(b,m) with K' = K at f0 = 1.  With f0 = 1
  // (static) K' is the K being written, so a system call accumulates the residual in the scatter loop
  // (lane-local over the lane's two columns b, then over the four lanes of the row); otherwise the
  // residual is the GEMM of the gradients with the per-point stress w σ (below).
  constexpr bool fuse = MODE == HX_SYS_FUSED, has_rhs = MODE != HX_MAT, has_values = MODE != HX_RES;
  // stress mode: per-point record stride (doubles) J^-1, w, w σ; even (16-byte loads) and ≡ 2·odd mod 16,
  // so the eight writer lanes (one per point) hit distinct bank pairs
  constexpr bool stress = has_rhs && !fuse;  // residual from the per-point stress (residual-only, f0 != 1)
  constexpr int RS = 22;
  // ---- geometry GEMM: A[r][a] = component r of point a (x,y,z,d1,d2,d3; rows 6,7 zero)
  double C3[3][2];
#pragma unroll
  for (int t = 0; t < 3; t++) { C3[t][0] = 0.0; C3[t][1] = 0.0; }
#pragma unroll
  for (int s = 0; s < 2; s++) {
    const double av = r < 6 ? hdat[r * HH + hv[4 * s + c]] : 0.0;
#pragma unroll
    for (int t = 0; t < 3; t++) dmma884(C3[t], av, L[32 * (s * 3 + t)]);
  }
  if (r < 6) {
#pragma unroll
    for (int t = 0; t < 3; t++) {
      sc[hx_goff(r) + 8 * t + 2 * c] = C3[t][0];
      sc[hx_goff(r) + 8 * t + 2 * c + 1] = C3[t][1];
    }
  }
  __syncwarp();
  const int q = r;
  double J[3][3], Dr[3][3];
#pragma unroll
  for (int i = 0; i < 3; i++)
#pragma unroll
    for (int j = 0; j < 3; j++) {
      J[i][j] = sc[hx_goff(i) + 3 * q + j];
      Dr[i][j] = sc[hx_goff(3 + i) + 3 * q + j];
    }
  const double c00 = J[1][1] * J[2][2] - J[1][2] * J[2][1];
  const double c01 = J[1][2] * J[2][0] - J[1][0] * J[2][2];
  const double c02 = J[1][0] * J[2][1] - J[1][1] * J[2][0];
  const double det = J[0][0] * c00 + J[0][1] * c01 + J[0][2] * c02;
  if (__any_sync(0xffffffffu, !(det > 0.0))) {
    if (lane == 0)
      atomicCAS((unsigned long long*)P.err, (unsigned long long)(-1LL),
                (unsigned long long)reinterpret_cast<const int32_t*>(sm + to.velem)[v]);
    if constexpr (ORDERED) {  // still pass the turn on, or later visits of these rows would wait forever
      const int li = own[r];
      if (c == 0 && li >= 0) {
        volatile int* tp = reinterpret_cast<volatile int*>(sm + to.turn) + li;
        const int t = SW ? (int)(reinterpret_cast<const uint16_t*>(sm + to.vseq)[v * 8 + r] & 0x3fff)
                         : (int)(sm + to.vseq)[v * 8 + r];
        while (*tp != t) __nanosleep(64);
        *tp = t + 1;
      }
    }
    __syncwarp();
    return;
  }
  __syncwarp();  // everyone has read the GEMM output; the scratch now takes the per-point records
  const double rr = 1.0 / det;
  double Ji[3][3];  // Ji[j][i] = (J^-1)_ji, in every lane of point group q
  Ji[0][0] = c00 * rr; Ji[1][0] = c01 * rr; Ji[2][0] = c02 * rr;
  Ji[0][1] = (J[0][2] * J[2][1] - J[0][1] * J[2][2]) * rr;
  Ji[1][1] = (J[0][0] * J[2][2] - J[0][2] * J[2][0]) * rr;
  Ji[2][1] = (J[0][1] * J[2][0] - J[0][0] * J[2][1]) * rr;
  Ji[0][2] = (J[0][1] * J[1][2] - J[0][2] * J[1][1]) * rr;
  Ji[1][2] = (J[0][2] * J[1][0] - J[0][0] * J[1][2]) * rr;
  Ji[2][2] = (J[0][0] * J[1][1] - J[0][1] * J[1][0]) * rr;
  const int a = r;
  double G0[3], G1[3], w0, w1;
  if constexpr (!stress) {
    // gradient exchange: lane (q, c) forms G_a(q) = J^-T ∇̂N_a(ξ_q) for a = c, c + 4 and stores it at
    // [i][q][a ^ 4((q >> 1) & 1)] (the swizzle makes stores and loads conflict-free); lane (a, c) then
    // loads G_a at its points c and c + 4 — the A/B fragment layout of the Gram GEMM
#pragma unroll
    for (int h = 0; h < 2; h++)
#pragma unroll
      for (int i = 0; i < 3; i++)
        sc[hx_gx(i, q, c + 4 * h)] = Ji[0][i] * L[32 * (12 + 3 * h)] + Ji[1][i] * L[32 * (13 + 3 * h)] + Ji[2][i] * L[32 * (14 + 3 * h)];
    if (c == 0) sc[192 + q] = det;  // w (unit Gauss-Legendre weights)
    __syncwarp();
#pragma unroll
    for (int i = 0; i < 3; i++) {
      G0[i] = sc[hx_gx(i, c, a)];
      G1[i] = sc[hx_gx(i, c + 4, a)];
    }
    w0 = sc[192 + c];
    w1 = sc[196 + c];
  } else {
    if (c == 0) {
      double* o = sc + q * RS;  // per-point records (the GEMM output has been consumed)
#pragma unroll
      for (int j = 0; j < 3; j++)
#pragma unroll
        for (int i = 0; i < 3; i++) o[j * 3 + i] = Ji[j][i];
      o[9] = det;  // w (unit Gauss-Legendre weights)
      // w σ_ij at the point: B operand of the residual GEMM below
      double gu[3][3];
#pragma unroll
      for (int k = 0; k < 3; k++)
#pragma unroll
        for (int i = 0; i < 3; i++) gu[k][i] = Dr[k][0] * Ji[0][i] + Dr[k][1] * Ji[1][i] + Dr[k][2] * Ji[2][i];
      const double lw = H.sl * det * (gu[0][0] + gu[1][1] + gu[2][2]), mw = H.sm * det;
#pragma unroll
      for (int i = 0; i < 3; i++)
#pragma unroll
        for (int j = 0; j < 3; j++) o[10 + i * 3 + j] = (i == j ? lw : 0.0) + mw * (gu[i][j] + gu[j][i]);
    }
    __syncwarp();
    // ---- fragment layout: node a = lane >> 2, points c and c + 4
    const double* o0 = sc + c * RS;
    const double* o1 = sc + (c + 4) * RS;
    double R0[10], R1[10];  // J^-1 (9) and w of points c and c + 4: 16-byte loads of broadcast records
#pragma unroll
    for (int k = 0; k < 5; k++) {
      const double2 x0 = reinterpret_cast<const double2*>(o0)[k], x1 = reinterpret_cast<const double2*>(o1)[k];
      R0[2 * k] = x0.x; R0[2 * k + 1] = x0.y;
      R1[2 * k] = x1.x; R1[2 * k + 1] = x1.y;
    }
#pragma unroll
    for (int i = 0; i < 3; i++) {
      G0[i] = R0[0 * 3 + i] * L[32 * 6] + R0[1 * 3 + i] * L[32 * 7] + R0[2 * 3 + i] * L[32 * 8];
      G1[i] = R1[0 * 3 + i] * L[32 * 9] + R1[1 * 3 + i] * L[32 * 10] + R1[2 * 3 + i] * L[32 * 11];
    }
    w0 = R0[9];
    w1 = R1[9];
  }
  const int li = own[a];
  // r_(a,i) = -Σ_γ Σ_j G_aj(γ) [w σ_ij](γ): a (8 nodes × 24) · (24 × 3) product, 6 DMMA whose A
  // fragments are the lane's own gradients (k = point) and whose B fragments are the per-point stress
  // rows i = lane >> 2 (zero for i >= 3); lane (a, c) receives r_(a, 2c) and r_(a, 2c + 1).
  double res[3] = {0.0, 0.0, 0.0};
  if constexpr (stress) {
    const double* o0 = sc + c * RS;
    const double* o1 = sc + (c + 4) * RS;
    double r2[2] = {0.0, 0.0};
#pragma unroll
    for (int j = 0; j < 3; j++) {
      dmma884(r2, G0[j], r < 3 ? o0[10 + r * 3 + j] : 0.0);
      dmma884(r2, G1[j], r < 3 ? o1[10 + r * 3 + j] : 0.0);
    }
    res[0] = r2[0];
    res[1] = r2[1];
  }
  // K entries before taking the turn (the critical section is the read-modify-write only):
  // M^jk_ab = Σ_γ w G_aj G_bk (18 DMMA), K_(a,i),(b,m) = -(cl M^im + cm M^mi + δ_im cm tr M) for the
  // lane's columns b = 2c + t; with fuse, the lane's part of r = K'd as well.
  double Kv[2][9];
  if constexpr (has_values) {
    double M[3][3][2];
#pragma unroll
    for (int j = 0; j < 3; j++)
#pragma unroll
      for (int k = 0; k < 3; k++) {
        M[j][k][0] = 0.0;
        M[j][k][1] = 0.0;
        dmma884(M[j][k], w0 * G0[j], G0[k]);
        dmma884(M[j][k], w1 * G1[j], G1[k]);
      }
#pragma unroll
    for (int t = 0; t < 2; t++) {
      const double tr = M[0][0][t] + M[1][1][t] + M[2][2][t];
#pragma unroll
      for (int i = 0; i < 3; i++)
#pragma unroll
        for (int m = 0; m < 3; m++) Kv[t][i * 3 + m] = -(H.cl * M[i][m][t] + H.cm * M[m][i][t] + (i == m ? H.cm * tr : 0.0));
    }
    if constexpr (fuse) {
#pragma unroll
      for (int t = 0; t < 2; t++) {
        const int hb = hv[2 * c + t];
#pragma unroll
        for (int m = 0; m < 3; m++) {
          const double dv = hdat[(3 + m) * HH + hb];
#pragma unroll
          for (int i = 0; i < 3; i++) res[i] = fma(Kv[t][i * 3 + m], dv, res[i]);
        }
      }
#pragma unroll
      for (int i = 0; i < 3; i++) res[i] = sum4(res[i]);
    }
  }
  double fres[3] = {0.0, 0.0, 0.0};  // boundary-term residual of row a (every lane of the row)
  if (vfm) {
    const uint32_t fm = vfm[v];
    if (fm) {
      __syncwarp();  // every lane is done with the per-point records in the scratch
      hex_el_facets<has_values, has_rhs>(P, fm, hdat, HH, hv, sc, Kv, fres);
    }
  }
  int* turn = reinterpret_cast<int*>(sm + to.turn);
  int my_turn = 0;
  unsigned sw_flags = 0;  // SW: bit 14 first touch of the row's life, bit 15 last touch
  if constexpr (ORDERED) {  // wait for this visit's turn on the owned row it writes (record order)
    if (li >= 0) {
      if constexpr (SW) {
        const unsigned w = reinterpret_cast<const uint16_t*>(sm + to.vseq)[v * 8 + a];
        my_turn = (int)(w & 0x3fffu);
        sw_flags = w;
      } else {
        my_turn = (sm + to.vseq)[v * 8 + a];
      }
      while (ld_acquire_cta(turn + li) != my_turn)  // acquire: the previous holder's row writes are visible
        if (P.spin_ns) __nanosleep(P.spin_ns);
    }
  }
  const bool row_first = SW && (sw_flags & (1u << 14));
  auto write_res = [&]() {  // GEMM residual: lane (a, c < 2) holds r_(a, 2c), r_(a, 2c + 1)
    if (has_rhs && !fuse && c < 2 && li >= 0) {
      double* racc = reinterpret_cast<double*>(sm + to.racc) + li + 2 * c * to.T;
      if constexpr (DET) {
        racc[0] = (row_first ? 0.0 : racc[0]) + ((c == 0 ? fres[0] : fres[2]) - res[0]);
        if (c == 0) racc[to.T] = (row_first ? 0.0 : racc[to.T]) + (fres[1] - res[1]);
      } else {
        atomicAdd(racc, (c == 0 ? fres[0] : fres[2]) - res[0]);
        if (c == 0) atomicAdd(racc + to.T, fres[1] - res[1]);
      }
    }
  };
  write_res();
  if constexpr (has_values) {
    if (li >= 0) {
      const int d = SWSR ? 27 : reinterpret_cast<const int32_t*>(sm + to.tdeg)[li];
      const int sr = SWSR ? SWSR : acc_row_stride(3, d, P.nnz_s);
      double* base = reinterpret_cast<double*>(sm + to.acc) + reinterpret_cast<const int32_t*>(sm + to.toff)[li];
      const uint8_t* lc = sm + to.vloc + v * 64 + a * 8 + 2 * c;
#pragma unroll
      for (int t = 0; t < 2; t++) {
        const unsigned lct = lc[t];
        double* rowb = base + (SW ? (lct & 0x7fu) : lct);
        if constexpr (DET) {  // independent read-modify-writes: loads first (d may alias for the compiler)
          const bool first = SW && (lct & 0x80u);  // first contribution to this block: store
#pragma unroll
          for (int i = 0; i < 3; i++) {
            double old[3];
#pragma unroll
            for (int m = 0; m < 3; m++) old[m] = first ? 0.0 : rowb[i * sr + m * d];
#pragma unroll
            for (int m = 0; m < 3; m++) rowb[i * sr + m * d] = old[m] + Kv[t][i * 3 + m];
          }
        } else {
#pragma unroll
          for (int e = 0; e < 9; e++) atomicAdd(rowb + (e / 3) * sr + (e % 3) * d, Kv[t][e]);
        }
      }
      if constexpr (fuse) {
        if (c == 0) {
          double* racc = reinterpret_cast<double*>(sm + to.racc) + li;
#pragma unroll
          for (int i = 0; i < 3; i++) {
            if constexpr (DET) racc[i * to.T] = (row_first ? 0.0 : racc[i * to.T]) + (res[i] + fres[i]);
            else atomicAdd(racc + i * to.T, res[i] + fres[i]);
          }
        }
      }
    }
  }
  __syncwarp();  // scratch is reused by the next visit; the row's four lanes have written
  if constexpr (SW) {
    // the rows this visit completes (last touch of their life) leave to HBM now: one TMA bulk store per
    // sub-row (its aligned middle; the 16-byte phase of the ring copy equals the destination's, see
    // acc_row_stride) plus at most two single doubles, issued by lane 0, which waits until the TMA has read
    // the ring before the turn passes on (the position's next life starts by storing into it).  Every
    // accumulator write of every visit is followed by a proxy fence (generic -> async proxy).
    fence_proxy_async_smem();
    __syncwarp();
    unsigned lastm = __ballot_sync(0xffffffffu, c == 0 && li >= 0 && (sw_flags & (1u << 15)));
    if (lastm) {
      const int32_t* tn = reinterpret_cast<const int32_t*>(sm + to.tnode);
      const int64_t* trp = reinterpret_cast<const int64_t*>(sm + to.trps);
      bool issued = false;
      while (lastm) {
        const int src_lane = __ffs(lastm) - 1;
        lastm &= lastm - 1;
        const int rl = own[src_lane >> 2];
        if constexpr (has_values) {
          const int d = reinterpret_cast<const int32_t*>(sm + to.tdeg)[rl];
          const int sr = SWSR ? SWSR : acc_row_stride(3, d, P.nnz_s);
          const double* srow = reinterpret_cast<const double*>(sm + to.acc) + reinterpret_cast<const int32_t*>(sm + to.toff)[rl];
          double* drow = P.values + (int64_t)3 * trp[rl];
          if (!SWSR || d == 27) {
            if (lane < 3) {  // lane k0 writes sub-row k0
              const double* s0 = srow + lane * sr;
              double* dst = drow + (int64_t)lane * 3 * P.nnz_s;
              const int len = 3 * d;
              const int head = ((uintptr_t)dst & 15) ? 1 : 0;
              const int mid = (len - head) & ~1;
              bulk_s2g(dst + head, s0 + head, 8u * (uint32_t)mid);
              issued = true;
              if (head) dst[0] = s0[0];
              if (head + mid < len) dst[len - 1] = s0[len - 1];
            }
          } else {  // a boundary row (d < 27) in the fixed 27-column layout: compact it while storing
            for (int idx = lane; idx < 9 * d; idx += 32) {
              const int k0 = idx / (3 * d), rem = idx - k0 * 3 * d, m = rem / d, col = rem - m * d;
              drow[(int64_t)k0 * 3 * P.nnz_s + rem] = srow[k0 * sr + 27 * m + col];
            }
          }
        }
        if (has_rhs && lane < 3)
          P.rhs[(int64_t)lane * P.n_own + (tn[rl] - P.own_lo)] =
              reinterpret_cast<const double*>(sm + to.racc)[rl + lane * to.T];
      }
      if (issued) {
        bulk_commit();
        bulk_wait_read_all();
      }
    }
    __syncwarp();  // the ring copies have been read: the positions' next lives may overwrite them
  }
  if constexpr (ORDERED) {  // hand the row to the next visit in record order: a release store, cumulative
    // over the row's four lanes whose writes this lane has observed through __syncwarp
    if (c == 0 && li >= 0) st_release_cta(turn + li, my_turn + 1);
  }
}

#ifndef FEM_HEX_THREADS
#define FEM_HEX_THREADS 512
#endif
constexpr int HEX_THREADS = FEM_HEX_THREADS;  // threads of the persistent hex kernel
constexpr int HEX_WARPS = HEX_THREADS / 32;

template <bool DET, int MODE>
__device__ __forceinline__ void hex_visits(const TiledParams& P, const TileOffs& to, const HexCoef& Hc,
                                           const double* lanetab, double* wsc, unsigned char* smem, int nv, int warp,
                                           const uint32_t* vfm) {
  for (int v = warp; v < nv; v += HEX_WARPS) hex_visit_el2<DET, MODE>(P, to, Hc, lanetab, wsc, v, smem, vfm);  // static split
}

template <int KH, bool DET>
__global__ void __launch_bounds__(HEX_THREADS, 1) k_hex_rec(const __grid_constant__ TiledParams P) {
  using C = TileCfg<ET_HEX, 1, KH, 2>;
  extern __shared__ __align__(16) unsigned char smem[];
  uint64_t* mbar = reinterpret_cast<uint64_t*>(smem);
  int* ctr = reinterpret_cast<int*>(smem + 64);
  __shared__ TileOffs to;
  __shared__ double lanetab[32 * LANE_TAB];
  __shared__ uint32_t vfmask[HEX_MAX_VISITS];  // in-visit boundary terms: bit 6 k + face per domain visit
#define RBUF(i) (smem + 128 + (size_t)(i) * P.rec_cap)
#define HBUF(i) (reinterpret_cast<double*>(smem + 128 + 2 * (size_t)P.rec_cap) + (size_t)(i) * P.hcap)
  double* acc = HBUF(2);
  // facet-phase arrays (generic warp path)
  TileSmem F;
  int* turn = reinterpret_cast<int*>(acc + P.acc_cap);
  unsigned char* fp = reinterpret_cast<unsigned char*>(turn + P.turn_cap);
  F.qp = fp;
  fp += std::max((size_t)P.rec_bytes * FACET_WARPS, (size_t)8 * HEX_SCRATCH * HEX_WARPS);
  F.vid = reinterpret_cast<int32_t*>(fp);
  fp += 4 * (size_t)P.fvmax;
  F.vnode = reinterpret_cast<int32_t*>(fp);
  fp += 4 * (size_t)P.fvmax * 8;
  F.vown = reinterpret_cast<int16_t*>(fp);
  fp += 2 * (size_t)P.fvmax * 8;
  F.vfac = reinterpret_cast<int8_t*>(fp);
  F.vhal = nullptr;
  F.hnode = nullptr;
  F.hdat = nullptr;
  F.H = 0;
  HexCoef Hc = {0, 0, 0, 0, 0, 0};
  for (int f = 0; f < P.n_dom; f++) {
    const FormArgs& Fm = P.dom[f];
    Hc.cl += Fm.f0 * Fm.lam; Hc.cm += Fm.f0 * Fm.mu; Hc.sl += Fm.lam; Hc.sm += Fm.mu;
    Hc.kf0 += Fm.p[1] * Fm.f0;
    if (Fm.nu_hat >= 1) Hc.Cf1 += Fm.p[0] * Fm.f1;
  }
  const int hmode = !P.rhs ? HX_MAT : !P.values ? HX_RES : (Hc.cl == Hc.sl && Hc.cm == Hc.sm) ? HX_SYS_FUSED : HX_SYS;
  const int tid = threadIdx.x, warp = tid >> 5;
  const GeoFrag GF = geo_frag();
  if (warp == 0) {  // per-lane constant table (same for every warp)
    double* Lt = lanetab + tid;  // transposed (constant k of lane l at 32 k + l): conflict-free loads
#pragma unroll
    for (int s = 0; s < 2; s++)
#pragma unroll
      for (int t = 0; t < 3; t++) Lt[32 * (s * 3 + t)] = GF.b[s][t];
    double g0[3], g1[3], N0, N1;
    hex_ref(tid >> 2, tid & 3, g0, N0);
    hex_ref(tid >> 2, (tid & 3) + 4, g1, N1);
    for (int i = 0; i < 3; i++) { Lt[32 * (6 + i)] = g0[i]; Lt[32 * (9 + i)] = g1[i]; }
    double gc[3], gc4[3], Nc, Nc4;  // writer role of the gradient exchange: lane 4q + c, nodes c and c + 4 at point q
    hex_ref(tid & 3, tid >> 2, gc, Nc);
    hex_ref((tid & 3) + 4, tid >> 2, gc4, Nc4);
    for (int i = 0; i < 3; i++) { Lt[32 * (12 + i)] = gc[i]; Lt[32 * (15 + i)] = gc4[i]; }
  }
  int64_t tile = blockIdx.x;
  if (tile >= P.n_tiles) return;
  if (tid == 0) {
    mbar_init(&mbar[0], 1);
    mbar_init(&mbar[1], 1);
    mbar_fence_init();
  }
  __syncthreads();
  if (tid == 0) {
    const uint32_t bytes = (uint32_t)(P.rec_off[tile + 1] - P.rec_off[tile]);
    mbar_expect_tx(&mbar[0], bytes);
    bulk_g2s(RBUF(0), P.rec + P.rec_off[tile], bytes, &mbar[0]);
  }
  mbar_wait(&mbar[0], 0);
  gather_halo(P, RBUF(0), HBUF(0));
  for (int it = 0; tile < P.n_tiles; it++) {
    const int cur = it & 1, oth = cur ^ 1;
    const int64_t next = tile + gridDim.x;
    if (tid == 0 && next < P.n_tiles) {  // prefetch the next record (its buffer was released last iteration)
      const uint32_t bytes = (uint32_t)(P.rec_off[next + 1] - P.rec_off[next]);
      mbar_expect_tx(&mbar[oth], bytes);
      bulk_g2s(RBUF(oth), P.rec + P.rec_off[next], bytes, &mbar[oth]);
    }
    const uint8_t* rec = RBUF(cur);
    const int32_t* hdr = reinterpret_cast<const int32_t*>(rec);
    const int T = hdr[0], H = hdr[1], nv = hdr[2], nr = hdr[3], acc_n = P.values ? hdr[4] : 0;
    const uint32_t fmask = (uint32_t)hdr[5];
    const RecLayout L = rec_layout_hdr(8, hdr);
    HexView V;
    V.vown = reinterpret_cast<const int16_t*>(rec + L.o_vown);
    V.vhal = reinterpret_cast<const uint16_t*>(rec + L.o_vhal);
    V.velem = reinterpret_cast<const int32_t*>(rec + L.o_velem);
    V.vloc = rec + L.o_vloc;
    V.hdat = HBUF(cur);
    V.H = H;
    V.tdeg = reinterpret_cast<const int32_t*>(rec + L.o_tdeg);
    V.toff = reinterpret_cast<const int32_t*>(rec + L.o_toff);
    V.acc = acc;
    V.racc = acc + acc_n;
    V.T = T;
    if (tid == 0) {
      *ctr = 0;
      const uint32_t rb = (uint32_t)(rec - smem);
      to.vown = rb + L.o_vown; to.vhal = rb + L.o_vhal; to.velem = rb + L.o_velem; to.vloc = rb + L.o_vloc;
      to.hdat = (uint32_t)(reinterpret_cast<const unsigned char*>(HBUF(cur)) - smem);
      to.tdeg = rb + L.o_tdeg; to.toff = rb + L.o_toff;
      to.acc = (uint32_t)(reinterpret_cast<unsigned char*>(acc) - smem);
      to.racc = to.acc + 8u * (uint32_t)acc_n;
      to.vseq = rb + L.o_vseq;
      to.turn = (uint32_t)(reinterpret_cast<unsigned char*>(turn) - smem);
      to.H = H;
      to.T = T;
    }
    for (int i = tid; i < (acc_n + KH * T + 1) / 2; i += blockDim.x)  // acc is 16-byte aligned, acc_cap even
      reinterpret_cast<double2*>(acc)[i] = make_double2(0.0, 0.0);
    if constexpr (DET)
      for (int i = tid; i < T; i += blockDim.x) turn[i] = 0;
    const bool finl = P.fac_inline && fmask;
    if (finl)
      for (int i = tid; i < nv; i += blockDim.x) vfmask[i] = 0u;
    cp_async_wait_all();
    __syncthreads();
    if (finl) {  // facet visit i of set k is face ffac[i] of domain visit fdv[i] (record layout)
      const int32_t* fcnt = reinterpret_cast<const int32_t*>(rec + L.o_fcnt);
      const int16_t* fdv = reinterpret_cast<const int16_t*>(rec + L.o_fdv);
      const int8_t* ffac = reinterpret_cast<const int8_t*>(rec + L.o_ffac);
      for (int k = 0; k < hdr[6]; k++)
        for (int i = fcnt[k] + tid; i < fcnt[k + 1]; i += blockDim.x) atomicOr(&vfmask[fdv[i]], 1u << (6 * k + ffac[i]));
      __syncthreads();
    }
    const uint32_t* vf = finl ? vfmask : nullptr;
    const int32_t* run = reinterpret_cast<const int32_t*>(rec + L.o_run);
    double* wsc = reinterpret_cast<double*>(F.qp) + (size_t)HEX_SCRATCH * warp;
    if constexpr (KH == 3) {
      // DET: visit v takes its turn on each accumulator row it writes (vseq), so every entry sums its
      // contributions in record order with plain adds, without block-wide barriers between colours
      switch (hmode) {
        case HX_MAT: hex_visits<DET, HX_MAT>(P, to, Hc, lanetab, wsc, smem, nv, warp, vf); break;
        case HX_RES: hex_visits<DET, HX_RES>(P, to, Hc, lanetab, wsc, smem, nv, warp, vf); break;
        case HX_SYS_FUSED: hex_visits<DET, HX_SYS_FUSED>(P, to, Hc, lanetab, wsc, smem, nv, warp, vf); break;
        default: hex_visits<DET, HX_SYS>(P, to, Hc, lanetab, wsc, smem, nv, warp, vf); break;
      }
    } else if constexpr (DET) {
      for (int r = 0; r < nr; r++) {  // colour runs: conflict-free, plain shared-memory adds
        for (int v = run[r] + warp; v < run[r + 1]; v += HEX_WARPS) hex_visit<KH, true>(P, V, Hc, v);
        __syncthreads();
      }
    } else {
      for (int v = warp; v < nv; v += HEX_WARPS) hex_visit<KH, false>(P, V, Hc, v);  // uniform: static split
    }
    if (next < P.n_tiles) {  // the next record has (almost surely) landed: start its halo gather
      mbar_wait(&mbar[oth], (uint32_t)(((it + 1) >> 1) & 1));
      gather_halo(P, RBUF(oth), HBUF(oth));
    }
    // shared-memory view of the tile for the facet phase and the epilogue
    F.tnode = const_cast<int32_t*>(reinterpret_cast<const int32_t*>(rec + L.o_tnode));
    F.tdeg = const_cast<int32_t*>(V.tdeg);
    F.toff = const_cast<int32_t*>(V.toff);
    F.trps = const_cast<int64_t*>(reinterpret_cast<const int64_t*>(rec + L.o_trps));
    F.acc = acc;
    F.racc = V.racc;
    F.T = T;
    F.vid = const_cast<int32_t*>(V.velem);
    F.vown = const_cast<int16_t*>(V.vown);
    F.vhal = const_cast<int16_t*>(reinterpret_cast<const int16_t*>(V.vhal));
    F.vloc = V.vloc;
    F.hdat = const_cast<double*>(V.hdat);
    F.H = H;
    if (fmask && !P.fac_inline)  // DET: node-disjoint facet segments, one barrier each
      rec_facets<ET_HEX, 1, KH, 2, FACET_WARPS, DET>(P, F, rec, L, F.qp + (size_t)P.rec_bytes * (warp % FACET_WARPS));
    tile_epilogue<KH>(P, F);
    __syncthreads();
    tile = next;
  }
}

// ---- z-sweep kernel (sweep.cu schedules): 15 consumer warps take the element visits of the steps of
// this CTA's sequences, in order; warp 15 is the producer: it streams the step records (TMA bulk copy)
// and their halo points (LDGSTS) into a 3-deep ring, signalled by mbarriers (full: record + halo landed,
// empty: every consumer warp is done with the step).  Consumers never wait for each other except through
// the per-row turns of the ordered accumulation (and one named barrier between sequences, which resets
// the turn counters): rows are zeroed by their first contribution and written by their last toucher.
constexpr int SW_CONSUMERS = HEX_WARPS - 1;
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void cp_async_mbar_arrive_noinc(uint64_t* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}

template <int MODE, int SW_NBUF, int SWSR>
__global__ void __launch_bounds__(HEX_THREADS, 1) k_hex_sweep(const __grid_constant__ TiledParams P) {
  extern __shared__ __align__(16) unsigned char smem[];
  static_assert(3 * SW_NBUF * 8 <= 128, "barriers fit the 128-byte head");
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);   // [SW_NBUF]
  uint64_t* empty = full + SW_NBUF;                     // [SW_NBUF]
  uint64_t* landed = empty + SW_NBUF;                   // [SW_NBUF] record bulk copies
  __shared__ double lanetab[32 * LANE_TAB];
  __shared__ TileOffs tofs[SW_NBUF];  // per ring buffer: the step's section offsets (written by the producer)
  __shared__ uint32_t tvfm[SW_NBUF];
  __shared__ int tnv[SW_NBUF];
  auto rbuf = [&](int b) { return smem + 128 + (size_t)b * P.rec_cap; };
  auto hbuf = [&](int b) { return reinterpret_cast<double*>(smem + 128 + (size_t)SW_NBUF * P.rec_cap) + (size_t)b * P.hcap; };
  double* acc = hbuf(SW_NBUF);
  int* turn = reinterpret_cast<int*>(acc + P.acc_cap);
  double* scratch = reinterpret_cast<double*>(turn + P.turn_cap);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  HexCoef Hc = {0, 0, 0, 0, 0, 0};
  for (int f = 0; f < P.n_dom; f++) {
    const FormArgs& Fm = P.dom[f];
    Hc.cl += Fm.f0 * Fm.lam; Hc.cm += Fm.f0 * Fm.mu; Hc.sl += Fm.lam; Hc.sm += Fm.mu;
  }
  if (warp == 0) {  // per-lane constant table (same for every warp), transposed
    const GeoFrag GF = geo_frag();
    double* Lt = lanetab + tid;
#pragma unroll
    for (int s2 = 0; s2 < 2; s2++)
#pragma unroll
      for (int t = 0; t < 3; t++) Lt[32 * (s2 * 3 + t)] = GF.b[s2][t];
    double g0[3], g1[3], N0, N1;
    hex_ref(tid >> 2, tid & 3, g0, N0);
    hex_ref(tid >> 2, (tid & 3) + 4, g1, N1);
    for (int i = 0; i < 3; i++) { Lt[32 * (6 + i)] = g0[i]; Lt[32 * (9 + i)] = g1[i]; }
    double gc[3], gc4[3], Nc, Nc4;
    hex_ref(tid & 3, tid >> 2, gc, Nc);
    hex_ref((tid & 3) + 4, tid >> 2, gc4, Nc4);
    for (int i = 0; i < 3; i++) { Lt[32 * (12 + i)] = gc[i]; Lt[32 * (15 + i)] = gc4[i]; }
  }
  if (tid == 0) {
    for (int b = 0; b < SW_NBUF; b++) {
      mbar_init(&full[b], 33);             // the producer's 32 lanes (cp.async arrive.noinc) + its offsets
      mbar_init(&empty[b], SW_CONSUMERS);  // one arrive per consumer warp
      mbar_init(&landed[b], 1);
    }
    mbar_fence_init();
  }
  for (int i = tid; i < P.turn_cap; i += blockDim.x) turn[i] = 0;
  __syncthreads();
  int64_t q = blockIdx.x;
  if (q >= P.n_seq) return;
  int64_t t = P.seq_off[q];
  auto next_of = [&](int64_t tt, int64_t& qq) -> int64_t {
    if (tt + 1 < P.seq_off[qq + 1]) return tt + 1;
    qq += gridDim.x;
    return qq < P.n_seq ? P.seq_off[qq] : P.n_tiles;
  };
  if (warp == SW_CONSUMERS) {
    // ---------------- producer
    for (int64_t k = 0; t < P.n_tiles; k++) {
      const int b = (int)(k % SW_NBUF);
      const uint32_t use = (uint32_t)(k / SW_NBUF);
      if (k >= SW_NBUF) mbar_wait_sleep(&empty[b], (use - 1) & 1u);  // all consumers left step k - SW_NBUF
      if (lane == 0) {
        const uint32_t bytes = (uint32_t)(P.rec_off[t + 1] - P.rec_off[t]);
        mbar_expect_tx(&landed[b], bytes);
        bulk_g2s(rbuf(b), P.rec + P.rec_off[t], bytes, &landed[b]);
      }
      mbar_wait(&landed[b], use & 1u);
      const uint8_t* rec = rbuf(b);
      const int32_t* hdr = reinterpret_cast<const int32_t*>(rec);
      const int H = hdr[1];
      const RecLayout L = rec_layout_hdr(8, hdr);
      const int32_t* hn = reinterpret_cast<const int32_t*>(rec + L.o_hnode);
      double* hb = hbuf(b);
      for (int c = 0; c < P.hcomp; c++) {
        const double* base = c < 3 ? P.coords + (int64_t)c * P.N : P.state + (int64_t)(c - 3) * P.N;
        for (int i = lane; i < H; i += 32) cp_async8(hb + c * H + i, base + hn[i]);
      }
      if (lane == 0) {  // the step's offsets for the consumers (released by the arrive below)
        TileOffs o;
        const uint32_t rb = (uint32_t)(rec - smem);
        const int acc_n = P.values ? hdr[4] : 0;
        o.vown = rb + L.o_vown; o.vhal = rb + L.o_vhal; o.velem = rb + L.o_velem; o.vloc = rb + L.o_vloc;
        o.hdat = (uint32_t)(reinterpret_cast<const unsigned char*>(hb) - smem);
        o.tdeg = rb + L.o_tdeg; o.toff = rb + L.o_toff; o.tnode = rb + L.o_tnode; o.trps = rb + L.o_trps;
        o.acc = (uint32_t)(reinterpret_cast<unsigned char*>(acc) - smem);
        o.racc = o.acc + 8u * (uint32_t)acc_n;
        o.vseq = rb + L.o_vsw;
        o.turn = (uint32_t)(reinterpret_cast<unsigned char*>(turn) - smem);
        o.H = H;
        o.T = hdr[0];
        tofs[b] = o;
        tvfm[b] = rb + L.o_vfm;
        tnv[b] = hdr[2];
        mbar_arrive(&full[b]);
      }
      cp_async_mbar_arrive_noinc(&full[b]);
      t = next_of(t, q);
    }
    return;
  }
  // ---------------- consumers
  double* wsc = scratch + (size_t)HEX_SCRATCH * warp;
  int rot = 0;
  for (int64_t k = 0; t < P.n_tiles; k++) {
    const int b = (int)(k % SW_NBUF);
    mbar_wait_sleep(&full[b], (uint32_t)(k / SW_NBUF) & 1u);
    mbar_wait(&landed[b], (uint32_t)(k / SW_NBUF) & 1u);  // (already complete) the record's bulk copy is visible
    const TileOffs to = tofs[b];
    const int nv = tnv[b];
    const uint32_t* vfm = reinterpret_cast<const uint32_t*>(smem + tvfm[b]);
    // visits round-robin over the consumers, continuing the rotation of the previous step (49 visits on 15
    // warps would otherwise always give warps 0-3 the extra visit and let them fall steps behind)
    for (int v = (warp - rot + SW_CONSUMERS) % SW_CONSUMERS; v < nv; v += SW_CONSUMERS)
      hex_visit_el2<true, MODE, true, true, SWSR>(P, to, Hc, lanetab, wsc, v, smem, vfm);
    rot = (rot + nv) % SW_CONSUMERS;
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[b]);
    const int64_t qprev = q;
    t = next_of(t, q);
    if (q != qprev) {  // sequence boundary: every consumer is done with the old rows; restart the turns
      asm volatile("bar.sync 1, %0;" ::"r"(SW_CONSUMERS * 32) : "memory");
      for (int i = tid; i < P.turn_cap; i += SW_CONSUMERS * 32) turn[i] = 0;
      asm volatile("bar.sync 1, %0;" ::"r"(SW_CONSUMERS * 32) : "memory");
    }
  }
}

static int run_hex_sweep(TiledParams& P, const TileSchedule& T, cudaStream_t s) {
  P.fac_inline = 1;  // elasticity boundary terms (fix / load) inside the owning element's visit
  for (int f = 0; f < P.n_fac; f++) {
    const int fo = P.fac[f].form;
    if ((fo != FEM_WF_ELAST_FIX_ALL && fo != FEM_WF_ELAST_FIX_D1 && fo != FEM_WF_ELAST_LOAD) || P.fac_set[f] > 4)
      P.fac_inline = 0;
  }
  if (!P.fac_inline) {
    set_error("hex sweep kernel: boundary terms must be integrated inside the visits (elasticity fix/load forms "
              "on boundary sets 0..4)");
    return FEM_E_UNSUPPORTED;
  }
  P.seq_off = T.seq_off;
  P.n_seq = T.n_seq;
  if (T.sw_lperm) {  // renumbered mesh: the halo ids are lattice ranks; stage from lattice-ordered copies
    const int ncomp = 3 * (P.nu_hat >= 1 ? 2 : 1);
    if (ncomp > T.sw_pstate_comps) {
      set_error("hex sweep kernel: state components exceed the lattice-ordered copy");
      return FEM_E_UNSUPPORTED;
    }
    const int rc = perm_gather(P.state, T.sw_pstate, T.sw_lperm, P.N, ncomp, s);
    if (rc) return rc;
    P.coords = T.sw_pcoords;
    P.state = T.sw_pstate;
  }
  P.rec = T.rec;
  P.rec_off = T.rec_off;
  P.n_tiles = T.n_tiles;
  P.hcomp = 3 + 3 * (P.nu_hat >= 1 ? 2 : 1);
  P.rec_cap = (int)((T.rec_max + 15) / 16 * 16);
  P.hcap = (int)(((T.max_halo * P.hcomp) + 1) / 2 * 2);
  P.acc_cap = (int)((P.values ? T.acc_max : 0) + (int64_t)3 * T.max_tile_nodes);
  P.acc_cap = (P.acc_cap + 1) / 2 * 2;
  P.turn_cap = (int)((T.max_tile_nodes + 3) / 4 * 4);
  // a 3-step record/halo ring next to the accumulator ring
  const size_t fixed = 128 + 8 * (size_t)P.acc_cap + 4 * (size_t)P.turn_cap + 8 * (size_t)HEX_SCRATCH * SW_CONSUMERS;
  const size_t per_buf = (size_t)P.rec_cap + 8 * (size_t)P.hcap;
  const int nbuf = 3;
  const size_t smem = fixed + nbuf * per_buf;
  P.spin_ns = 32;  // back-off of a visit waiting for its row turn
  HexCoef Hc = {0, 0, 0, 0, 0, 0};
  for (int f = 0; f < P.n_dom; f++) {
    Hc.cl += P.dom[f].f0 * P.dom[f].lam; Hc.cm += P.dom[f].f0 * P.dom[f].mu;
    Hc.sl += P.dom[f].lam; Hc.sm += P.dom[f].mu;
  }
  const int hmode = !P.rhs ? HX_MAT : !P.values ? HX_RES : (Hc.cl == Hc.sl && Hc.cm == Hc.sm) ? HX_SYS_FUSED : HX_SYS;
  auto launch = [&](auto kern) -> int {
    cudaFuncAttributes fa;
    FEM_CUDA_TRY(cudaFuncGetAttributes(&fa, kern));
    if (smem + fa.sharedSizeBytes > 227 * 1024) {
      set_error("hex sweep kernel: shared memory request too large (" + std::to_string(smem) + " B dynamic)");
      return FEM_E_UNSUPPORTED;
    }
    FEM_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    if (T.n_tiles <= 0) return 0;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t grid = std::min<int64_t>(T.n_seq, sms);
    kern<<<(unsigned)grid, HEX_THREADS, smem, s>>>(P);
    FEM_CUDA_TRY(cudaGetLastError());
    return 0;
  };
  if (nbuf != 3) {
    set_error("hex sweep kernel: the record ring does not fit (3 steps)");
    return FEM_E_UNSUPPORTED;
  }
  auto by_mode = [&](auto srp) -> int {
    constexpr int SR = decltype(srp)::value;
    switch (hmode) {
      case HX_MAT: return launch(k_hex_sweep<HX_MAT, 3, SR>);
      case HX_RES: return launch(k_hex_sweep<HX_RES, 3, SR>);
      case HX_SYS_FUSED: return launch(k_hex_sweep<HX_SYS_FUSED, 3, SR>);
      default: return launch(k_hex_sweep<HX_SYS, 3, SR>);
    }
  };
  if (T.sweep_sr == 81) return by_mode(std::integral_constant<int, 81>());
  if (T.sweep_sr == 82) return by_mode(std::integral_constant<int, 82>());
  set_error("hex sweep kernel: unexpected ring row stride");
  return FEM_E_UNSUPPORTED;
}

template <int KH, bool DET>
static int run_hex_rec(TiledParams& P, const TileSchedule& T, cudaStream_t s) {
  using C = TileCfg<ET_HEX, 1, KH, 2>;
  P.rec_bytes = (int)((sizeof(typename C::QPG) * C::NQF + 15) / 16 * 16);
  int fv = 1;
  for (int f = 0; f < P.n_fac; f++) fv = std::max<int>(fv, (int)P.fvis[f].max_per_tile);
  P.fvmax = fv;
  P.vmax = fv;
  P.hmax = 0;
  P.hcomp = 3 + KH * (P.nu_hat >= 1 ? 2 : 1);
  P.rec = T.rec;
  P.rec_off = T.rec_off;
  P.n_tiles = T.n_tiles;
  P.rec_cap = (int)((T.rec_max + 15) / 16 * 16);
  P.hcap = (int)(((T.max_halo * P.hcomp) + 1) / 2 * 2);
  P.acc_cap = (int)((P.values ? T.acc_max : 0) + (int64_t)KH * T.max_tile_nodes);
  P.acc_cap = (P.acc_cap + 1) / 2 * 2;
  P.turn_cap = (int)((T.max_tile_nodes + 3) / 4 * 4);
  P.spin_ns = 0;
  // elasticity boundary terms (fix / load) inside the owning element's visit: no facet phase, no barriers
  P.fac_inline = KH == 3 && T.dom.max_per_tile <= HEX_MAX_VISITS;
  for (int f = 0; f < P.n_fac; f++) {
    const int fo = P.fac[f].form;
    if ((fo != FEM_WF_ELAST_FIX_ALL && fo != FEM_WF_ELAST_FIX_D1 && fo != FEM_WF_ELAST_LOAD) || P.fac_set[f] > 4)
      P.fac_inline = 0;
  }
  const size_t fac_bytes = std::max((size_t)P.rec_bytes * FACET_WARPS, (size_t)8 * HEX_SCRATCH * HEX_WARPS) + (size_t)fv * (4 + 8 * 4 + 8 * 2 + 1) + 16;
  const size_t smem = 128 + 2 * (size_t)P.rec_cap + 2 * 8 * (size_t)P.hcap + 8 * (size_t)P.acc_cap + 4 * (size_t)P.turn_cap + fac_bytes;
  cudaFuncAttributes fa;
  FEM_CUDA_TRY(cudaFuncGetAttributes(&fa, k_hex_rec<KH, DET>));
  if (smem + fa.sharedSizeBytes > 227 * 1024) {  // + static shared memory (tile offsets, lane table)
    set_error("hex record kernel: shared memory request too large (" + std::to_string(smem) + " B dynamic + " +
              std::to_string(fa.sharedSizeBytes) + " B static)");
    return FEM_E_UNSUPPORTED;
  }
  FEM_CUDA_TRY(cudaFuncSetAttribute(k_hex_rec<KH, DET>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  if (T.n_tiles <= 0) return 0;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t grid = std::min<int64_t>(T.n_tiles, sms);
  k_hex_rec<KH, DET><<<(unsigned)grid, HEX_THREADS, smem, s>>>(P);
  FEM_CUDA_TRY(cudaGetLastError());
  return 0;
}

// Q1 hex, 2x2x2 points, domain terms all ELAST_DOMAIN (κ̂ = 3) or all THERMAL_DOMAIN (κ̂ = 1).
int launch_hex_tiled(TiledParams& P, const TileSchedule& T, int kh, bool det, cudaStream_t s, bool* handled) {
  *handled = false;
  if (T.sweep) {  // sweep records are read only by the sweep kernel
    *handled = true;
    for (int f = 0; f < P.n_dom; f++)
      if (P.dom[f].form != FEM_WF_ELAST_DOMAIN) {
        set_error("tiled scatter: the sweep schedule of this mesh takes the elasticity domain form only");
        return FEM_E_UNSUPPORTED;
      }
    return run_hex_sweep(P, T, s);  // ordered: deterministic in both tiled modes
  }
  if (P.n_dom == 0) return 0;
  for (int f = 0; f < P.n_dom; f++) {
    if (kh == 3 && P.dom[f].form != FEM_WF_ELAST_DOMAIN) return 0;
    if (kh == 1 && P.dom[f].form != FEM_WF_THERMAL_DOMAIN) return 0;
  }
  if (kh != 1 && kh != 3) return 0;
  *handled = true;
  if (det && kh == 3 && T.max_turns > 255) {
    set_error("tiled scatter: a tile point is touched by more than 255 element visits (8-bit turns); use "
              "FEM_SCATTER_COLOURED or FEM_SCATTER_TILED_UNORDERED");
    return FEM_E_UNSUPPORTED;
  }
  if (det) return kh == 3 ? run_hex_rec<3, true>(P, T, s) : run_hex_rec<1, true>(P, T, s);
  return kh == 3 ? run_hex_rec<3, false>(P, T, s) : run_hex_rec<1, false>(P, T, s);
}


// ---- FEM_SCATTER_STORED element pass for Q1-hex elasticity (stored.cu): one warp per element, the visit
// arithmetic of hex_visit_el2 (geometry GEMM, per-point records with J^-1, w and w σ, the residual GEMM,
// the 18-DMMA Gram and K) with the element's points gathered straight from HBM; the upper blocks a <= b
// (36 of 64) and the 24 residual rows are staged in shared memory and stored as one coalesced stream at the
// element's Morton position: ek[pos][blk][i][m], er[pos][a][i].
constexpr int HXE_WARPS = 8;
template <bool HAS_V, bool HAS_R>
__global__ void __launch_bounds__(32 * HXE_WARPS) k_hex_el(const double* __restrict__ coords, const double* __restrict__ state,
                                                          const int32_t* __restrict__ conn, int64_t N, int64_t E,
                                                          const int32_t* __restrict__ eperm, HexCoef H,
                                                          double* __restrict__ ek, double* __restrict__ er, long long* err) {
  __shared__ double lanetab[32 * LANE_TAB];
  __shared__ __align__(16) double scr[HXE_WARPS][HEX_SCRATCH];
  __shared__ double stage[HXE_WARPS][36 * 9 + 24];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (warp == 0) {  // per-lane constant table, as in the sweep kernel
    const GeoFrag GF = geo_frag();
    double* Lt = lanetab + tid;
#pragma unroll
    for (int s2 = 0; s2 < 2; s2++)
#pragma unroll
      for (int t = 0; t < 3; t++) Lt[32 * (s2 * 3 + t)] = GF.b[s2][t];
    double g0[3], g1[3], N0, N1;
    hex_ref(tid >> 2, tid & 3, g0, N0);
    hex_ref(tid >> 2, (tid & 3) + 4, g1, N1);
    for (int i = 0; i < 3; i++) { Lt[32 * (6 + i)] = g0[i]; Lt[32 * (9 + i)] = g1[i]; }
    double gc[3], gc4[3], Nc, Nc4;
    hex_ref(tid & 3, tid >> 2, gc, Nc);
    hex_ref((tid & 3) + 4, tid >> 2, gc4, Nc4);
    for (int i = 0; i < 3; i++) { Lt[32 * (12 + i)] = gc[i]; Lt[32 * (15 + i)] = gc4[i]; }
  }
  __syncthreads();
  const int c = lane & 3, r = lane >> 2, q = r, a = r;
  const double* L = lanetab + lane;
  double* sc = scr[warp];
  double* stg = stage[warp];
  constexpr int RS = 22;
  const int64_t nw = (int64_t)gridDim.x * HXE_WARPS;
  for (int64_t pos = (int64_t)blockIdx.x * HXE_WARPS + warp; pos < E; pos += nw) {
    const int64_t e = __ldg(eperm + pos);
    const int nd = lane < 8 ? __ldg(conn + (int64_t)lane * E + e) : 0;
    double av[2];
#pragma unroll
    for (int s = 0; s < 2; s++) {
      const int node = __shfl_sync(0xffffffffu, nd, 4 * s + c);
      av[s] = r < 3 ? __ldg(coords + (int64_t)r * N + node)
                    : (HAS_R && r < 6) ? __ldg(state + (int64_t)(r - 3) * N + node) : 0.0;
    }
    double C3[3][2];
#pragma unroll
    for (int t = 0; t < 3; t++) { C3[t][0] = 0.0; C3[t][1] = 0.0; }
#pragma unroll
    for (int s = 0; s < 2; s++)
#pragma unroll
      for (int t = 0; t < 3; t++) dmma884(C3[t], av[s], L[32 * (s * 3 + t)]);
    if (r < 6) {
#pragma unroll
      for (int t = 0; t < 3; t++) {
        sc[hx_goff(r) + 8 * t + 2 * c] = C3[t][0];
        sc[hx_goff(r) + 8 * t + 2 * c + 1] = C3[t][1];
      }
    }
    __syncwarp();
    double J[3][3], Dr[3][3];
#pragma unroll
    for (int i = 0; i < 3; i++)
#pragma unroll
      for (int j = 0; j < 3; j++) {
        J[i][j] = sc[hx_goff(i) + 3 * q + j];
        Dr[i][j] = HAS_R ? sc[hx_goff(3 + i) + 3 * q + j] : 0.0;
      }
    const double c00 = J[1][1] * J[2][2] - J[1][2] * J[2][1];
    const double c01 = J[1][2] * J[2][0] - J[1][0] * J[2][2];
    const double c02 = J[1][0] * J[2][1] - J[1][1] * J[2][0];
    const double det = J[0][0] * c00 + J[0][1] * c01 + J[0][2] * c02;
    if (__any_sync(0xffffffffu, !(det > 0.0))) {
      if (lane == 0) atomicCAS((unsigned long long*)err, (unsigned long long)(-1LL), (unsigned long long)e);
      __syncwarp();
      continue;
    }
    __syncwarp();  // the GEMM output is consumed; the scratch takes the per-point records
    const double rr = 1.0 / det;
    double Ji[3][3];
    Ji[0][0] = c00 * rr; Ji[1][0] = c01 * rr; Ji[2][0] = c02 * rr;
    Ji[0][1] = (J[0][2] * J[2][1] - J[0][1] * J[2][2]) * rr;
    Ji[1][1] = (J[0][0] * J[2][2] - J[0][2] * J[2][0]) * rr;
    Ji[2][1] = (J[0][1] * J[2][0] - J[0][0] * J[2][1]) * rr;
    Ji[0][2] = (J[0][1] * J[1][2] - J[0][2] * J[1][1]) * rr;
    Ji[1][2] = (J[0][2] * J[1][0] - J[0][0] * J[1][2]) * rr;
    Ji[2][2] = (J[0][0] * J[1][1] - J[0][1] * J[1][0]) * rr;
    if (c == 0) {
      double* o = sc + q * RS;
#pragma unroll
      for (int j = 0; j < 3; j++)
#pragma unroll
        for (int i = 0; i < 3; i++) o[j * 3 + i] = Ji[j][i];
      o[9] = det;  // w (unit Gauss-Legendre weights)
      if constexpr (HAS_R) {  // w σ_ij at the point
        double gu[3][3];
#pragma unroll
        for (int k = 0; k < 3; k++)
#pragma unroll
          for (int i = 0; i < 3; i++) gu[k][i] = Dr[k][0] * Ji[0][i] + Dr[k][1] * Ji[1][i] + Dr[k][2] * Ji[2][i];
        const double lw = H.sl * det * (gu[0][0] + gu[1][1] + gu[2][2]), mw = H.sm * det;
#pragma unroll
        for (int i = 0; i < 3; i++)
#pragma unroll
          for (int j = 0; j < 3; j++) o[10 + i * 3 + j] = (i == j ? lw : 0.0) + mw * (gu[i][j] + gu[j][i]);
      }
    }
    __syncwarp();
    const double* o0 = sc + c * RS;
    const double* o1 = sc + (c + 4) * RS;
    double G0[3], G1[3];
#pragma unroll
    for (int i = 0; i < 3; i++) {
      G0[i] = o0[0 * 3 + i] * L[32 * 6] + o0[1 * 3 + i] * L[32 * 7] + o0[2 * 3 + i] * L[32 * 8];
      G1[i] = o1[0 * 3 + i] * L[32 * 9] + o1[1 * 3 + i] * L[32 * 10] + o1[2 * 3 + i] * L[32 * 11];
    }
    const double w0 = o0[9], w1 = o1[9];
    if constexpr (HAS_R) {  // r_(a,i) = -Σ_γ Σ_j G_aj [w σ_ij]: lane (a, c < 2) gets rows (a, 2c), (a, 2c + 1)
      double r2[2] = {0.0, 0.0};
#pragma unroll
      for (int j = 0; j < 3; j++) {
        dmma884(r2, G0[j], r < 3 ? o0[10 + r * 3 + j] : 0.0);
        dmma884(r2, G1[j], r < 3 ? o1[10 + r * 3 + j] : 0.0);
      }
      if (c == 0) { stg[324 + a * 3 + 0] = -r2[0]; stg[324 + a * 3 + 1] = -r2[1]; }
      if (c == 1) stg[324 + a * 3 + 2] = -r2[0];
    }
    if constexpr (HAS_V) {  // Gram (18 DMMA) and K for columns b = 2c + t; upper blocks b >= a staged
      double M[3][3][2];
#pragma unroll
      for (int j = 0; j < 3; j++)
#pragma unroll
        for (int k = 0; k < 3; k++) {
          M[j][k][0] = 0.0;
          M[j][k][1] = 0.0;
          dmma884(M[j][k], w0 * G0[j], G0[k]);
          dmma884(M[j][k], w1 * G1[j], G1[k]);
        }
#pragma unroll
      for (int t = 0; t < 2; t++) {
        const int b = 2 * c + t;
        if (b >= a) {
          const double tr = M[0][0][t] + M[1][1][t] + M[2][2][t];
          double* dst = stg + (a * 8 - a * (a - 1) / 2 + (b - a)) * 9;
#pragma unroll
          for (int i = 0; i < 3; i++)
#pragma unroll
            for (int m = 0; m < 3; m++) dst[i * 3 + m] = -(H.cl * M[i][m][t] + H.cm * M[m][i][t] + (i == m ? H.cm * tr : 0.0));
        }
      }
    }
    __syncwarp();
    if constexpr (HAS_V) {
      double* dst = ek + pos * 324;
      for (int k = lane; k < 324; k += 32) dst[k] = stg[k];
    }
    if constexpr (HAS_R) {
      if (lane < 24) er[pos * 24 + lane] = stg[324 + lane];
    }
    __syncwarp();  // scratch and stage are rewritten by the next element
  }
}

// Q1 hexes, 2x2x2 points, every domain term ELAST_DOMAIN: the stored-mode element pass (all domain terms).
int launch_hex_el(const fem_mesh_s* m, const fem_problem* prob, const double* state, const int32_t* eperm,
                  double* ek, double* er, cudaStream_t s, bool* handled) {
  *handled = false;
  if (m->etype != ET_HEX || m->order != 1 || m->kh != 3 || m->physics != FEM_ELASTICITY || prob->quad_order != 2)
    return 0;
  HexCoef H = {0, 0, 0, 0, 0, 0};
  int n_dom = 0;
  for (int t = 0; t < prob->n_terms; t++) {
    const fem_term& T = prob->terms[t];
    if (T.region >= 0) continue;
    if (T.form != FEM_WF_ELAST_DOMAIN) return 0;
    const FormArgs F = make_form_args(prob, T);
    H.cl += F.f0 * F.lam; H.cm += F.f0 * F.mu; H.sl += F.lam; H.sm += F.mu;
    n_dom++;
  }
  if (!n_dom) return 0;
  *handled = true;
  if (m->E == 0) return 0;
  int dev = 0, sms = 148, per_sm = 1;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  auto go = [&](auto kern) -> int {
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 32 * HXE_WARPS, 0);
    const int64_t grid = std::min<int64_t>((m->E + HXE_WARPS - 1) / HXE_WARPS, (int64_t)sms * std::max(per_sm, 1));
    kern<<<(unsigned)grid, 32 * HXE_WARPS, 0, s>>>(m->coords, state, m->conn, m->N, m->E, eperm, H, ek, er, m->err);
    FEM_CUDA_TRY(cudaGetLastError());
    return 0;
  };
  if (ek && er) return go(k_hex_el<true, true>);
  if (ek) return go(k_hex_el<true, false>);
  return go(k_hex_el<false, true>);
}

}  // namespace fem
