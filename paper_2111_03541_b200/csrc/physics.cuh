// physics.cuh — the fixed device integrands of the paper's three example physics.
//
// The paper's rule-based CAS (§3) differentiates each base term w.r.t. each operand ("complete
// gradient"); here the results are written out by hand (north_star: the CAS is not
// rebuilt).  res() = base term × dual word for test row (a, κ0) (D-2);
// tan() = Σ_λ (D0 N̄_a)(D_λ N_b) ∂L^a/∂λ for trial column (b, κλ) (D-3), times the time
// factor f_ν of the operand (Eq. gen_alpha).
//   Thermal     P:821-823 (code P:832-835)   κ̂ = 1
//   Elasticity  P:900-906 (code P:913-923)   κ̂ = dim, λ = Eν/((1+ν)(1-2ν)), μ = E/(2(1+ν))
//   NS + SUPG   P:979-992 (code P:998-1025)  κ̂ = dim+1 (u_1..u_dim, p); Rm carries −μ u_i,kk, which
//               vanishes on P1 (L10) and is carried by the QP's Laplacian tables on every other element
#pragma once
#include "../../include/libfem.h"

namespace fem {

// NS records on elements whose shape functions have non-zero second derivatives carry the physical
// Laplacian of every shape function L_a = Σ_k ∂²N_a/∂x_k² and of every operand, lu_κ = Σ_b L_b φ̃^κ_b
// (for μ u_i,kk in Rm_i).  P1 simplices (NL = DIM + 1) have none.
template <int DIM, int NL, int KH>
constexpr bool qp_has_lap() { return KH == DIM + 1 && NL > DIM + 1; }
template <int NL, int KH, bool LAP> struct QPLap {};
template <int NL, int KH> struct QPLap<NL, KH, true> {
  double L[NL];
  double lu[KH];
};

template <int DIM, int NL, int KH>
struct QP : QPLap<NL, KH, qp_has_lap<DIM, NL, KH>()> {
  double w;           // physical weight ŵ|det J| or ŵ·dA (reading L1)
  double x[DIM];      // physical point
  double n[DIM];      // outward unit normal (facets only)
  double N[NL];       // N_a(x)
  double G[NL][DIM];  // ∇N_a(x)
  double u[2][KH];    // effective values ∂_t^ν φ̃^κ, ν = 0, 1
  double gu[KH][DIM]; // ∇φ̃^κ
};

struct FormArgs {
  int form;
  int nu_hat;
  double f0, f1;   // time factors f_0 = c1 (static 1), f_1 = c2/(b1 Δt)
  double lam, mu;  // elasticity: λ = Eν/((1+ν)(1-2ν)), μ = E/(2(1+ν)), precomputed per call
  double p[FEM_MAX_PARAMS];
};

__device__ __forceinline__ double sq(double x) { return x * x; }

// ------------------------------------------------------------------ residual row (a, κ0)
template <int DIM, int NL, int KH>
__device__ __forceinline__ double form_res(const FormArgs& F, const QP<DIM, NL, KH>& q, int a, int k0) {
  const double* p = F.p;
  const double Na = q.N[a];
  switch (F.form) {
    case FEM_WF_THERMAL_DOMAIN: {
      double s = p[2];
      if (p[3] != 0.0) {
#pragma unroll
        for (int d = 0; d < DIM; d++) s *= sin(M_PI * q.x[d]);
      }
      double gg = 0.0;
#pragma unroll
      for (int d = 0; d < DIM; d++) gg += q.G[a][d] * q.gu[0][d];
      double r = Na * s - p[1] * gg;
      if (F.nu_hat >= 1) r -= p[0] * Na * q.u[1][0];
      return r;
    }
    case FEM_WF_THERMAL_CONV_RAD: {
      const double T = q.u[0][0], T2 = T * T, Te2 = p[1] * p[1];
      return Na * (p[0] * (p[1] - T) + p[2] * p[3] * (Te2 * Te2 - T2 * T2));
    }
    case FEM_WF_THERMAL_FIX: {
      double dn = 0.0;
#pragma unroll
      for (int d = 0; d < DIM; d++) dn += q.n[d] * q.gu[0][d];
      return Na * (p[0] * (p[1] - q.u[0][0]) + p[2] * dn);
    }
    case FEM_WF_ELAST_DOMAIN: {
      if (KH != DIM) return 0.0;
      const double lam = F.lam, mu = F.mu;
      double div = 0.0;
#pragma unroll
      for (int d = 0; d < DIM; d++) div += q.gu[d][d];
      double r = 0.0;  // -σ_ij G_aj with σ_ij = λ δ_ij div + μ(d_i,j + d_j,i)
#pragma unroll
      for (int j = 0; j < DIM; j++) {
        const double sij = (k0 == j ? lam * div : 0.0) + mu * (q.gu[k0 % KH][j] + q.gu[j % KH][k0]);
        r -= sij * q.G[a][j];
      }
      return r;
    }
    case FEM_WF_ELAST_FIX_ALL: return p[0] * Na * (p[1 + k0] - q.u[0][k0]);
    case FEM_WF_ELAST_FIX_D1: return k0 == 0 ? p[0] * Na * (p[1] - q.u[0][0]) : 0.0;
    case FEM_WF_ELAST_LOAD: {
      double t = 0.0;
#pragma unroll
      for (int j = 0; j < DIM; j++) t += p[3 * k0 + j] * q.n[j];
      return Na * t;
    }
    default: break;
  }
  if constexpr (KH == DIM + 1) {
    // ---- Navier-Stokes
    const double rho = p[0], mu = p[1];
    const double pr = q.u[0][DIM];
    const bool is_p = (k0 == DIM);
    const int i = is_p ? 0 : k0;
    double Ga_n = 0.0, un = 0.0;
#pragma unroll
    for (int d = 0; d < DIM; d++) { Ga_n += q.G[a][d] * q.n[d]; un += q.u[0][d] * q.n[d]; }
    if (F.form == FEM_WF_NS_DOMAIN) {
      const double tm = p[2], tc = p[3];
      double Rc = 0.0, Rm_i = q.gu[DIM][i], Aa = 0.0;
#pragma unroll
      for (int k = 0; k < DIM; k++) {
        Rc += q.gu[k][k];
        Rm_i += rho * q.u[0][k] * q.gu[i][k];
        Aa += q.G[a][k] * q.u[0][k];
      }
      if constexpr (qp_has_lap<DIM, NL, KH>()) Rm_i -= mu * q.lu[i];  // − μ u_i,kk
      if (!is_p) {
        double r = -q.G[a][i] * pr + tc * q.G[a][i] * Rc + tm * rho * Aa * Rm_i;
#pragma unroll
        for (int j = 0; j < DIM; j++) r += q.G[a][j] * (mu * q.gu[i][j] - rho * q.u[0][i] * q.u[0][j]);
        return r;
      }
      double r = Na * Rc;
#pragma unroll
      for (int ii = 0; ii < DIM; ii++) {
        double Rm = q.gu[DIM][ii];
#pragma unroll
        for (int k = 0; k < DIM; k++) Rm += rho * q.u[0][k] * q.gu[ii][k];
        if constexpr (qp_has_lap<DIM, NL, KH>()) Rm -= mu * q.lu[ii];
        r += tm * q.G[a][ii] * Rm;
      }
      return r;
    }
    // boundary groups = BASE + part
    double r = 0.0;
    if (!is_p) {
      double gn = 0.0;
#pragma unroll
      for (int j = 0; j < DIM; j++) gn += q.gu[i][j] * q.n[j];
      r = Na * (pr * q.n[i] - mu * gn);
    }
    if (F.form == FEM_WF_NS_BND_INFLOW) {
      const double U = p[3], H = p[4];
      const double y = q.x[1], z = q.x[DIM - 1];
      const double uw0 = 16.0 * U * (H - y) * (H - z) * y * z / (H * H * H * H);
      const double uwn = uw0 * q.n[0];
      if (!is_p) {
        const double uwi = (i == 0) ? uw0 : 0.0;
        r += rho * Na * uwi * uwn + mu * Ga_n * (uwi - q.u[0][i]) + p[2] * rho * Na * (q.u[0][i] - uwi);
      } else {
        r += Na * (uwn - un);
      }
    } else if (F.form == FEM_WF_NS_BND_OUTFLOW) {
      if (!is_p) r += rho * Na * q.u[0][i] * un;
    } else if (F.form == FEM_WF_NS_BND_FIX) {
      if (!is_p) r += (p[2] * rho * Na - mu * Ga_n) * q.u[0][i];
      else r -= Na * un;
    }
    return r;
  }
  return 0.0;
}

// ------------------------------------------------------------------ tangent entry (a,κ0)x(b,κλ)
template <int DIM, int NL, int KH>
__device__ __forceinline__ double form_tan(const FormArgs& F, const QP<DIM, NL, KH>& q, int a, int k0, int b,
                                           int kl) {
  const double* p = F.p;
  const double Na = q.N[a], Nb = q.N[b];
  double GaGb = 0.0;
#pragma unroll
  for (int d = 0; d < DIM; d++) GaGb += q.G[a][d] * q.G[b][d];
  switch (F.form) {
    case FEM_WF_THERMAL_DOMAIN: {
      double v = -p[1] * GaGb * F.f0;
      if (F.nu_hat >= 1) v -= p[0] * Na * Nb * F.f1;
      return v;
    }
    case FEM_WF_THERMAL_CONV_RAD: {
      const double T = q.u[0][0];
      return -Na * Nb * (p[0] + 4.0 * p[2] * p[3] * T * T * T) * F.f0;
    }
    case FEM_WF_THERMAL_FIX: {
      double Gbn = 0.0;
#pragma unroll
      for (int d = 0; d < DIM; d++) Gbn += q.G[b][d] * q.n[d];
      return Na * (p[2] * Gbn - p[0] * Nb) * F.f0;
    }
    case FEM_WF_ELAST_DOMAIN: {
      const double lam = F.lam, mu = F.mu;
      const int i = k0 % DIM, m = kl % DIM;
      double v = lam * q.G[a][i] * q.G[b][m] + mu * q.G[a][m] * q.G[b][i];
      if (i == m) v += mu * GaGb;
      return -v * F.f0;
    }
    case FEM_WF_ELAST_FIX_ALL: return (k0 == kl) ? -p[0] * Na * Nb * F.f0 : 0.0;
    case FEM_WF_ELAST_FIX_D1: return (k0 == 0 && kl == 0) ? -p[0] * Na * Nb * F.f0 : 0.0;
    case FEM_WF_ELAST_LOAD: return 0.0;
    default: break;
  }
  if constexpr (KH == DIM + 1) {
    const double rho = p[0], mu = p[1];
    const bool row_p = (k0 == DIM), col_p = (kl == DIM);
    const int i = row_p ? 0 : k0, m = col_p ? 0 : kl;
    if (F.form == FEM_WF_NS_DOMAIN) {
      const double tm = p[2], tc = p[3];
      double Aa = 0.0, Bb = 0.0;
#pragma unroll
      for (int k = 0; k < DIM; k++) { Aa += q.G[a][k] * q.u[0][k]; Bb += q.u[0][k] * q.G[b][k]; }
      double v;
      if (!row_p && !col_p) {
        double Rm_i = q.gu[DIM][i];
#pragma unroll
        for (int k = 0; k < DIM; k++) Rm_i += rho * q.u[0][k] * q.gu[i][k];
        const double dim_ = (i == m) ? 1.0 : 0.0;
        double dlap = 0.0;  // ∂(−μ u_i,kk)/∂φ_(b,m) = −μ δ_im L_b
        if constexpr (qp_has_lap<DIM, NL, KH>()) {
          Rm_i -= mu * q.lu[i];
          dlap = -mu * dim_ * q.L[b];
        }
        v = -rho * Nb * (dim_ * Aa + q.u[0][i] * q.G[a][m]) + mu * dim_ * GaGb +
            tm * rho * Nb * q.G[a][m] * Rm_i + tm * rho * Aa * (rho * (Nb * q.gu[i][m] + dim_ * Bb) + dlap) +
            tc * q.G[a][i] * q.G[b][m];
      } else if (!row_p && col_p) {
        v = -q.G[a][i] * Nb + tm * rho * Aa * q.G[b][i];
      } else if (row_p && !col_p) {
        double s = 0.0;
#pragma unroll
        for (int ii = 0; ii < DIM; ii++) s += q.G[a][ii] * q.gu[ii][m];
        v = Na * q.G[b][m] + tm * rho * (Nb * s + q.G[a][m] * Bb);
        if constexpr (qp_has_lap<DIM, NL, KH>()) v -= tm * mu * q.G[a][m] * q.L[b];
      } else {
        v = tm * GaGb;
      }
      return v * F.f0;
    }
    double Ga_n = 0.0, Gb_n = 0.0, un = 0.0;
#pragma unroll
    for (int d = 0; d < DIM; d++) {
      Ga_n += q.G[a][d] * q.n[d];
      Gb_n += q.G[b][d] * q.n[d];
      un += q.u[0][d] * q.n[d];
    }
    double v = 0.0;
    if (!row_p) {  // BASE
      if (!col_p && i == m) v -= mu * Na * Gb_n;
      if (col_p) v += Na * Nb * q.n[i];
    }
    if (F.form == FEM_WF_NS_BND_INFLOW || F.form == FEM_WF_NS_BND_FIX) {
      if (!row_p && !col_p && i == m) v += -mu * Ga_n * Nb + p[2] * rho * Na * Nb;
      if (row_p && !col_p) v -= Na * Nb * q.n[m];
    } else if (F.form == FEM_WF_NS_BND_OUTFLOW) {
      if (!row_p && !col_p) v += rho * Na * Nb * ((i == m ? un : 0.0) + q.u[0][i] * q.n[m]);
    }
    return v * F.f0;
  }
  return 0.0;
}

}  // namespace fem
