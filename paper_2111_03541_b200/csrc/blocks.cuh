// blocks.cuh — per-pair local blocks for the tiled (owner-gather) kernel.
//
// pair_block() returns, for test node a and trial node b of one element, the κ̂×κ̂ block
//   K_e[(a,κ0),(b,κλ)] = Σ_γ w_γ f_ν (D0 N̄_a D_λ N_b) ∂L^a/∂λ        (D-3)
// summed over the element's quadrature points; row_res() the residual row r_e[(a,κ0)] (D-2).
// The heavy domain forms have hand-hoisted formulations (elasticity through the Gram tensor
// M_ab^{jk} = Σ_γ w G_aj G_bk, so K_ab^{im} = -f0 (λ M^{im} + μ M^{mi} + μ δ_im tr M); NS with the
// per-point strong residuals Rm_i, Rc precomputed); boundary forms use the entry-wise integrands of
// physics.cuh.  All formulas: physics.cuh header.
#pragma once
#include "physics.cuh"

namespace fem {

template <int DIM, int NL, int KH>
struct QPX : QP<DIM, NL, KH> {
  // per-point precomputations of the batch's first domain form:
  //   ELAST_DOMAIN: ext[i*DIM+j] = w σ_ij (σ_ij = λ δ_ij d_k,k + μ (d_i,j + d_j,i))
  //   NS_DOMAIN:    ext[i] = Rm_i = ρ u_k u_i,k + p_,i (u_i,kk = 0 on P1, L10), ext[DIM] = Rc = u_k,k
  double ext[DIM * DIM + 1];
};

template <int DIM, int NL, int KH, int NQ>
__device__ __forceinline__ void pair_block(const FormArgs& F, const QPX<DIM, NL, KH>* __restrict__ qe, int a, int b,
                                           double (&K)[KH][KH]) {
  const double* p = F.p;
  if (F.form == FEM_WF_ELAST_DOMAIN && KH == DIM) {
    double M[DIM][DIM];
#pragma unroll
    for (int j = 0; j < DIM; j++)
#pragma unroll
      for (int k = 0; k < DIM; k++) M[j][k] = 0.0;
#pragma unroll
    for (int g = 0; g < NQ; g++) {
      const QPX<DIM, NL, KH>& q = qe[g];
      double wa[DIM], gb[DIM];
#pragma unroll
      for (int j = 0; j < DIM; j++) { wa[j] = q.w * q.G[a][j]; gb[j] = q.G[b][j]; }
#pragma unroll
      for (int j = 0; j < DIM; j++)
#pragma unroll
        for (int k = 0; k < DIM; k++) M[j][k] = fma(wa[j], gb[k], M[j][k]);
    }
    const double lam = F.lam, mu = F.mu;
    double tr = 0.0;
#pragma unroll
    for (int j = 0; j < DIM; j++) tr += M[j][j];
#pragma unroll
    for (int i = 0; i < DIM; i++)
#pragma unroll
      for (int m = 0; m < DIM; m++)
        K[i % KH][m % KH] -= F.f0 * (lam * M[i][m] + mu * M[m][i] + (i == m ? mu * tr : 0.0));
    return;
  }
  if (F.form == FEM_WF_THERMAL_DOMAIN) {
    double s = 0.0, mm = 0.0;
#pragma unroll
    for (int g = 0; g < NQ; g++) {
      const QPX<DIM, NL, KH>& q = qe[g];
      double d = 0.0;
#pragma unroll
      for (int j = 0; j < DIM; j++) d = fma(q.G[a][j], q.G[b][j], d);
      s = fma(q.w, d, s);
      mm = fma(q.w * q.N[a], q.N[b], mm);
    }
    double v = -p[1] * F.f0 * s;
    if (F.nu_hat >= 1) v -= p[0] * F.f1 * mm;
    K[0][0] += v;
    return;
  }
  if constexpr (KH == DIM + 1) {
    if (F.form == FEM_WF_NS_DOMAIN) {
      const double rho = p[0], mu = p[1], tm = p[2], tc = p[3];
      double acc[KH][KH];
#pragma unroll
      for (int i = 0; i < KH; i++)
#pragma unroll
        for (int m = 0; m < KH; m++) acc[i][m] = 0.0;
#pragma unroll
      for (int g = 0; g < NQ; g++) {
        const QPX<DIM, NL, KH>& q = qe[g];
        const double w = q.w, Na = q.N[a], Nb = q.N[b];
        double Aa = 0.0, Bb = 0.0, GaGb = 0.0, s[DIM];
#pragma unroll
        for (int k = 0; k < DIM; k++) {
          Aa = fma(q.G[a][k], q.u[0][k], Aa);
          Bb = fma(q.u[0][k], q.G[b][k], Bb);
          GaGb = fma(q.G[a][k], q.G[b][k], GaGb);
        }
#pragma unroll
        for (int m = 0; m < DIM; m++) {
          double t = 0.0;
#pragma unroll
          for (int i = 0; i < DIM; i++) t = fma(q.G[a][i], q.gu[i][m], t);
          s[m] = t;
        }
        const double wNb = w * Nb;
        const double diag = w * (-rho * Nb * Aa + mu * GaGb + tm * rho * rho * Aa * Bb);
        const double c_uu = w * tm * rho * rho * Aa * Nb;  // × u_i,m
        const double c_rm = tm * rho * wNb;                 // × G_am Rm_i
#pragma unroll
        for (int i = 0; i < DIM; i++) {
#pragma unroll
          for (int m = 0; m < DIM; m++) {
            double v = -rho * wNb * q.u[0][i] * q.G[a][m] + c_rm * q.G[a][m] * q.ext[i] + c_uu * q.gu[i][m] +
                       tc * w * q.G[a][i] * q.G[b][m];
            if (i == m) v += diag;
            acc[i][m] += v;
          }
          acc[i][DIM] += w * (-q.G[a][i] * Nb + tm * rho * Aa * q.G[b][i]);
          acc[DIM][i] += w * (Na * q.G[b][i] + tm * rho * (Nb * s[i] + q.G[a][i] * Bb));
        }
        acc[DIM][DIM] += w * tm * GaGb;
      }
#pragma unroll
      for (int i = 0; i < KH; i++)
#pragma unroll
        for (int m = 0; m < KH; m++) K[i][m] += F.f0 * acc[i][m];
      return;
    }
  }
  // entry-wise fallback (boundary forms, rare domain forms)
#pragma unroll
  for (int g = 0; g < NQ; g++) {
    const QP<DIM, NL, KH>& q = qe[g];
#pragma unroll
    for (int i = 0; i < KH; i++)
#pragma unroll
      for (int m = 0; m < KH; m++) K[i][m] += q.w * form_tan<DIM, NL, KH>(F, q, a, i, b, m);
  }
}

template <int DIM, int NL, int KH, int NQ>
__device__ __forceinline__ void row_res(const FormArgs& F, const QPX<DIM, NL, KH>* __restrict__ qe, int a,
                                        double (&r)[KH], bool ext_valid) {
  if (ext_valid && F.form == FEM_WF_ELAST_DOMAIN && KH == DIM) {  // r_(a,i) = -Σ_γ w σ_ij G_aj
#pragma unroll
    for (int g = 0; g < NQ; g++) {
      const QPX<DIM, NL, KH>& q = qe[g];
#pragma unroll
      for (int i = 0; i < DIM; i++) {
        double t = 0.0;
#pragma unroll
        for (int j = 0; j < DIM; j++) t = fma(q.ext[i * DIM + j], q.G[a][j], t);
        r[i % KH] -= t;
      }
    }
    return;
  }
#pragma unroll
  for (int g = 0; g < NQ; g++) {
    const QP<DIM, NL, KH>& q = qe[g];
#pragma unroll
    for (int i = 0; i < KH; i++) r[i] += q.w * form_res<DIM, NL, KH>(F, q, a, i);
  }
}

}  // namespace fem
