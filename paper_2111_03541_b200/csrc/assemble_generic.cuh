// assemble_generic.cu — element-batch assembly kernel (atomic and coloured scatter modes).
//
// One CTA processes a batch of BE elements (or boundary facets) at a time:
//   stage 0  coalesced SoA read of conn[a][e] -> smem node ids                       (A4)
//   stage 1  one thread per (element, quadrature point): J, det J, J^{-1}, ∇N_a, w,
//            field values/gradients -> smem QP records                               (A5, A6)
//   stage 2  one thread per (element, test node a, component κ0): residual row and
//            tangent row over (b, κλ), summed over the quadrature points, scattered
//            through the slot map with RED.F64 (atomic) or plain RMW (coloured)      (A7, A9)
// D-2 / D-3 of PAPER.md; the element loop order is free ("(atomic) increment").
#pragma once
#include <cmath>

#include "elements.cuh"
#include "fem_internal.cuh"
#include "stored.cuh"

namespace fem {

template <int ET, int ORD, int KH, int Q, bool FACET>
struct GenCfg {
  using EL = Elem<ET, ORD>;
  static constexpr int DIM = EL::DIM, NL = EL::NL;
  static constexpr int NQ = FACET ? EL::fac_nq(Q) : EL::vol_nq(Q);
  using QPt = QP<DIM, NL, KH>;
  static constexpr int BUDGET = 40 * 1024;
  static constexpr int BE0 = BUDGET / (NQ * (int)sizeof(QPt) + NL * 4 + 4);
  static constexpr int BE = BE0 < 1 ? 1 : (BE0 > 32 ? 32 : BE0);
  static constexpr size_t SMEM = (size_t)BE * NQ * sizeof(QPt) + (size_t)BE * NL * 4 + BE * 4 + 16;
};

__device__ __forceinline__ void report_bad(long long* err, long long e) {
  atomicCAS((unsigned long long*)err, (unsigned long long)(-1LL), (unsigned long long)e);
}

template <int DIM>
__device__ __forceinline__ double inv_jac(const double (*J)[DIM], double (*Ji)[DIM]) {
  if constexpr (DIM == 2) {
    const double det = J[0][0] * J[1][1] - J[0][1] * J[1][0];
    const double r = 1.0 / det;
    Ji[0][0] = J[1][1] * r;  Ji[0][1] = -J[0][1] * r;
    Ji[1][0] = -J[1][0] * r; Ji[1][1] = J[0][0] * r;
    return det;
  } else {
    const double c00 = J[1][1] * J[2][2] - J[1][2] * J[2][1];
    const double c01 = J[1][2] * J[2][0] - J[1][0] * J[2][2];
    const double c02 = J[1][0] * J[2][1] - J[1][1] * J[2][0];
    const double det = J[0][0] * c00 + J[0][1] * c01 + J[0][2] * c02;
    const double r = 1.0 / det;
    Ji[0][0] = c00 * r;
    Ji[1][0] = c01 * r;
    Ji[2][0] = c02 * r;
    Ji[0][1] = (J[0][2] * J[2][1] - J[0][1] * J[2][2]) * r;
    Ji[1][1] = (J[0][0] * J[2][2] - J[0][2] * J[2][0]) * r;
    Ji[2][1] = (J[0][1] * J[2][0] - J[0][0] * J[2][1]) * r;
    Ji[0][2] = (J[0][1] * J[1][2] - J[0][2] * J[1][1]) * r;
    Ji[1][2] = (J[0][2] * J[1][0] - J[0][0] * J[1][2]) * r;
    Ji[2][2] = (J[0][0] * J[1][1] - J[0][1] * J[1][0]) * r;
    return det;
  }
}

struct GenParams {
  FormArgs F;
  int64_t N, E, own_lo, own_hi, n_own, nnz_s;
  const double* coords;
  const int32_t* conn;
  const double* state;
  int nu_hat;
  const int32_t* task_elem;
  const int8_t* task_facet;
  int64_t task_begin, task_count;
  double* values;
  double* rhs;
  const int32_t* slot;
  const int64_t* rowptr_s;
  int plain;
  long long* err;
  double* ek = nullptr;  // FEM_SCATTER_STORED: element blocks [E][ek_nb][st_bs(KH)] (values unused)
  int ek_nb = 0;
  double* er = nullptr;  // FEM_SCATTER_STORED: element residuals [E][NL][KH] (rhs unused)
  int ek_add = 0;        // 0: store (first domain term), 1: add
  const int32_t* ek_map = nullptr;  // storage index of element e (null: e); < 0: not stored
};

template <int ET, int ORD, int KH, int Q, bool FACET>
__global__ void __launch_bounds__(128) k_generic(const GenParams P) {
  using C = GenCfg<ET, ORD, KH, Q, FACET>;
  using EL = typename C::EL;
  constexpr int DIM = C::DIM, NL = C::NL, NQ = C::NQ, BE = C::BE;
  using QPt = typename C::QPt;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  QPt* qs = reinterpret_cast<QPt*>(smem_raw);
  int* nodes = reinterpret_cast<int*>(qs + BE * NQ);
  int* bad = nodes + BE * NL;

  for (int64_t base = (int64_t)blockIdx.x * BE; base < P.task_count; base += (int64_t)gridDim.x * BE) {
    // ---- stage 0: node ids of the batch
    for (int t = threadIdx.x; t < BE * NL; t += blockDim.x) {
      const int be = t / NL, a = t % NL;
      const int64_t task = base + be;
      int node = -1;
      if (task < P.task_count) {
        const int64_t ti = P.task_begin + task;
        const int64_t e = P.task_elem ? P.task_elem[ti] : ti;
        node = P.conn[(int64_t)a * P.E + e];
      }
      nodes[t] = node;
    }
    for (int t = threadIdx.x; t < BE; t += blockDim.x) bad[t] = 0;
    __syncthreads();
    // ---- stage 1: geometry + fields per quadrature point
    for (int t = threadIdx.x; t < BE * NQ; t += blockDim.x) {
      const int be = t / NQ, g = t % NQ;
      const int64_t task = base + be;
      if (task >= P.task_count) continue;
      const int64_t ti = P.task_begin + task;
      const int* nd = nodes + be * NL;
      double xi[3] = {0, 0, 0}, wref, mref[3] = {0, 0, 0};
      if constexpr (FACET) EL::fac_qp(Q, P.task_facet[ti], g, xi, wref, mref);
      else EL::vol_qp(Q, g, xi, wref);
      double N[NL], dN[NL][DIM];
      EL::shape(xi, N, dN);
      double X[NL][DIM];
#pragma unroll
      for (int a = 0; a < NL; a++)
#pragma unroll
        for (int d = 0; d < DIM; d++) X[a][d] = P.coords[(int64_t)d * P.N + nd[a]];
      double J[DIM][DIM], Ji[DIM][DIM];
#pragma unroll
      for (int i = 0; i < DIM; i++)
#pragma unroll
        for (int j = 0; j < DIM; j++) {
          double s = 0.0;
#pragma unroll
          for (int a = 0; a < NL; a++) s += X[a][i] * dN[a][j];
          J[i][j] = s;
        }
      const double det = inv_jac<DIM>(J, Ji);
      QPt& q = qs[be * NQ + g];
      if (!(det > 0.0)) {
        bad[be] = 1;
        const int64_t e = P.task_elem ? P.task_elem[ti] : ti;
        report_bad(P.err, e);
        continue;
      }
#pragma unroll
      for (int a = 0; a < NL; a++) {
        q.N[a] = N[a];
#pragma unroll
        for (int i = 0; i < DIM; i++) {
          double s = 0.0;
#pragma unroll
          for (int j = 0; j < DIM; j++) s += Ji[j][i] * dN[a][j];
          q.G[a][i] = s;
        }
      }
#pragma unroll
      for (int d = 0; d < DIM; d++) {
        double s = 0.0;
#pragma unroll
        for (int a = 0; a < NL; a++) s += N[a] * X[a][d];
        q.x[d] = s;
        q.n[d] = 0.0;
      }
      if constexpr (FACET) {
        // Nanson: n dA = det(J) J^{-T} m̂ dÂ
        double nv[DIM], nn = 0.0;
#pragma unroll
        for (int i = 0; i < DIM; i++) {
          double s = 0.0;
#pragma unroll
          for (int j = 0; j < DIM; j++) s += Ji[j][i] * mref[j];
          nv[i] = det * s;
          nn += nv[i] * nv[i];
        }
        const double dA = sqrt(nn);
#pragma unroll
        for (int i = 0; i < DIM; i++) q.n[i] = nv[i] / dA;
        q.w = wref * dA;
      } else {
        q.w = wref * det;
      }
      if constexpr (qp_has_lap<DIM, NL, KH>() && !FACET) {  // (boundary forms do not use Rm)
        // L_a = tr H_a with H = J^{-T} (∂²N/∂ξ² − Σ_i G_i ∂²x_i/∂ξ²) J^{-1} (chain rule twice); first the
        // geometry's second derivatives Xh_i = Σ_a x_ai ∂²N_a/∂ξ², then per node (Hessians recomputed)
        double Xh[DIM][DIM][DIM];
#pragma unroll
        for (int i = 0; i < DIM; i++)
#pragma unroll
          for (int j = 0; j < DIM; j++)
#pragma unroll
            for (int l = 0; l < DIM; l++) Xh[i][j][l] = 0.0;
        for (int a = 0; a < NL; a++) {
          double h[3][3];
          EL::node_hess(a, xi, h);
#pragma unroll
          for (int i = 0; i < DIM; i++)
#pragma unroll
            for (int j = 0; j < DIM; j++)
#pragma unroll
              for (int l = 0; l < DIM; l++) Xh[i][j][l] += X[a][i] * h[j][l];
        }
        double JJ[DIM][DIM];  // J^{-1} J^{-T}: tr(J^{-T} A J^{-1}) = Σ_jl A_jl (J^{-1} J^{-T})_lj
#pragma unroll
        for (int l = 0; l < DIM; l++)
#pragma unroll
          for (int j = 0; j < DIM; j++) {
            double t = 0.0;
#pragma unroll
            for (int i = 0; i < DIM; i++) t += Ji[l][i] * Ji[j][i];
            JJ[l][j] = t;
          }
        for (int a = 0; a < NL; a++) {
          double h[3][3];
          EL::node_hess(a, xi, h);
          double L = 0.0;
#pragma unroll
          for (int j = 0; j < DIM; j++)
#pragma unroll
            for (int l = 0; l < DIM; l++) {
              double A = h[j][l];
#pragma unroll
              for (int i = 0; i < DIM; i++) A -= q.G[a][i] * Xh[i][j][l];
              L += A * JJ[l][j];
            }
          q.L[a] = L;
        }
#pragma unroll
        for (int k = 0; k < KH; k++) {
          double t = 0.0;
          for (int a = 0; a < NL; a++) t += q.L[a] * P.state[(int64_t)k * P.N + nd[a]];
          q.lu[k] = t;
        }
      }
      // fields
#pragma unroll
      for (int k = 0; k < KH; k++) {
        double v0 = 0.0, v1 = 0.0, gk[DIM];
#pragma unroll
        for (int d = 0; d < DIM; d++) gk[d] = 0.0;
#pragma unroll
        for (int a = 0; a < NL; a++) {
          const double s0 = P.state[(int64_t)k * P.N + nd[a]];
          v0 += N[a] * s0;
          if (P.nu_hat >= 1) v1 += N[a] * P.state[((int64_t)KH + k) * P.N + nd[a]];
#pragma unroll
          for (int d = 0; d < DIM; d++) gk[d] += q.G[a][d] * s0;
        }
        q.u[0][k] = v0;
        q.u[1][k] = v1;
#pragma unroll
        for (int d = 0; d < DIM; d++) q.gu[k][d] = gk[d];
      }
    }
    __syncthreads();
    // ---- stage 2: rows (element, a, κ0)
    for (int t = threadIdx.x; t < BE * NL * KH; t += blockDim.x) {
      const int be = t / (NL * KH), rem = t % (NL * KH), a = rem / KH, k0 = rem % KH;
      const int64_t task = base + be;
      if (task >= P.task_count || bad[be]) continue;
      const int node = nodes[be * NL + a];
      // stored mode: every row of the element (a symmetric block (a, b), a <= b, serves the owned row b even
      // when row a belongs to another part)
      const bool owned = node >= P.own_lo && node < P.own_hi;
      if (!owned && !P.ek && !P.er) continue;
      const int64_t li = node - P.own_lo;
      const QPt* qe = qs + be * NQ;
      const int64_t ti = P.task_begin + task;
      const int64_t e = P.task_elem ? P.task_elem[ti] : ti;
      const int64_t es = P.ek_map ? (int64_t)P.ek_map[e] : e;  // element storage index (stored mode)
      if (P.er) {  // FEM_SCATTER_STORED: the element's own residual rows (stored, or added by later terms)
        double r = 0.0;
#pragma unroll
        for (int g = 0; g < NQ; g++) r += qe[g].w * form_res<DIM, NL, KH>(P.F, qe[g], a, k0);
        double* dst = P.er + (es * NL + a) * KH + k0;
        *dst = (P.ek_add ? *dst : 0.0) + r;
      } else if (P.rhs && owned) {
        double r = 0.0;
#pragma unroll
        for (int g = 0; g < NQ; g++) r += qe[g].w * form_res<DIM, NL, KH>(P.F, qe[g], a, k0);
        double* dst = P.rhs + (int64_t)k0 * P.n_own + li;
        if (P.plain) *dst += r;
        else atomicAdd(dst, r);
      }
      if (P.ek && P.F.form != FEM_WF_ELAST_LOAD) {  // FEM_SCATTER_STORED: block (a, b) of the element
        // symmetric physics (ek_nb = NL(NL+1)/2): the blocks b >= a only, packed row by row
        const bool sym = P.ek_nb != NL * NL;
        const int64_t eb = es * P.ek_nb;
        for (int b = sym ? a : 0; b < NL; b++) {
          const int blk = sym ? a * NL - a * (a - 1) / 2 + (b - a) : a * NL + b;
          double* dst = P.ek + (eb + blk) * st_bs(KH) + k0 * KH;
#pragma unroll
          for (int kl = 0; kl < KH; kl++) {
            double v = 0.0;
#pragma unroll
            for (int g = 0; g < NQ; g++) v += qe[g].w * form_tan<DIM, NL, KH>(P.F, qe[g], a, k0, b, kl);
            dst[kl] = (P.ek_add ? dst[kl] : 0.0) + v;
          }
        }
      } else if (P.values && P.F.form != FEM_WF_ELAST_LOAD && owned) {
        const int64_t rps = P.rowptr_s[li];
        const int64_t deg = P.rowptr_s[li + 1] - rps;
        const int64_t rowbase = (int64_t)k0 * KH * P.nnz_s + (int64_t)KH * rps;
        for (int b = 0; b < NL; b++) {
          const int64_t off = (int64_t)P.slot[((int64_t)a * NL + b) * P.E + e] - rps;
#pragma unroll
          for (int kl = 0; kl < KH; kl++) {
            double v = 0.0;
#pragma unroll
            for (int g = 0; g < NQ; g++) v += qe[g].w * form_tan<DIM, NL, KH>(P.F, qe[g], a, k0, b, kl);
            double* dst = P.values + rowbase + (int64_t)kl * deg + off;
            if (P.plain) *dst += v;
            else atomicAdd(dst, v);
          }
        }
      }
    }
    __syncthreads();
  }
}

template <int ET, int ORD, int KH, int Q, bool FACET>
inline int run(const GenParams& P, cudaStream_t s) {
  using C = GenCfg<ET, ORD, KH, Q, FACET>;
  auto kern = k_generic<ET, ORD, KH, Q, FACET>;
  static bool attr_set = false;
  if (!attr_set) {
    FEM_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM));
    attr_set = true;
  }
  if (P.task_count <= 0) return 0;
  int64_t blocks = (P.task_count + C::BE - 1) / C::BE;
  const int64_t cap = 148 * 16;
  if (blocks > cap) blocks = cap;
  kern<<<(unsigned)blocks, 128, C::SMEM, s>>>(P);
  FEM_CUDA_TRY(cudaGetLastError());
  return 0;
}

template <int ET, int ORD, int KH, bool FACET>
inline int run_q(int q, const GenParams& P, cudaStream_t s) {
  if constexpr ((ET == ET_HEX || ET == ET_HEXS) && ORD == 2) {  // quadratic cubes: 2 or 3 points per axis
    if (q == 2) return run<ET, ORD, KH, 2, FACET>(P, s);
    if (q == 3) return run<ET, ORD, KH, 3, FACET>(P, s);
  } else if constexpr (ET == ET_HEX) {
    if (q == 1) return run<ET, ORD, KH, 1, FACET>(P, s);
    if (q == 2) return run<ET, ORD, KH, 2, FACET>(P, s);
    if (q == 3) return run<ET, ORD, KH, 3, FACET>(P, s);
  } else {
    if (q == 1) return run<ET, ORD, KH, 1, FACET>(P, s);
    if (q == 2) return run<ET, ORD, KH, 2, FACET>(P, s);
  }
  set_error("unsupported quadrature order");
  return FEM_E_UNSUPPORTED;
}

int gen_dispatch_tri(int kh, int q, const GenParams& P, cudaStream_t s, bool facet);
int gen_dispatch_hex(int kh, int q, const GenParams& P, cudaStream_t s, bool facet);
int gen_dispatch_tet1(int kh, int q, const GenParams& P, cudaStream_t s, bool facet);
int gen_dispatch_tet2(int kh, int q, const GenParams& P, cudaStream_t s, bool facet);
int gen_dispatch_hex2(int kh, int q, const GenParams& P, cudaStream_t s, bool facet);
int gen_dispatch_hexs2(int kh, int q, const GenParams& P, cudaStream_t s, bool facet);

}  // namespace fem
