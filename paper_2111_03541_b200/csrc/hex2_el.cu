// hex2_el.cu — NEXT-2 hot path: the elasticity domain form -(ε_ij, σ_ij) on quadratic cubes
// (27-node Lagrange, 20-node serendipity) with 2x2x2 or 3x3x3 Gauss points, one element per CTA,
// the element Gram on the fp64 tensor cores.
//
// D-3 gives per element, with G_a(γ) = J^{-T} ∇̂N_a(ξ_γ) and w_γ = ŵ_γ det J (reading L1),
//   K_(a,i),(b,m) = -f0 (λ M^im_ab + μ M^mi_ab + μ δ_im tr M_ab),   M^jk_ab = Σ_γ w_γ G_aj(γ) G_bk(γ),
// i.e. M is the (3 NL) x (3 NL) Gram matrix of the gradient table Gm[(a,j)][γ] under the weights w:
// 81 x 81 (Q2) or 60 x 60 (serendipity) with 27 or 8 inner terms.  It is symmetric, so the CTA's warps
// compute the upper 8x8 tiles with mma.m8n8k4.f64 (66 tiles x 7 k-steps = 462 DMMA for Q2) and mirror
// them into shared memory; then one thread per node pair (a, b) forms the 3x3 block of K from the
// 9 entries of M's (a, b) block and scatters it through the slot map — fp64 RED (FEM_SCATTER_ATOMIC) or
// plain read-modify-write inside one colour (FEM_SCATTER_COLOURED, deterministic).  The residual
// r_(a,i) = -Σ_γ Σ_j G_aj(γ) w_γ σ_ij(γ) (D-2) comes from the per-point stress of ∇d(γ) = Σ_b d_b ⊗ G_b(γ).
// Boundary terms stay in the generic facet kernel.
#include <cstdint>

#include "assemble_generic.cuh"

namespace fem {

constexpr int Q2_THREADS = 256;

__device__ __forceinline__ void dmma884_q2(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

// reference gradient of node a of the quadratic cube at ξ (one node at a time: no 27 x 3 register arrays)
template <int ET>
__device__ __forceinline__ void q2_node_grad(int a, const double* xi, double* g) {
  if constexpr (ET == ET_HEXS) {
    const SerendipityNode sn(a, xi);
    g[0] = sn.g[0]; g[1] = sn.g[1]; g[2] = sn.g[2];
  } else {
    double v[3], d1[3], d2[3];
    for (int d = 0; d < 3; d++) lq1(qc_coord(a, d), xi[d], v[d], d1[d], d2[d]);
    g[0] = d1[0] * v[1] * v[2];
    g[1] = v[0] * d1[1] * v[2];
    g[2] = v[0] * v[1] * d1[2];
  }
}

template <int ET, int Q1D>
struct Q2Cfg {
  static constexpr int NL = ET == ET_HEXS ? 20 : 27;
  static constexpr int NQ = Q1D * Q1D * Q1D;
  static constexpr int KP = (NQ + 3) / 4 * 4;  // inner dimension padded to the k-step
  static constexpr int R = 3 * NL;              // rows (a, j)
  static constexpr int RP = (R + 7) / 8 * 8;    // padded to the 8-row tiles
  static constexpr int NT = RP / 8;             // tiles per side
  static constexpr int MS = RP + 1;             // row stride of M in shared memory (odd: fewer conflicts)
  // shared memory (doubles): X[3][NL] | D[3][NL] | Gm[RP][KP] | w[KP] | Ji[NQ][9] | Sw[NQ][9] | M[RP][MS] |
  // ref[NQ][NL][3] (the reference gradients ∇̂N_a(ξ_γ), the same for every element: built once per CTA)
  static constexpr int O_X = 0, O_D = 3 * NL, O_G = 6 * NL, O_W = O_G + RP * KP, O_JI = O_W + KP,
                       O_S = O_JI + 9 * NQ, O_M = O_S + 9 * NQ, O_REF = O_M + RP * MS, TOTAL = O_REF + 3 * NQ * NL;
};

template <int ET, int Q1D, bool HAS_V, bool HAS_R>
__global__ void __launch_bounds__(Q2_THREADS) k_q2_elast(const GenParams P) {
  using C = Q2Cfg<ET, Q1D>;
  constexpr int NL = C::NL, NQ = C::NQ, KP = C::KP, RP = C::RP, NT = C::NT, MS = C::MS;
  extern __shared__ __align__(16) double q2s[];
  double* X = q2s + C::O_X;
  double* Dn = q2s + C::O_D;
  double* Gm = q2s + C::O_G;
  double* Wq = q2s + C::O_W;
  double* Ji = q2s + C::O_JI;
  double* Sw = q2s + C::O_S;
  double* M = q2s + C::O_M;
  double* ref = q2s + C::O_REF;
  __shared__ int nodes[NL];
  __shared__ int bad;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int t = tid; t < NQ * NL; t += Q2_THREADS) {
    const int q = t / NL, a = t % NL;
    double xi[3], wr;
    Elem<ET_HEX, 1>::vol_qp(Q1D, q, xi, wr);
    q2_node_grad<ET>(a, xi, ref + 3 * t);
  }
  __syncthreads();
  const double lam = P.F.lam, mu = P.F.mu, f0 = P.F.f0;
  for (int64_t task = blockIdx.x; task < P.task_count; task += gridDim.x) {
    const int64_t ti = P.task_begin + task;
    const int64_t e = P.task_elem ? P.task_elem[ti] : ti;
    if (tid < NL) nodes[tid] = P.conn[(int64_t)tid * P.E + e];
    if (tid == 0) bad = 0;
    __syncthreads();
    for (int t = tid; t < 3 * NL; t += Q2_THREADS) {
      const int d = t / NL, a = t % NL;
      X[t] = P.coords[(int64_t)d * P.N + nodes[a]];
      if (HAS_R) Dn[t] = P.state[(int64_t)d * P.N + nodes[a]];
    }
    // zero the padding of the gradient table (rows >= 3 NL, points >= NQ)
    for (int t = tid; t < RP * KP; t += Q2_THREADS) {
      const int r = t / KP, k = t % KP;
      if (r >= 3 * NL || k >= NQ) Gm[t] = 0.0;
    }
    __syncthreads();
    // ---- geometry per point: J = Σ_a x_a ⊗ ∇̂N_a, det, J^{-1}, w = ŵ det J
    if (tid < NQ) {
      double xi[3], wr;
      Elem<ET_HEX, 1>::vol_qp(Q1D, tid, xi, wr);
      double J[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
      for (int a = 0; a < NL; a++) {
        const double* g = ref + 3 * (tid * NL + a);
#pragma unroll
        for (int i = 0; i < 3; i++)
#pragma unroll
          for (int j = 0; j < 3; j++) J[i][j] = fma(X[i * NL + a], g[j], J[i][j]);
      }
      double Jinv[3][3];
      const double det = inv_jac<3>(J, Jinv);
      if (!(det > 0.0)) {
        bad = 1;
        report_bad(P.err, e);
      }
      Wq[tid] = wr * det;
#pragma unroll
      for (int k = 0; k < 9; k++) Ji[tid * 9 + k] = Jinv[k / 3][k % 3];
    }
    __syncthreads();
    if (bad) { __syncthreads(); continue; }
    // ---- gradient table Gm[(a, j)][γ] = (J^{-T} ∇̂N_a(ξ_γ))_j
    for (int t = tid; t < NL * NQ; t += Q2_THREADS) {
      const int a = t / NQ, q = t % NQ;
      const double* g = ref + 3 * (q * NL + a);
      const double* J = Ji + q * 9;
#pragma unroll
      for (int i = 0; i < 3; i++) Gm[(3 * a + i) * KP + q] = J[0 * 3 + i] * g[0] + J[1 * 3 + i] * g[1] + J[2 * 3 + i] * g[2];
    }
    __syncthreads();
    if constexpr (HAS_R) {  // per point: w σ(∇d), ∇d_kj = Σ_b d_bk G_bj
      if (tid < NQ) {
        double gu[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
        for (int b = 0; b < NL; b++)
#pragma unroll
          for (int k = 0; k < 3; k++)
#pragma unroll
            for (int j = 0; j < 3; j++) gu[k][j] = fma(Dn[k * NL + b], Gm[(3 * b + j) * KP + tid], gu[k][j]);
        const double w = Wq[tid], div = gu[0][0] + gu[1][1] + gu[2][2];
#pragma unroll
        for (int i = 0; i < 3; i++)
#pragma unroll
          for (int j = 0; j < 3; j++) Sw[tid * 9 + i * 3 + j] = w * ((i == j ? lam * div : 0.0) + mu * (gu[i][j] + gu[j][i]));
      }
    }
    // ---- Gram M = Gm diag(w) Gm^T on the tensor cores: upper tiles (I <= J), mirrored
    if constexpr (HAS_V) {
      constexpr int NTILE = NT * (NT + 1) / 2;
      for (int tt = warp; tt < NTILE; tt += Q2_THREADS / 32) {
        int I = 0, rem = tt;
        while (rem >= NT - I) { rem -= NT - I; I++; }
        const int Jt = I + rem;
        double acc[2] = {0.0, 0.0};
        const int ra = 8 * I + (lane >> 2), rb = 8 * Jt + (lane >> 2);
#pragma unroll
        for (int k0 = 0; k0 < KP; k0 += 4) {
          const int k = k0 + (lane & 3);
          dmma884_q2(acc, Wq[k < NQ ? k : 0] * Gm[ra * KP + k], Gm[rb * KP + k]);
        }
        const int r = 8 * I + (lane >> 2), c0 = 8 * Jt + 2 * (lane & 3);
#pragma unroll
        for (int t = 0; t < 2; t++) {
          M[r * MS + c0 + t] = acc[t];
          if (Jt != I) M[(c0 + t) * MS + r] = acc[t];  // diagonal tiles: each entry written once
        }
      }
    }
    __syncthreads();
    // ---- rows of the owned nodes: K blocks and residual, scattered through the slot map
    for (int t = tid; t < NL * NL; t += Q2_THREADS) {
      const int a = t / NL, b = t % NL;
      const int node = nodes[a];
      if (node < P.own_lo || node >= P.own_hi) continue;
      const int64_t li = node - P.own_lo;
      const int64_t rps = P.rowptr_s[li];
      if constexpr (HAS_V) {
        if (P.values) {
          const int64_t deg = P.rowptr_s[li + 1] - rps;
          const int64_t off = (int64_t)P.slot[((int64_t)a * NL + b) * P.E + e] - rps;
          const double* Mab = M + (3 * a) * MS + 3 * b;  // M[(a, j)][(b, k)] = Mab[j * MS + k]
          const double tr = Mab[0] + Mab[MS + 1] + Mab[2 * MS + 2];
#pragma unroll
          for (int i = 0; i < 3; i++) {
            double* rowp = P.values + (int64_t)i * 3 * P.nnz_s + 3 * rps + off;
#pragma unroll
            for (int m = 0; m < 3; m++) {
              const double kv = -f0 * (lam * Mab[i * MS + m] + mu * Mab[m * MS + i] + (i == m ? mu * tr : 0.0));
              double* dst = rowp + m * deg;
              if (P.plain) *dst += kv;
              else atomicAdd(dst, kv);
            }
          }
        }
      }
    }
    if constexpr (HAS_R) {
      for (int t = tid; t < 3 * NL; t += Q2_THREADS) {
        const int a = t / 3, i = t % 3;
        const int node = nodes[a];
        if (node < P.own_lo || node >= P.own_hi) continue;
        double r = 0.0;
        for (int q = 0; q < NQ; q++)
#pragma unroll
          for (int j = 0; j < 3; j++) r = fma(Sw[q * 9 + i * 3 + j], Gm[(3 * a + j) * KP + q], r);
        double* dst = P.rhs + (int64_t)i * P.n_own + (node - P.own_lo);
        if (P.plain) *dst -= r;
        else atomicAdd(dst, -r);
      }
    }
    __syncthreads();
  }
}

template <int ET, int Q1D, bool HAS_V, bool HAS_R>
static int run_q2(const GenParams& P, cudaStream_t s) {
  using C = Q2Cfg<ET, Q1D>;
  auto kern = k_q2_elast<ET, Q1D, HAS_V, HAS_R>;
  const size_t smem = sizeof(double) * C::TOTAL;
  FEM_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  if (P.task_count <= 0) return 0;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t grid = std::min<int64_t>(P.task_count, (int64_t)sms * 2);
  kern<<<(unsigned)grid, Q2_THREADS, smem, s>>>(P);
  FEM_CUDA_TRY(cudaGetLastError());
  return 0;
}

template <int ET, int Q1D>
static int run_q2_kind(const GenParams& P, cudaStream_t s) {
  if (P.values && P.rhs) return run_q2<ET, Q1D, true, true>(P, s);
  if (P.values) return run_q2<ET, Q1D, true, false>(P, s);
  return run_q2<ET, Q1D, false, true>(P, s);
}

// Quadratic-cube elasticity domain term (ELAST_DOMAIN, κ̂ = 3): 1 if handled.
int launch_q2_elast(const AsmArgs& A, int* handled) {
  *handled = 0;
  const fem_mesh_s* m = A.m;
  if (A.ek || A.er || m->order != 2 || (m->etype != ET_HEX && m->etype != ET_HEXS) || m->kh != 3 ||
      A.F.form != FEM_WF_ELAST_DOMAIN || (A.quad_order != 2 && A.quad_order != 3))
    return 0;
  *handled = 1;
  GenParams P;
  P.F = A.F;
  P.N = m->N; P.E = m->E; P.own_lo = m->own_lo; P.own_hi = m->own_hi; P.n_own = m->n_own;
  P.nnz_s = A.pat ? A.pat->nnz_s : 0;
  P.coords = m->coords; P.conn = m->conn; P.state = A.state;
  P.nu_hat = A.F.nu_hat;
  P.task_elem = A.task_elem; P.task_facet = nullptr;
  P.task_begin = A.task_begin; P.task_count = A.task_count;
  P.values = A.values; P.rhs = A.rhs;
  P.slot = A.pat ? A.pat->slot : nullptr;
  P.rowptr_s = A.pat ? A.pat->rowptr_s : nullptr;
  P.plain = A.plain;
  P.err = m->err;
  if (m->etype == ET_HEX)
    return A.quad_order == 3 ? run_q2_kind<ET_HEX, 3>(P, A.stream) : run_q2_kind<ET_HEX, 2>(P, A.stream);
  return A.quad_order == 3 ? run_q2_kind<ET_HEXS, 3>(P, A.stream) : run_q2_kind<ET_HEXS, 2>(P, A.stream);
}

}  // namespace fem
