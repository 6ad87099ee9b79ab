// tet2_el.cu — the c3 hot path: linear elasticity -(ε_ij, σ_ij) on P2 (10-node)
// tetrahedra with the 4-point degree-2 rule, node-tile owner gather (tiled.cu records).
//
// One warp per element visit, everything as small GEMMs on the fp64 tensor cores:
//   geometry   [J(γ) | ∇̂d(γ)]_{r,(γ,j)} = Σ_a [x_a; d_a]_r ∇̂N_a(ξ_γ)_j   (6 x 10) · (10 x 12): 6 DMMA
//              (J is evaluated at every point, so curved P2 elements stay exact);
//   Gram       M^{jk}_{ab} = Σ_γ w_γ G_aj(γ) G_bk(γ) over the 4 points = one k-step of m8n8k4:
//              lane l = 4a + c holds ∇N_{a}(ξ_c) and ∇N_{8+(a&1)}(ξ_c), the A/B fragments of three 8x8
//              node tiles that with the symmetry of K cover the 10x10 node block: 27 DMMA;
//   K_(a,i),(b,m) = -f0 (λ M^im + μ M^mi + μ δ_im tr M);  r_(a,i) = -Σ_γ w σ_ij G_aj.
// Contributions go to the tile accumulator in record order under per-row turns (FEM_SCATTER_TILED,
// deterministic) or with shared-memory fp64 atomics (FEM_SCATTER_TILED_UNORDERED).
#include <algorithm>
#include <cstdlib>
#include <string>

#include "tiled.cuh"

namespace fem {

__device__ __forceinline__ void dmma884_t2(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

__device__ __forceinline__ double sum4_t2(double v) {
  v += __shfl_xor_sync(0xffffffffu, v, 1);
  v += __shfl_xor_sync(0xffffffffu, v, 2);
  return v;
}

struct P2Offs {
  uint32_t vown, vhal, velem, vloc, hdat, tdeg, toff, acc, racc, vseq, turn;
  int H, T;
};
constexpr int P2_LANE_TAB = 12;   // GEMM B fragments (3 k-steps x 2 n-tiles) | ∇̂N_a0(ξ_c) | ∇̂N_{8+(a0&1)}(ξ_c)
constexpr int P2_SCRATCH = 80;    // doubles per warp: GEMM output (6 x 12) then 4 point records of 20
constexpr int P2_FACET_WARPS = 8;

struct P2Coef {
  double cl, cm, sl, sm;  // Σ f0 λ, Σ f0 μ (matrix); Σ λ, Σ μ (residual)
};

// acquire / release on a shared-memory turn counter (scope CTA)
__device__ __forceinline__ int p2_ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.cta.shared::cta.b32 %0, [%1];" : "=r"(v) : "r"((uint32_t)__cvta_generic_to_shared(p)) : "memory");
  return v;
}
__device__ __forceinline__ void p2_st_release(int* p, int v) {
  asm volatile("st.release.cta.shared::cta.b32 [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(p)), "r"(v) : "memory");
}

// HAS_V / HAS_R: the call kind (matrix, residual, both) fixed per launch, so each body compiles lean.
// ORD (FEM_SCATTER_TILED): every contribution is formed first; the visit then takes its turn (record
// order, vseq) on each tile row it writes, adds with plain read-modify-writes and passes the turns on, so
// each accumulator entry sums its contributions in a fixed order.  !ORD: shared-memory fp64 atomics.
template <bool HAS_V, bool HAS_R, bool ORD = false>
__device__ __forceinline__ void p2_visit(const TiledParams& P, const P2Offs& to, const P2Coef& H,
                                         const double* __restrict__ lt, double* sc, int v, unsigned char* sm) {
  const int lane = threadIdx.x & 31;
  const int c = lane & 3, r = lane >> 2;
  const int16_t* own = reinterpret_cast<const int16_t*>(sm + to.vown) + v * 10;
  const uint16_t* hv = reinterpret_cast<const uint16_t*>(sm + to.vhal) + v * 10;
  const double* hdat = reinterpret_cast<const double*>(sm + to.hdat);
  const int HH = to.H;
  const double* L = lt + lane;  // lane table, transposed: L[32 k] = constant k of this lane (conflict-free)
  // ---- geometry GEMM
  double C2[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
#pragma unroll
  for (int s = 0; s < 3; s++) {
    const int k = 4 * s + c;
    const double av = (r < 6 && k < 10) ? hdat[r * HH + hv[k]] : 0.0;
#pragma unroll
    for (int t = 0; t < 2; t++) dmma884_t2(C2[t], av, L[32 * (s * 2 + t)]);
  }
  if (r < 6) {
#pragma unroll
    for (int t = 0; t < 2; t++)
#pragma unroll
      for (int i = 0; i < 2; i++) {
        const int n = 8 * t + 2 * c + i;
        if (n < 12) sc[r * 12 + n] = C2[t][i];
      }
  }
  __syncwarp();
  // ---- per point q = lane >> 3 (8 lanes per point)
  const int q = lane >> 3;
  double J[3][3], Dr[3][3];
#pragma unroll
  for (int i = 0; i < 3; i++)
#pragma unroll
    for (int j = 0; j < 3; j++) {
      J[i][j] = sc[i * 12 + 3 * q + j];
      if constexpr (HAS_R) Dr[i][j] = sc[(3 + i) * 12 + 3 * q + j];
    }
  const double c00 = J[1][1] * J[2][2] - J[1][2] * J[2][1];
  const double c01 = J[1][2] * J[2][0] - J[1][0] * J[2][2];
  const double c02 = J[1][0] * J[2][1] - J[1][1] * J[2][0];
  const double det = J[0][0] * c00 + J[0][1] * c01 + J[0][2] * c02;
  if (__any_sync(0xffffffffu, !(det > 0.0))) {
    if (lane == 0)
      atomicCAS((unsigned long long*)P.err, (unsigned long long)(-1LL),
                (unsigned long long)reinterpret_cast<const int32_t*>(sm + to.velem)[v]);
    if constexpr (ORD) {  // pass the turns on, or later visits of these rows would wait forever
      const int16_t* ow = reinterpret_cast<const int16_t*>(sm + to.vown) + v * 10;
      const uint8_t* sq = sm + to.vseq + v * 10;
      int* turn = reinterpret_cast<int*>(sm + to.turn);
      if (lane < 10 && ow[lane] >= 0) {
        while (p2_ld_acquire(turn + ow[lane]) != sq[lane]) __nanosleep(32);
        p2_st_release(turn + ow[lane], sq[lane] + 1);
      }
    }
    __syncwarp();
    return;
  }
  __syncwarp();
  if ((lane & 7) == 0) {
    const double rr = 1.0 / det;
    double Ji[3][3];
    Ji[0][0] = c00 * rr; Ji[1][0] = c01 * rr; Ji[2][0] = c02 * rr;
    Ji[0][1] = (J[0][2] * J[2][1] - J[0][1] * J[2][2]) * rr;
    Ji[1][1] = (J[0][0] * J[2][2] - J[0][2] * J[2][0]) * rr;
    Ji[2][1] = (J[0][1] * J[2][0] - J[0][0] * J[2][1]) * rr;
    Ji[0][2] = (J[0][1] * J[1][2] - J[0][2] * J[1][1]) * rr;
    Ji[1][2] = (J[0][2] * J[1][0] - J[0][0] * J[1][2]) * rr;
    Ji[2][2] = (J[0][0] * J[1][1] - J[0][1] * J[1][0]) * rr;
    double* o = sc + q * 20;
#pragma unroll
    for (int j = 0; j < 3; j++)
#pragma unroll
      for (int i = 0; i < 3; i++) o[j * 3 + i] = Ji[j][i];
    const double w = det * (1.0 / 24.0);  // 4-point rule weight 1/24
    o[9] = w;
    if constexpr (HAS_R) {
      double gu[3][3];
#pragma unroll
      for (int k = 0; k < 3; k++)
#pragma unroll
        for (int i = 0; i < 3; i++) gu[k][i] = Dr[k][0] * Ji[0][i] + Dr[k][1] * Ji[1][i] + Dr[k][2] * Ji[2][i];
      const double lw = H.sl * w * (gu[0][0] + gu[1][1] + gu[2][2]), mw = H.sm * w;
#pragma unroll
      for (int i = 0; i < 3; i++)
#pragma unroll
        for (int j = 0; j < 3; j++) o[10 + i * 3 + j] = (i == j ? lw : 0.0) + mw * (gu[i][j] + gu[j][i]);
    }
  }
  __syncwarp();
  // ---- fragment layout: lane (a0, c) holds G of node a0 and of node a1 = 8 + (a0 & 1) at point c
  const int a0 = r, a1 = 8 + (r & 1);
  const double* o = sc + c * 20;
  double G0[3], G1[3];
#pragma unroll
  for (int i = 0; i < 3; i++) {
    G0[i] = o[0 * 3 + i] * L[32 * 6] + o[1 * 3 + i] * L[32 * 7] + o[2 * 3 + i] * L[32 * 8];
    G1[i] = o[0 * 3 + i] * L[32 * 9] + o[1 * 3 + i] * L[32 * 10] + o[2 * 3 + i] * L[32 * 11];
  }
  const double w = o[9];
  const int li0 = own[a0], li1 = own[a1];
  double res0[3] = {0.0, 0.0, 0.0}, res1[3] = {0.0, 0.0, 0.0};
  if constexpr (HAS_R) {  // r_(a,i) = -Σ_γ w σ_ij G_aj, reduced over the 4 points (lanes c)
#pragma unroll
    for (int i = 0; i < 3; i++) {
      double t0 = 0.0, t1 = 0.0;
#pragma unroll
      for (int j = 0; j < 3; j++) {
        t0 = fma(o[10 + i * 3 + j], G0[j], t0);
        t1 = fma(o[10 + i * 3 + j], G1[j], t1);
      }
      res0[i] = -sum4_t2(t0);
      res1[i] = -sum4_t2(t1);
      if constexpr (!ORD) {
        double* racc = reinterpret_cast<double*>(sm + to.racc);
        if (c == 0 && li0 >= 0) atomicAdd(racc + i * to.T + li0, res0[i]);
        if (c == 0 && r < 2 && li1 >= 0) atomicAdd(racc + i * to.T + li1, res1[i]);
      }
    }
  }
  if constexpr (!HAS_V && !ORD) {
    __syncwarp();
    return;
  }
  const int32_t* tdeg = reinterpret_cast<const int32_t*>(sm + to.tdeg);
  const int32_t* toff = reinterpret_cast<const int32_t*>(sm + to.toff);
  double* acc = reinterpret_cast<double*>(sm + to.acc);
  const uint8_t* vloc = sm + to.vloc + v * 100;
  // K_(a,i),(b,m) = -(cl M^im_ab + cm M^mi_ab + cm δ_im tr M_ab) is symmetric: K_(b,m),(a,i) = K_(a,i),(b,m).
  // Three 8x8 node tiles cover all 100 (a,b) blocks: [0..7]x[0..7] (both orders), [0..7]x{8,9} (each
  // result written as the block and its transpose) and {8,9}x{8,9}; the columns of the last two are
  // the nodes 8 + (n & 1), so lane (a0, c) holds pair (.., 8 + t) twice over c and picks t = c & 1.
  double M[3][3][2];
  auto gram = [&](const double* A, const double* B) {
#pragma unroll
    for (int j = 0; j < 3; j++)
#pragma unroll
      for (int k = 0; k < 3; k++) {
        M[j][k][0] = 0.0;
        M[j][k][1] = 0.0;
        dmma884_t2(M[j][k], w * A[j], B[k]);
      }
  };
  double K1[2][9], K2[9], K3[9];  // the lane's contributions: tile 1 (two blocks), tile 2, tile 3
  if constexpr (HAS_V) {
    gram(G0, G0);
#pragma unroll
    for (int t = 0; t < 2; t++) {
      const double tr = M[0][0][t] + M[1][1][t] + M[2][2][t];
#pragma unroll
      for (int i = 0; i < 3; i++)
#pragma unroll
        for (int m = 0; m < 3; m++) K1[t][i * 3 + m] = -(H.cl * M[i][m][t] + H.cm * M[m][i][t] + (i == m ? H.cm * tr : 0.0));
    }
    gram(G0, G1);
    {
      const int t = c & 1;
      double Ms[3][3];
#pragma unroll
      for (int j = 0; j < 3; j++)
#pragma unroll
        for (int k = 0; k < 3; k++) Ms[j][k] = t ? M[j][k][1] : M[j][k][0];
      const double tr = Ms[0][0] + Ms[1][1] + Ms[2][2];
#pragma unroll
      for (int i = 0; i < 3; i++)
#pragma unroll
        for (int m = 0; m < 3; m++) K2[i * 3 + m] = -(H.cl * Ms[i][m] + H.cm * Ms[m][i] + (i == m ? H.cm * tr : 0.0));
    }
    gram(G1, G1);
    {
      const int t = c & 1;
      double Ms[3][3];
#pragma unroll
      for (int j = 0; j < 3; j++)
#pragma unroll
        for (int k = 0; k < 3; k++) Ms[j][k] = t ? M[j][k][1] : M[j][k][0];
      const double tr = Ms[0][0] + Ms[1][1] + Ms[2][2];
#pragma unroll
      for (int i = 0; i < 3; i++)
#pragma unroll
        for (int m = 0; m < 3; m++) K3[i * 3 + m] = -(H.cl * Ms[i][m] + H.cm * Ms[m][i] + (i == m ? H.cm * tr : 0.0));
    }
  }
  // ---- ordered: the turns of the rows this visit writes (rows a0 by lanes (a0, 0); rows 8, 9 by (0..1, 1))
  int* turn = reinterpret_cast<int*>(sm + to.turn);
  const uint8_t* sq = sm + to.vseq + v * 10;
  const int trow = c == 0 ? li0 : ((c == 1 && r < 2) ? li1 : -1);
  const int tturn = c == 0 ? sq[a0] : ((c == 1 && r < 2) ? sq[8 + r] : 0);
  if constexpr (ORD) {
    if (trow >= 0)
      while (p2_ld_acquire(turn + trow) != tturn) __nanosleep(32);
    __syncwarp();
  }
  auto add = [&](double* p, double x) {
    if constexpr (ORD) *p += x;
    else atomicAdd(p, x);
  };
  if constexpr (HAS_V) {
    // tile 1: rows a0, columns b = 2c + t
    if (li0 >= 0) {
      const int d = tdeg[li0], sr = acc_row_stride(3, d, P.nnz_s);
      double* base = acc + toff[li0];
#pragma unroll
      for (int t = 0; t < 2; t++) {
        double* rowb = base + vloc[a0 * 10 + 2 * c + t];
#pragma unroll
        for (int i = 0; i < 3; i++)
#pragma unroll
          for (int m = 0; m < 3; m++) add(rowb + i * sr + m * d, K1[t][i * 3 + m]);
      }
    }
    // tile 2: pair (a0, 8 + t); c < 2 writes block (a0, 8 + c), c >= 2 the transposed block (8 + c - 2, a0)
    {
      const int t = c & 1;
      const bool tr_blk = c >= 2;
      const int ra = tr_blk ? 8 + t : a0, cb = tr_blk ? a0 : 8 + t;
      const int li = own[ra];
      if (li >= 0) {
        double* rowb = acc + toff[li] + vloc[ra * 10 + cb];
        const int d = tdeg[li], sr = acc_row_stride(3, d, P.nnz_s);
#pragma unroll
        for (int i = 0; i < 3; i++)
#pragma unroll
          for (int m = 0; m < 3; m++) add(rowb + (tr_blk ? m * sr + i * d : i * sr + m * d), K2[i * 3 + m]);
      }
    }
    // tile 3: pair (8 + (a0 & 1), 8 + t): lanes a0 < 2, c < 2 write block (8 + a0, 8 + c)
    if (r < 2 && c < 2 && li1 >= 0) {
      double* rowb = acc + toff[li1] + vloc[a1 * 10 + 8 + c];
      const int d = tdeg[li1], sr = acc_row_stride(3, d, P.nnz_s);
#pragma unroll
      for (int i = 0; i < 3; i++)
#pragma unroll
        for (int m = 0; m < 3; m++) add(rowb + i * sr + m * d, K3[i * 3 + m]);
    }
  }
  if constexpr (HAS_R && ORD) {
    double* racc = reinterpret_cast<double*>(sm + to.racc);
#pragma unroll
    for (int i = 0; i < 3; i++) {
      if (c == 0 && li0 >= 0) racc[i * to.T + li0] += res0[i];
      if (c == 0 && r < 2 && li1 >= 0) racc[i * to.T + li1] += res1[i];
    }
  }
  __syncwarp();
  if constexpr (ORD) {
    if (trow >= 0) p2_st_release(turn + trow, tturn + 1);
  }
  __syncwarp();
}

__device__ __forceinline__ void p2_gather_halo(const TiledParams& P, const uint8_t* rec, double* hbuf) {
  const int32_t* hdr = reinterpret_cast<const int32_t*>(rec);
  const RecLayout L = rec_layout_hdr(10, hdr);
  const int32_t* hn = reinterpret_cast<const int32_t*>(rec + L.o_hnode);
  const int H = hdr[1];
  for (int cc = 0; cc < P.hcomp; cc++) {  // component-major: no integer division per element
    const double* base = cc < 3 ? P.coords + (int64_t)cc * P.N : P.state + (int64_t)(cc - 3) * P.N;
    for (int i = threadIdx.x; i < H; i += blockDim.x) cp_async8(hbuf + cc * H + i, base + hn[i]);
  }
  cp_async_commit();
}

template <bool ORD>
__global__ void __launch_bounds__(TILED_THREADS, 1) k_p2_rec(const __grid_constant__ TiledParams P) {
  using C = TileCfg<ET_TET, 2, 3, 2>;
  extern __shared__ __align__(16) unsigned char smem[];
  uint64_t* mbar = reinterpret_cast<uint64_t*>(smem);
  int* ctr = reinterpret_cast<int*>(smem + 64);
  __shared__ P2Offs to;
  __shared__ double lanetab[32 * P2_LANE_TAB];
#define P2RBUF(i) (smem + 128 + (size_t)(i) * P.rec_cap)
#define P2HBUF(i) (reinterpret_cast<double*>(smem + 128 + 2 * (size_t)P.rec_cap) + (size_t)(i) * P.hcap)
  double* acc = P2HBUF(2);
  int* turn = reinterpret_cast<int*>(acc + P.acc_cap);
  TileSmem F;
  unsigned char* fp = reinterpret_cast<unsigned char*>(turn + P.turn_cap);
  F.qp = fp;
  fp += std::max((size_t)P.rec_bytes * P2_FACET_WARPS, (size_t)8 * P2_SCRATCH * C::WARPS);
  F.vid = reinterpret_cast<int32_t*>(fp);
  F.vnode = nullptr;
  F.vfac = nullptr;
  F.hnode = nullptr;
  F.hdat = nullptr;
  F.H = 0;
  P2Coef Hc = {0, 0, 0, 0};
  for (int f = 0; f < P.n_dom; f++) {
    const FormArgs& Fm = P.dom[f];
    Hc.cl += Fm.f0 * Fm.lam; Hc.cm += Fm.f0 * Fm.mu; Hc.sl += Fm.lam; Hc.sm += Fm.mu;
  }
  const int tid = threadIdx.x, warp = tid >> 5;
  if (warp == 0) {  // per-lane constants: GEMM B fragments and reference gradients at the lane's point
    using EL = Elem<ET_TET, 2>;
    double* Lt = lanetab + tid;  // transposed: constant k of lane l at 32 k + l
    for (int s = 0; s < 3; s++)
      for (int t = 0; t < 2; t++) {
        const int k = 4 * s + (tid & 3), n = 8 * t + (tid >> 2);
        double val = 0.0;
        if (k < 10 && n < 12) {
          double xi[3], wq, N[10], dN[10][3];
          EL::vol_qp(2, n / 3, xi, wq);
          EL::shape(xi, N, dN);
          val = dN[k][n % 3];
        }
        Lt[32 * (s * 2 + t)] = val;
      }
    double xi[3], wq, N[10], dN[10][3];
    EL::vol_qp(2, tid & 3, xi, wq);
    EL::shape(xi, N, dN);
    const int a0 = tid >> 2, a1 = 8 + (a0 & 1);
    for (int i = 0; i < 3; i++) {
      Lt[32 * (6 + i)] = dN[a0][i];
      Lt[32 * (9 + i)] = dN[a1][i];
    }
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
    bulk_g2s(P2RBUF(0), P.rec + P.rec_off[tile], bytes, &mbar[0]);
  }
  mbar_wait(&mbar[0], 0);
  p2_gather_halo(P, P2RBUF(0), P2HBUF(0));
  for (int it = 0; tile < P.n_tiles; it++, tile += gridDim.x) {
    const int cur = it & 1, oth = cur ^ 1;
    const int64_t next = tile + gridDim.x;
    if (tid == 0 && next < P.n_tiles) {
      const uint32_t bytes = (uint32_t)(P.rec_off[next + 1] - P.rec_off[next]);
      mbar_expect_tx(&mbar[oth], bytes);
      bulk_g2s(P2RBUF(oth), P.rec + P.rec_off[next], bytes, &mbar[oth]);
    }
    const uint8_t* rec = P2RBUF(cur);
    const int32_t* hdr = reinterpret_cast<const int32_t*>(rec);
    const int T = hdr[0], H = hdr[1], nv = hdr[2], acc_n = P.values ? hdr[4] : 0;
    const uint32_t fmask = (uint32_t)hdr[5];
    const RecLayout L = rec_layout_hdr(10, hdr);
    if (tid == 0) {
      *ctr = 0;
      const uint32_t rb = (uint32_t)(rec - smem);
      to.vown = rb + L.o_vown; to.vhal = rb + L.o_vhal; to.velem = rb + L.o_velem; to.vloc = rb + L.o_vloc;
      to.hdat = (uint32_t)(reinterpret_cast<const unsigned char*>(P2HBUF(cur)) - smem);
      to.tdeg = rb + L.o_tdeg; to.toff = rb + L.o_toff;
      to.acc = (uint32_t)(reinterpret_cast<unsigned char*>(acc) - smem);
      to.racc = to.acc + 8u * (uint32_t)acc_n;
      to.vseq = rb + L.o_vseq;
      to.turn = (uint32_t)(reinterpret_cast<unsigned char*>(turn) - smem);
      to.H = H;
      to.T = T;
    }
    for (int i = tid; i < acc_n + 3 * T; i += blockDim.x) acc[i] = 0.0;
    if constexpr (ORD)
      for (int i = tid; i < T; i += blockDim.x) turn[i] = 0;
    cp_async_wait_all();
    __syncthreads();
    double* wsc = reinterpret_cast<double*>(F.qp) + (size_t)P2_SCRATCH * warp;
    if (P.values && P.rhs)
      for (int v = grab_visits(ctr, 1); v < nv; v = grab_visits(ctr, 1)) p2_visit<true, true, ORD>(P, to, Hc, lanetab, wsc, v, smem);
    else if (P.values)
      for (int v = grab_visits(ctr, 1); v < nv; v = grab_visits(ctr, 1)) p2_visit<true, false, ORD>(P, to, Hc, lanetab, wsc, v, smem);
    else
      for (int v = grab_visits(ctr, 1); v < nv; v = grab_visits(ctr, 1)) p2_visit<false, true, ORD>(P, to, Hc, lanetab, wsc, v, smem);
    if (next < P.n_tiles) {
      mbar_wait(&mbar[oth], (uint32_t)(((it + 1) >> 1) & 1));
      p2_gather_halo(P, P2RBUF(oth), P2HBUF(oth));
    }
    F.tnode = const_cast<int32_t*>(reinterpret_cast<const int32_t*>(rec + L.o_tnode));
    F.tdeg = const_cast<int32_t*>(reinterpret_cast<const int32_t*>(rec + L.o_tdeg));
    F.toff = const_cast<int32_t*>(reinterpret_cast<const int32_t*>(rec + L.o_toff));
    F.trps = const_cast<int64_t*>(reinterpret_cast<const int64_t*>(rec + L.o_trps));
    F.acc = acc;
    F.racc = acc + acc_n;
    F.T = T;
    F.vid = const_cast<int32_t*>(reinterpret_cast<const int32_t*>(rec + L.o_velem));
    F.vown = const_cast<int16_t*>(reinterpret_cast<const int16_t*>(rec + L.o_vown));
    F.vhal = const_cast<int16_t*>(reinterpret_cast<const int16_t*>(rec + L.o_vhal));
    F.vloc = rec + L.o_vloc;
    F.hdat = P2HBUF(cur);
    F.H = H;
    if (fmask) rec_facets<ET_TET, 2, 3, 2, P2_FACET_WARPS, ORD>(P, F, rec, L, F.qp + (size_t)P.rec_bytes * (warp % P2_FACET_WARPS));
    tile_epilogue<3>(P, F);
    __syncthreads();
  }
#undef P2RBUF
#undef P2HBUF
}

// P2 tets, 4-point rule, domain terms all ELAST_DOMAIN.
int launch_p2_tiled(TiledParams& P, const TileSchedule& T, bool det, cudaStream_t s, bool* handled) {
  *handled = false;
  if (P.n_dom == 0 || !T.rec) return 0;
  for (int f = 0; f < P.n_dom; f++)
    if (P.dom[f].form != FEM_WF_ELAST_DOMAIN) return 0;
  *handled = true;
  if (det && T.max_turns > 255) {
    set_error("tiled scatter: a tile point is touched by more than 255 element visits (8-bit turns); use "
              "FEM_SCATTER_COLOURED or FEM_SCATTER_TILED_UNORDERED");
    return FEM_E_UNSUPPORTED;
  }
  P.turn_cap = (int)((T.max_tile_nodes + 3) / 4 * 4);
  using C = TileCfg<ET_TET, 2, 3, 2>;
  P.rec_bytes = (int)((sizeof(typename C::QPG) * C::NQF + 15) / 16 * 16);
  P.fvmax = 1;
  P.vmax = 1;
  P.hmax = 0;
  P.hcomp = 3 + 3 * (P.nu_hat >= 1 ? 2 : 1);
  P.rec = T.rec;
  P.rec_off = T.rec_off;
  P.n_tiles = T.n_tiles;
  P.rec_cap = (int)((T.rec_max + 15) / 16 * 16);
  P.hcap = (int)(((T.max_halo * P.hcomp) + 1) / 2 * 2);
  P.acc_cap = (int)((P.values ? T.acc_max : 0) + (int64_t)3 * T.max_tile_nodes);
  P.acc_cap = (P.acc_cap + 1) / 2 * 2;
  const size_t fac_bytes = std::max((size_t)P.rec_bytes * P2_FACET_WARPS, (size_t)8 * P2_SCRATCH * C::WARPS) + 16;
  const size_t smem = 128 + 2 * (size_t)P.rec_cap + 2 * 8 * (size_t)P.hcap + 8 * (size_t)P.acc_cap +
                      4 * (size_t)P.turn_cap + fac_bytes;
  if (smem + 4096 > 227 * 1024) {
    set_error("P2 record kernel: shared memory request too large (" + std::to_string(smem) + " B)");
    return FEM_E_UNSUPPORTED;
  }
  auto kern = det ? k_p2_rec<true> : k_p2_rec<false>;
  FEM_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  if (T.n_tiles <= 0) return 0;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t grid = std::min<int64_t>(T.n_tiles, sms);
  kern<<<(unsigned)grid, TILED_THREADS, smem, s>>>(P);
  FEM_CUDA_TRY(cudaGetLastError());
  return 0;
}


// ---- FEM_SCATTER_STORED element pass (stored.cu): one warp per element, the visit arithmetic above with the
// element's points gathered straight from HBM (the warp's next element's node ids and coordinates load while
// the current one computes); the upper blocks a <= b of the symmetric 10 x 10 block matrix K^e (55 of 100:
// tile 1 where b >= a, tile 2 without its transposes, tile 3 where b >= a) and the residual rows are staged
// in shared memory and stored as one contiguous coalesced stream at the element's Morton position pos:
// ek[pos][blk][i][m] (blk packed row by row), er[pos][a][i].
constexpr int P2E_WARPS = 8;
__device__ __forceinline__ int p2_ublk(int a, int b) { return a * 10 - a * (a - 1) / 2 + (b - a); }

template <bool HAS_V, bool HAS_R>
__global__ void __launch_bounds__(32 * P2E_WARPS) k_p2_el(const double* __restrict__ coords, const double* __restrict__ state,
                                                         const int32_t* __restrict__ conn, int64_t N, int64_t E,
                                                         const int32_t* __restrict__ eperm, P2Coef H,
                                                         double* __restrict__ ek, double* __restrict__ er, long long* err) {
  __shared__ double lanetab[32 * P2_LANE_TAB];
  __shared__ double scr[P2E_WARPS][P2_SCRATCH];
  // per-warp staging of the element's 55 blocks (+ 30 residual rows): the lanes' scattered 72-byte blocks
  // leave as one contiguous, coalesced 3960-byte store stream per element
  __shared__ double stage[P2E_WARPS][55 * 9 + 30];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (warp == 0) {  // per-lane constants, as in k_p2_rec
    using EL = Elem<ET_TET, 2>;
    double* Lt = lanetab + tid;
    for (int s = 0; s < 3; s++)
      for (int t = 0; t < 2; t++) {
        const int k = 4 * s + (tid & 3), n = 8 * t + (tid >> 2);
        double val = 0.0;
        if (k < 10 && n < 12) {
          double xi[3], wq, Nn[10], dN[10][3];
          EL::vol_qp(2, n / 3, xi, wq);
          EL::shape(xi, Nn, dN);
          val = dN[k][n % 3];
        }
        Lt[32 * (s * 2 + t)] = val;
      }
    double xi[3], wq, Nn[10], dN[10][3];
    EL::vol_qp(2, tid & 3, xi, wq);
    EL::shape(xi, Nn, dN);
    const int a0 = tid >> 2, a1 = 8 + (a0 & 1);
    for (int i = 0; i < 3; i++) {
      Lt[32 * (6 + i)] = dN[a0][i];
      Lt[32 * (9 + i)] = dN[a1][i];
    }
  }
  __syncthreads();
  const int c = lane & 3, r = lane >> 2;
  const double* L = lanetab + lane;
  double* sc = scr[warp];
  // A fragments of the geometry GEMM for element e: component r (x, y, z, d1, d2, d3) of node 4s + c
  auto load_av = [&](int64_t e, double (&av)[3]) {
    const int nd = (lane < 10 && e >= 0) ? __ldg(conn + (int64_t)lane * E + e) : 0;
#pragma unroll
    for (int s = 0; s < 3; s++) {
      const int k = 4 * s + c;
      const int node = __shfl_sync(0xffffffffu, nd, k < 10 ? k : 0);
      av[s] = 0.0;
      if (k < 10 && e >= 0) {
        if (r < 3) av[s] = __ldg(coords + (int64_t)r * N + node);
        else if (HAS_R && r < 6) av[s] = __ldg(state + (int64_t)(r - 3) * N + node);
      }
    }
  };
  const int64_t nw = (int64_t)gridDim.x * P2E_WARPS;
  int64_t pos = (int64_t)blockIdx.x * P2E_WARPS + warp;
  double av[3];
  load_av(pos < E ? (int64_t)__ldg(eperm + pos) : -1, av);
  for (; pos < E; pos += nw) {
    const int64_t e = __ldg(eperm + pos);
    const int64_t pn = pos + nw;
    double C2[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
#pragma unroll
    for (int s = 0; s < 3; s++)
#pragma unroll
      for (int t = 0; t < 2; t++) dmma884_t2(C2[t], av[s], L[32 * (s * 2 + t)]);
    load_av(pn < E ? (int64_t)__ldg(eperm + pn) : -1, av);  // prefetch: in flight while this element computes
    if (r < 6) {
#pragma unroll
      for (int t = 0; t < 2; t++)
#pragma unroll
        for (int i = 0; i < 2; i++) {
          const int n = 8 * t + 2 * c + i;
          if (n < 12) sc[r * 12 + n] = C2[t][i];
        }
    }
    __syncwarp();
    const int q = lane >> 3;
    double J[3][3], Dr[3][3];
#pragma unroll
    for (int i = 0; i < 3; i++)
#pragma unroll
      for (int j = 0; j < 3; j++) {
        J[i][j] = sc[i * 12 + 3 * q + j];
        if constexpr (HAS_R) Dr[i][j] = sc[(3 + i) * 12 + 3 * q + j];
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
    __syncwarp();
    if ((lane & 7) == 0) {
      const double rr = 1.0 / det;
      double Ji[3][3];
      Ji[0][0] = c00 * rr; Ji[1][0] = c01 * rr; Ji[2][0] = c02 * rr;
      Ji[0][1] = (J[0][2] * J[2][1] - J[0][1] * J[2][2]) * rr;
      Ji[1][1] = (J[0][0] * J[2][2] - J[0][2] * J[2][0]) * rr;
      Ji[2][1] = (J[0][1] * J[2][0] - J[0][0] * J[2][1]) * rr;
      Ji[0][2] = (J[0][1] * J[1][2] - J[0][2] * J[1][1]) * rr;
      Ji[1][2] = (J[0][2] * J[1][0] - J[0][0] * J[1][2]) * rr;
      Ji[2][2] = (J[0][0] * J[1][1] - J[0][1] * J[1][0]) * rr;
      double* o = sc + q * 20;
#pragma unroll
      for (int j = 0; j < 3; j++)
#pragma unroll
        for (int i = 0; i < 3; i++) o[j * 3 + i] = Ji[j][i];
      const double w = det * (1.0 / 24.0);
      o[9] = w;
      if constexpr (HAS_R) {
        double gu[3][3];
#pragma unroll
        for (int k = 0; k < 3; k++)
#pragma unroll
          for (int i = 0; i < 3; i++) gu[k][i] = Dr[k][0] * Ji[0][i] + Dr[k][1] * Ji[1][i] + Dr[k][2] * Ji[2][i];
        const double lw = H.sl * w * (gu[0][0] + gu[1][1] + gu[2][2]), mw = H.sm * w;
#pragma unroll
        for (int i = 0; i < 3; i++)
#pragma unroll
          for (int j = 0; j < 3; j++) o[10 + i * 3 + j] = (i == j ? lw : 0.0) + mw * (gu[i][j] + gu[j][i]);
      }
    }
    __syncwarp();
    const int a0 = r;
    const double* o = sc + c * 20;
    double G0[3], G1[3];
#pragma unroll
    for (int i = 0; i < 3; i++) {
      G0[i] = o[0 * 3 + i] * L[32 * 6] + o[1 * 3 + i] * L[32 * 7] + o[2 * 3 + i] * L[32 * 8];
      G1[i] = o[0 * 3 + i] * L[32 * 9] + o[1 * 3 + i] * L[32 * 10] + o[2 * 3 + i] * L[32 * 11];
    }
    const double w = o[9];
    if constexpr (HAS_R) {  // r_(a,i) = -Σ_γ w σ_ij G_aj over the 4 points (lanes c)
      double res0[3], res1[3];
#pragma unroll
      for (int i = 0; i < 3; i++) {
        double t0 = 0.0, t1 = 0.0;
#pragma unroll
        for (int j = 0; j < 3; j++) {
          t0 = fma(o[10 + i * 3 + j], G0[j], t0);
          t1 = fma(o[10 + i * 3 + j], G1[j], t1);
        }
        res0[i] = -sum4_t2(t0);
        res1[i] = -sum4_t2(t1);
      }
      double* eo = stage[warp] + 55 * 9;
      if (c == 0) {
#pragma unroll
        for (int i = 0; i < 3; i++) eo[a0 * 3 + i] = res0[i];
      }
      if (c == 1 && r < 2) {
#pragma unroll
        for (int i = 0; i < 3; i++) eo[(8 + r) * 3 + i] = res1[i];
      }
    }
    if constexpr (HAS_V) {
      double M[3][3][2];
      auto gram = [&](const double* A, const double* B) {
#pragma unroll
        for (int j = 0; j < 3; j++)
#pragma unroll
          for (int k = 0; k < 3; k++) {
            M[j][k][0] = 0.0;
            M[j][k][1] = 0.0;
            dmma884_t2(M[j][k], w * A[j], B[k]);
          }
      };
      double* eb = stage[warp];
      // tile 1: blocks (a0, 2c + t), upper ones only
      gram(G0, G0);
#pragma unroll
      for (int t = 0; t < 2; t++) {
        const int b = 2 * c + t;
        if (b >= a0) {
          const double tr = M[0][0][t] + M[1][1][t] + M[2][2][t];
          double* dst = eb + p2_ublk(a0, b) * 9;
#pragma unroll
          for (int i = 0; i < 3; i++)
#pragma unroll
            for (int m = 0; m < 3; m++) dst[i * 3 + m] = -(H.cl * M[i][m][t] + H.cm * M[m][i][t] + (i == m ? H.cm * tr : 0.0));
        }
      }
      // tile 2: block (a0, 8 + c) for c < 2 (always upper)
      gram(G0, G1);
      if (c < 2) {
        double Ms[3][3];
#pragma unroll
        for (int j = 0; j < 3; j++)
#pragma unroll
          for (int k = 0; k < 3; k++) Ms[j][k] = c ? M[j][k][1] : M[j][k][0];
        const double tr = Ms[0][0] + Ms[1][1] + Ms[2][2];
        double* dst = eb + p2_ublk(a0, 8 + c) * 9;
#pragma unroll
        for (int i = 0; i < 3; i++)
#pragma unroll
          for (int m = 0; m < 3; m++) dst[i * 3 + m] = -(H.cl * Ms[i][m] + H.cm * Ms[m][i] + (i == m ? H.cm * tr : 0.0));
      }
      // tile 3: blocks (8 + a0, 8 + c) for a0 <= c < 2
      gram(G1, G1);
      if (r < 2 && c < 2 && c >= r) {
        double Ms[3][3];
#pragma unroll
        for (int j = 0; j < 3; j++)
#pragma unroll
          for (int k = 0; k < 3; k++) Ms[j][k] = c ? M[j][k][1] : M[j][k][0];
        const double tr = Ms[0][0] + Ms[1][1] + Ms[2][2];
        double* dst = eb + p2_ublk(8 + r, 8 + c) * 9;
#pragma unroll
        for (int i = 0; i < 3; i++)
#pragma unroll
          for (int m = 0; m < 3; m++) dst[i * 3 + m] = -(H.cl * Ms[i][m] + H.cm * Ms[m][i] + (i == m ? H.cm * tr : 0.0));
      }
    }
    __syncwarp();
    if constexpr (HAS_V) {
      double* dst = ek + pos * (55 * 9);
      for (int k = lane; k < 55 * 9; k += 32) dst[k] = stage[warp][k];
    }
    if constexpr (HAS_R) {
      if (lane < 30) er[pos * 30 + lane] = stage[warp][55 * 9 + lane];
    }
    __syncwarp();  // the scratch and the stage are rewritten by the next element
  }
}

// P2 tets, 4-point rule, every domain term ELAST_DOMAIN: the stored-mode element pass (all domain terms).
int launch_p2_el(const fem_mesh_s* m, const fem_problem* prob, const double* state, const int32_t* eperm,
                 double* ek, double* er, cudaStream_t s, bool* handled) {
  *handled = false;
  if (m->etype != ET_TET || m->order != 2 || m->kh != 3 || m->physics != FEM_ELASTICITY || prob->quad_order != 2)
    return 0;
  P2Coef H = {0, 0, 0, 0};
  int n_dom = 0;
  for (int t = 0; t < prob->n_terms; t++) {
    const fem_term& T = prob->terms[t];
    if (T.region >= 0) continue;
    if (T.form != FEM_WF_ELAST_DOMAIN) return 0;
    const FormArgs Fa = make_form_args(prob, T);
    H.cl += Fa.f0 * Fa.lam; H.cm += Fa.f0 * Fa.mu; H.sl += Fa.lam; H.sm += Fa.mu;
    n_dom++;
  }
  if (!n_dom) return 0;
  *handled = true;
  if (m->E == 0) return 0;
  int dev = 0, sms = 148, per_sm = 1;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  auto go = [&](auto kern) -> int {
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 32 * P2E_WARPS, 0);
    const int64_t grid = std::min<int64_t>((m->E + P2E_WARPS - 1) / P2E_WARPS, (int64_t)sms * std::max(per_sm, 1));
    kern<<<(unsigned)grid, 32 * P2E_WARPS, 0, s>>>(m->coords, state, m->conn, m->N, m->E, eperm, H, ek, er, m->err);
    FEM_CUDA_TRY(cudaGetLastError());
    return 0;
  };
  if (ek && er) return go(k_p2_el<true, true>);
  if (ek) return go(k_p2_el<true, false>);
  return go(k_p2_el<false, true>);
}

}  // namespace fem
