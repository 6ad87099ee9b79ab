// tet1_ns.cu — the c4 hot path: SUPG/PSPG-stabilised Navier-Stokes (code P:1002-1022) on
// P1/P1 tetrahedra with the 4-point degree-2 rule, node-tile owner gather (tiled.cu records).
//
// P1 tets are affine: J, det J, ∇N_a and every operand gradient (∇u_k, ∇p, Rc = u_k,k) are constant
// over the element; only the values N_a(γ) = α or β (barycentric 4-point rule) and u(γ) vary, and
// Rm_i(γ) = ρ u_k(γ) u_i,k + p_,i is linear in u(γ) (u_i,kk = 0, reading L10).  A warp takes two
// element visits at once: lane (h, a, b) with h = lane>>4 computes the geometry of visit h and the
// 4x4 block of the pair (a, b) summed over the 4 points; the same lanes then take the residual rows
// (a, κ0).  Contributions go to the tile accumulator with plain read-modify-writes in record order under
// per-row turns (FEM_SCATTER_TILED: bit-identical run to run) or with shared-memory fp64 atomics
// (FEM_SCATTER_TILED_UNORDERED).  Boundary groups (inflow/outflow/fix) run as the coloured generic facet
// pass.  The element arithmetic (ns_compute) is shared with the stored-mode element pass k_ns_el.
#include <algorithm>
#include <cstdlib>
#include <string>

#include "stored.cuh"
#include "tiled.cuh"

namespace fem {

struct NsCoef {
  double rho, mu, tm, tc, f0;
};

// Per-visit data in the warp scratch (doubles): G[4][3] | gu[4][3] | Rc | w | u[4 points][4] | Rm[4][3] at
// 0..53, then the quadrature moments of the visit (offsets NSM_*): every point-dependent factor of the
// NS tangent and residual is linear in the point (affine P1: N_b(γ), u(γ), Rm(γ) = ρ u_k(γ) u_i,k
// + p_,i), so the 4-point sums of the 16 pair blocks collapse to contractions of these 49 moments with the
// constant gradients (the sums are hoisted out of the pair loop; the quadrature itself is kept,
// so the result is the oracle's 4-point sum, not the exact integral).
constexpr int NSM_U1 = 54;   // U1[b][i] = Σ_γ w N_b(γ) u_i(γ)          (4 x 3)
constexpr int NSM_R1 = 66;   // R1[b][i] = Σ_γ w N_b(γ) Rm_i(γ)         (4 x 3)
constexpr int NSM_UU = 78;   // UU[i][j] = Σ_γ w u_i(γ) u_j(γ)          (3 x 3)
constexpr int NSM_UR = 87;   // UR[j][i] = Σ_γ w u_j(γ) Rm_i(γ)         (3 x 3)
constexpr int NSM_U0 = 96;   // U0[i] = Σ_γ w u_i(γ)                      (3)
constexpr int NSM_R0 = 99;   // R0[i] = Σ_γ w Rm_i(γ)                     (3)
constexpr int NSM_P0 = 102;  // P0 = Σ_γ w p(γ)                           (1)
constexpr int NS_SC = 104;   // doubles per visit (even)

// The per-element arithmetic of a P1 NS visit, for the two elements of a warp (half-warp h = lane >> 4 takes
// one; called by all 32 lanes).  val(k, n): component k (x, y, z, u1, u2, u3, p) of node n of the half's
// element; sc: the half's NS_SC scratch doubles.  Returns false when some lane's element has det J <= 0
// (*bad set on that lane; acc/res untouched), else lane (a, b) = (l16 >> 2, l16 & 3) receives the 4x4
// block of the pair (a, b) summed over the points (without f0) and the residual entry of row (a, κ0 = b).
template <class Val>
__device__ __forceinline__ bool ns_compute(const NsCoef& c, double* sc, bool valid, Val&& val, bool* bad_out,
                                           double (&acc)[4][4], double& res) {
  const int lane = threadIdx.x & 31;
  const int l16 = lane & 15;
  const double al = 0.13819660112501051518, be = 0.58541019662496845446;  // (5-√5)/20, (5+3√5)/20
  // ---- phase 1: the 16 lanes of each half-warp compute the visit's constants (affine P1 tet): the
  // geometry redundantly (SIMT: same issue cost as one lane), the per-lane values split over the lanes
  bool bad = false;
  {
    double X[4][3];
#pragma unroll
    for (int n = 0; n < 4; n++)
#pragma unroll
      for (int d = 0; d < 3; d++) X[n][d] = val(d, n);
    double J[3][3];
#pragma unroll
    for (int i = 0; i < 3; i++)
#pragma unroll
      for (int j = 0; j < 3; j++) J[i][j] = X[j + 1][i] - X[0][i];
    const double c00 = J[1][1] * J[2][2] - J[1][2] * J[2][1];
    const double c01 = J[1][2] * J[2][0] - J[1][0] * J[2][2];
    const double c02 = J[1][0] * J[2][1] - J[1][1] * J[2][0];
    const double det = J[0][0] * c00 + J[0][1] * c01 + J[0][2] * c02;
    bad = valid && !(det > 0.0);
    const double rr = 1.0 / det;
    double Ji[3][3];
    Ji[0][0] = c00 * rr; Ji[1][0] = c01 * rr; Ji[2][0] = c02 * rr;
    Ji[0][1] = (J[0][2] * J[2][1] - J[0][1] * J[2][2]) * rr;
    Ji[1][1] = (J[0][0] * J[2][2] - J[0][2] * J[2][0]) * rr;
    Ji[2][1] = (J[0][1] * J[2][0] - J[0][0] * J[2][1]) * rr;
    Ji[0][2] = (J[0][1] * J[1][2] - J[0][2] * J[1][1]) * rr;
    Ji[1][2] = (J[0][2] * J[1][0] - J[0][0] * J[1][2]) * rr;
    Ji[2][2] = (J[0][0] * J[1][1] - J[0][1] * J[1][0]) * rr;
    double G[4][3];  // ∇N_0 = -(row sums of J^{-1}), ∇N_k = row k-1 of J^{-1}
#pragma unroll
    for (int i = 0; i < 3; i++) {
      G[1][i] = Ji[0][i];
      G[2][i] = Ji[1][i];
      G[3][i] = Ji[2][i];
      G[0][i] = -(Ji[0][i] + Ji[1][i] + Ji[2][i]);
    }
    // lane l16 < 12: G[n][i] and gu[k][i] = u_k,i = Σ_n U[k][n] G[n][i] for (k, i) = (l16 / 3, l16 % 3);
    // every lane: u_k(γ) for (γ, k) = (l16 / 4, l16 % 4)
    if (l16 < 12) {
      const int k = l16 / 3, i = l16 % 3;
      double g = 0.0;
#pragma unroll
      for (int n = 0; n < 4; n++) g = fma(val(3 + k, n), G[n][i], g);
      sc[12 + l16] = g;
      double gsel = G[0][0];
#pragma unroll
      for (int n = 0; n < 4; n++)
#pragma unroll
        for (int ii = 0; ii < 3; ii++)
          if (n * 3 + ii == l16) gsel = G[n][ii];
      sc[l16] = gsel;
    }
    {
      const int q = l16 >> 2, k = l16 & 3;
      double us = 0.0, uq = 0.0;
#pragma unroll
      for (int n = 0; n < 4; n++) {
        const double U = val(3 + k, n);
        us += U;
        if (n == q) uq = U;
      }
      sc[26 + q * 4 + k] = al * us + (be - al) * uq;
    }
    if (l16 == 0) sc[25] = det * (1.0 / 24.0);  // w (4-point rule weight 1/24)
    __syncwarp();
    if (l16 == 12) sc[24] = sc[12 + 0] + sc[12 + 4] + sc[12 + 8];  // Rc = u_k,k
    if (l16 < 12) {  // Rm_i(γ) = ρ u_k(γ) u_i,k + p_,i for (γ, i) = (l16 / 3, l16 % 3)
      const int q = l16 / 3, i = l16 % 3;
      const double* u = sc + 26 + q * 4;
      sc[42 + q * 3 + i] = sc[12 + 9 + i] + c.rho * (u[0] * sc[12 + i * 3 + 0] + u[1] * sc[12 + i * 3 + 1] + u[2] * sc[12 + i * 3 + 2]);
    }
    __syncwarp();
    // ---- phase 1b: the visit's quadrature moments (lanes of the half split them)
    {
      const double wq = sc[25];
      if (l16 < 12) {  // U1[b][i], R1[b][i] for (b, i) = (l16 / 3, l16 % 3)
        const int bb = l16 / 3, i = l16 % 3;
        double u1 = 0.0, r1 = 0.0;
#pragma unroll
        for (int q = 0; q < 4; q++) {
          const double wn = wq * (q == bb ? be : al);
          u1 = fma(wn, sc[26 + q * 4 + i], u1);
          r1 = fma(wn, sc[42 + q * 3 + i], r1);
        }
        sc[NSM_U1 + l16] = u1;
        sc[NSM_R1 + l16] = r1;
      }
      if (l16 < 9) {  // UU[i][j], UR[i][j] = Σ w u_i Rm_j for (i, j) = (l16 / 3, l16 % 3)
        const int i = l16 / 3, j = l16 % 3;
        double uu = 0.0, ur = 0.0;
#pragma unroll
        for (int q = 0; q < 4; q++) {
          uu = fma(wq * sc[26 + q * 4 + i], sc[26 + q * 4 + j], uu);
          ur = fma(wq * sc[26 + q * 4 + i], sc[42 + q * 3 + j], ur);
        }
        sc[NSM_UU + l16] = uu;
        sc[NSM_UR + l16] = ur;
      } else if (l16 < 12) {  // U0[i], R0[i]
        const int i = l16 - 9;
        double u0 = 0.0, r0 = 0.0;
#pragma unroll
        for (int q = 0; q < 4; q++) {
          u0 = fma(wq, sc[26 + q * 4 + i], u0);
          r0 = fma(wq, sc[42 + q * 3 + i], r0);
        }
        sc[NSM_U0 + i] = u0;
        sc[NSM_R0 + i] = r0;
      } else if (l16 == 12) {  // P0
        double p0 = 0.0;
#pragma unroll
        for (int q = 0; q < 4; q++) p0 = fma(wq, sc[26 + q * 4 + 3], p0);
        sc[NSM_P0] = p0;
      }
    }
  }
  *bad_out = bad;
  if (__any_sync(0xffffffffu, bad)) return false;
  __syncwarp();
  const double rho = c.rho, mu = c.mu, tm = c.tm, tc = c.tc;
  const int a = l16 >> 2, b = l16 & 3;
  double Ga[3], Gb[3];
#pragma unroll
  for (int i = 0; i < 3; i++) { Ga[i] = sc[a * 3 + i]; Gb[i] = sc[b * 3 + i]; }
  const double w = sc[25], Rc = sc[24];
  double GaGb = 0.0, smv[3];
#pragma unroll
  for (int k = 0; k < 3; k++) GaGb = fma(Ga[k], Gb[k], GaGb);
#pragma unroll
  for (int m = 0; m < 3; m++) smv[m] = Ga[0] * sc[12 + 0 * 3 + m] + Ga[1] * sc[12 + 1 * 3 + m] + Ga[2] * sc[12 + 2 * 3 + m];
  // ---- the 4x4 pair block and the residual row as contractions of the moments (phase 1b)
  const double W = 4.0 * w, Wq = w;  // Σ_γ w = |T|;  Σ_γ w N_b(γ) = w (β + 3α = 1)
  const double* U1b = sc + NSM_U1 + b * 3;
  const double* R1b = sc + NSM_R1 + b * 3;
  const double* UU = sc + NSM_UU;
  const double* UR = sc + NSM_UR;
  const double* U0 = sc + NSM_U0;
  double s1 = 0.0, s2 = 0.0, aU0 = 0.0, bU0 = 0.0;  // G_a·U1_b, G_a^T UU G_b, G_a·U0, U0·G_b
#pragma unroll
  for (int k = 0; k < 3; k++) {
    s1 = fma(Ga[k], U1b[k], s1);
    aU0 = fma(Ga[k], U0[k], aU0);
    bU0 = fma(Gb[k], U0[k], bU0);
    double t = 0.0;
#pragma unroll
    for (int j = 0; j < 3; j++) t = fma(UU[k * 3 + j], Gb[j], t);
    s2 = fma(Ga[k], t, s2);
  }
  const double diag = -rho * s1 + mu * W * GaGb + tm * rho * rho * s2;
#pragma unroll
  for (int i = 0; i < 3; i++) {
#pragma unroll
    for (int m = 0; m < 3; m++) {
      double t = Ga[m] * (tm * rho * R1b[i] - rho * U1b[i]) + tm * rho * rho * s1 * sc[12 + i * 3 + m] +
                 tc * W * Ga[i] * Gb[m];
      if (i == m) t += diag;
      acc[i][m] = t;
    }
    acc[i][3] = -Ga[i] * Wq + tm * rho * Gb[i] * aU0;
    acc[3][i] = Wq * Gb[i] + tm * rho * (Wq * smv[i] + Ga[i] * bU0);
  }
  acc[3][3] = tm * W * GaGb;
  if (b < 3) {  // residual row (a, u_b): BASE + SUPG of NS_domain
    const int i = b;
    res = -Ga[i] * sc[NSM_P0] + tc * W * Ga[i] * Rc;
#pragma unroll
    for (int j = 0; j < 3; j++)
      res += Ga[j] * (tm * rho * UR[j * 3 + i] + mu * W * sc[12 + i * 3 + j] - rho * UU[i * 3 + j]);
  } else {      // residual row (a, p)
    res = Wq * Rc + tm * (Ga[0] * sc[NSM_R0] + Ga[1] * sc[NSM_R0 + 1] + Ga[2] * sc[NSM_R0 + 2]);
  }
  return true;
}

template <bool DET>
__device__ __forceinline__ void ns_visit2(const TiledParams& P, const TileSmem& D, const NsCoef& c, int v0, int nv,
                                          double* scw, const uint8_t* vseq, int* turn) {
  const int lane = threadIdx.x & 31;
  const int h = lane >> 4, l16 = lane & 15;
  const int v = v0 + h;
  const bool valid = v < nv;
  const int vv = valid ? v : v0;
  double* sc = scw + h * NS_SC;
  double acc[4][4], res = 0.0;
  bool bad = false;
  const bool ok = ns_compute(c, sc, valid, [&](int k, int n) { return D.hdat[k * D.H + (uint16_t)D.vhal[vv * 4 + n]]; },
                             &bad, acc, res);
  if (!ok) {
    if (bad) atomicCAS((unsigned long long*)P.err, (unsigned long long)(-1LL), (unsigned long long)D.vid[v]);
    if constexpr (DET) {  // still pass the turns on, or later visits of these rows would wait forever
      const int a = l16 >> 2, li = D.vown[vv * 4 + a];
      if (valid && li >= 0 && (l16 & 3) == 0) {
        volatile int* tp = turn + li;
        const int t = vseq[vv * 4 + a];
        while (*tp != t) {
        }
        __threadfence_block();
        *tp = t + 1;
      }
    }
    __syncwarp();
    return;
  }
  const int a = l16 >> 2, b = l16 & 3;
  const int li = D.vown[vv * 4 + a];
  if constexpr (DET) {
    // ordered: visit v takes its turn (vseq) on the accumulator row of each owned node, so every entry
    // sums its contributions in record order with plain read-modify-writes (bit-identical run to run).
    // Visits are grabbed in increasing order, so an awaited turn belongs to a running visit (possibly
    // the other half of this warp, which independent thread scheduling lets finish).
    const unsigned half = 0xffffu << (16 * h);
    int my_turn = 0;
    if (valid && li >= 0) {
      my_turn = vseq[vv * 4 + a];
      while (*reinterpret_cast<volatile int*>(turn + li) != my_turn) __nanosleep(32);  // (frees issue slots)
      __threadfence_block();
      if (P.values) {
        const int d = D.tdeg[li], sr = acc_row_stride(4, d, P.nnz_s);
        double* rowb = D.acc + D.toff[li] + D.vloc[vv * 16 + a * 4 + b];
#pragma unroll
        for (int i = 0; i < 4; i++) {
          double old[4];
#pragma unroll
          for (int m = 0; m < 4; m++) old[m] = rowb[i * sr + m * d];
#pragma unroll
          for (int m = 0; m < 4; m++) rowb[i * sr + m * d] = fma(c.f0, acc[i][m], old[m]);
        }
      }
      if (P.rhs) D.racc[b * D.T + li] += res;
    }
    __syncwarp(half);  // the row's four lanes have written
    __threadfence_block();
    if (valid && li >= 0 && b == 0) *reinterpret_cast<volatile int*>(turn + li) = my_turn + 1;
  } else if (valid && li >= 0) {
    if (P.values) {
      const int d = D.tdeg[li], sr = acc_row_stride(4, d, P.nnz_s);
      double* rowb = D.acc + D.toff[li] + D.vloc[vv * 16 + a * 4 + b];
#pragma unroll
      for (int i = 0; i < 4; i++)
#pragma unroll
        for (int m = 0; m < 4; m++) atomicAdd(rowb + i * sr + m * d, c.f0 * acc[i][m]);
    }
    if (P.rhs) atomicAdd(D.racc + b * D.T + li, res);
  }
  __syncwarp();  // scratch reused by the next pair of visits
}

template <bool DET>
__global__ void __launch_bounds__(TILED_THREADS, 1) k_ns_rec(const __grid_constant__ TiledParams P) {
  using C = TileCfg<ET_TET, 1, 4, 2>;
  constexpr int NL = 4, DIM = 3;
  extern __shared__ __align__(16) unsigned char smem[];
  uint64_t* mbar = reinterpret_cast<uint64_t*>(smem);
  int* ctr = reinterpret_cast<int*>(smem + 64);
  unsigned char* rbuf[2] = {smem + 128, smem + 128 + P.rec_cap};
  double* hbuf = reinterpret_cast<double*>(smem + 128 + 2 * (size_t)P.rec_cap);
  double* acc = hbuf + P.hcap;
  TileSmem S;
  int* turn = reinterpret_cast<int*>(acc + P.acc_cap);
  unsigned char* fp = reinterpret_cast<unsigned char*>(turn + P.turn_cap);
  S.qp = fp;
  fp += std::max((size_t)P.rec_bytes * 8, (size_t)8 * 2 * NS_SC * C::WARPS);
  S.vid = reinterpret_cast<int32_t*>(fp);
  fp += 4 * (size_t)P.fvmax;
  S.vnode = reinterpret_cast<int32_t*>(fp);
  fp += 4 * (size_t)P.fvmax * NL;
  S.vown = reinterpret_cast<int16_t*>(fp);
  fp += 2 * (size_t)P.fvmax * NL;
  S.vfac = reinterpret_cast<int8_t*>(fp);
  S.vhal = nullptr;
  S.hnode = nullptr;
  S.hdat = nullptr;
  S.H = 0;
  NsCoef cf;
  cf.rho = P.dom[0].p[0]; cf.mu = P.dom[0].p[1]; cf.tm = P.dom[0].p[2]; cf.tc = P.dom[0].p[3]; cf.f0 = P.dom[0].f0;
  const int tid = threadIdx.x, warp = tid >> 5;
  unsigned char* slot = S.qp + (size_t)P.rec_bytes * (warp % 8);
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
    bulk_g2s(rbuf[0], P.rec + P.rec_off[tile], bytes, &mbar[0]);
  }
  for (int it = 0; tile < P.n_tiles; it++, tile += gridDim.x) {
    const int cur = it & 1, oth = cur ^ 1;
    const int64_t next = tile + gridDim.x;
    mbar_wait(&mbar[cur], (uint32_t)((it >> 1) & 1));
    if (tid == 0 && next < P.n_tiles) {
      const uint32_t bytes = (uint32_t)(P.rec_off[next + 1] - P.rec_off[next]);
      mbar_expect_tx(&mbar[oth], bytes);
      bulk_g2s(rbuf[oth], P.rec + P.rec_off[next], bytes, &mbar[oth]);
    }
    const uint8_t* rec = rbuf[cur];
    {  // stage the tile's halo points
      const int32_t* hdr = reinterpret_cast<const int32_t*>(rec);
      const RecLayout L = rec_layout_hdr(NL, hdr);
      const int32_t* hn = reinterpret_cast<const int32_t*>(rec + L.o_hnode);
      const int H = hdr[1];
      for (int cc = 0; cc < P.hcomp; cc++) {  // component-major: no integer division per element
        const double* base = cc < DIM ? P.coords + (int64_t)cc * P.N : P.state + (int64_t)(cc - DIM) * P.N;
        for (int i = tid; i < H; i += blockDim.x) cp_async8(hbuf + cc * H + i, base + hn[i]);
      }
      cp_async_commit();
    }
    const int32_t* hdr = reinterpret_cast<const int32_t*>(rec);
    const int T = hdr[0], H = hdr[1], nv = hdr[2], acc_n = P.values ? hdr[4] : 0;
    const uint32_t fmask = (uint32_t)hdr[5];
    const RecLayout L = rec_layout_hdr(NL, hdr);
    TileSmem D = S;
    D.tnode = const_cast<int32_t*>(reinterpret_cast<const int32_t*>(rec + L.o_tnode));
    D.tdeg = const_cast<int32_t*>(reinterpret_cast<const int32_t*>(rec + L.o_tdeg));
    D.toff = const_cast<int32_t*>(reinterpret_cast<const int32_t*>(rec + L.o_toff));
    D.trps = const_cast<int64_t*>(reinterpret_cast<const int64_t*>(rec + L.o_trps));
    D.vid = const_cast<int32_t*>(reinterpret_cast<const int32_t*>(rec + L.o_velem));
    D.vown = const_cast<int16_t*>(reinterpret_cast<const int16_t*>(rec + L.o_vown));
    D.vhal = const_cast<int16_t*>(reinterpret_cast<const int16_t*>(rec + L.o_vhal));
    D.vloc = rec + L.o_vloc;
    D.hdat = hbuf;
    D.H = H;
    D.acc = acc;
    D.racc = acc + acc_n;
    D.T = T;
    for (int i = tid; i < acc_n + 4 * T; i += blockDim.x) acc[i] = 0.0;
    if constexpr (DET)
      for (int i = tid; i < T; i += blockDim.x) turn[i] = 0;
    if (tid == 0) *ctr = 0;
    cp_async_wait_all();
    __syncthreads();
    double* scw = reinterpret_cast<double*>(S.qp) + (size_t)2 * NS_SC * warp;
    const uint8_t* vseq = rec + L.o_vseq;
    for (int v0 = grab_visits(ctr, 2); v0 < nv; v0 = grab_visits(ctr, 2)) ns_visit2<DET>(P, D, cf, v0, nv, scw, vseq, turn);
    if (fmask) rec_facets<ET_TET, 1, 4, 2, 8, DET>(P, D, rec, L, slot);
    tile_epilogue<4>(P, D);
    __syncthreads();
  }
}

// NS on P1 tets, 4-point rule, exactly one domain term NS_DOMAIN.
int launch_ns_tiled(TiledParams& P, const TileSchedule& T, bool det, cudaStream_t s, bool* handled) {
  *handled = false;
  if (P.n_dom != 1 || P.dom[0].form != FEM_WF_NS_DOMAIN || !T.rec) return 0;
  *handled = true;
  if (det && T.max_turns > 255) {
    set_error("tiled scatter: a tile point is touched by more than 255 element visits (8-bit turns); use "
              "FEM_SCATTER_COLOURED or FEM_SCATTER_TILED_UNORDERED");
    return FEM_E_UNSUPPORTED;
  }
  using C = TileCfg<ET_TET, 1, 4, 2>;
  constexpr int NL = 4;
  P.rec_bytes = (int)((sizeof(typename C::QPG) * C::NQF + 15) / 16 * 16);
  int fv = 1;
  for (int f = 0; f < P.n_fac; f++) fv = std::max<int>(fv, (int)P.fvis[f].max_per_tile);
  P.fvmax = fv;
  P.vmax = fv;
  P.hmax = 0;
  P.hcomp = 3 + 4;
  P.rec = T.rec;
  P.rec_off = T.rec_off;
  P.n_tiles = T.n_tiles;
  P.rec_cap = (int)((T.rec_max + 15) / 16 * 16);
  P.hcap = (int)(((T.max_halo * P.hcomp) + 1) / 2 * 2);
  P.acc_cap = (int)((P.values ? T.acc_max : 0) + (int64_t)4 * T.max_tile_nodes);
  P.acc_cap = (P.acc_cap + 1) / 2 * 2;
  P.turn_cap = (int)((T.max_tile_nodes + 3) / 4 * 4);
  const size_t fac_bytes = std::max((size_t)P.rec_bytes * 8, (size_t)8 * 2 * NS_SC * C::WARPS) + (size_t)fv * (4 + NL * 6 + 1) + 16;
  const size_t smem = 128 + 2 * (size_t)P.rec_cap + 8 * (size_t)P.hcap + 8 * (size_t)P.acc_cap + 4 * (size_t)P.turn_cap + fac_bytes;
  if (smem > 227 * 1024) {
    set_error("NS record kernel: shared memory request too large (" + std::to_string(smem) + " B)");
    return FEM_E_UNSUPPORTED;
  }
  if (det) FEM_CUDA_TRY(cudaFuncSetAttribute(k_ns_rec<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  else FEM_CUDA_TRY(cudaFuncSetAttribute(k_ns_rec<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  if (T.n_tiles <= 0) return 0;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t grid = std::min<int64_t>(T.n_tiles, sms);
  if (det) k_ns_rec<true><<<(unsigned)grid, TILED_THREADS, smem, s>>>(P);
  else k_ns_rec<false><<<(unsigned)grid, TILED_THREADS, smem, s>>>(P);
  FEM_CUDA_TRY(cudaGetLastError());
  return 0;
}


// ---- FEM_SCATTER_STORED element pass (stored.cu): the visit arithmetic of ns_compute for one element per
// half-warp, its points gathered from node-major copies (coordinates x y z 0 and state u1 u2 u3 p, 32 bytes
// per point: one 256-bit load each) into the half's scratch; lane (a, b) stores the 4x4 block
// (a, b) — f0·K, 16 doubles, four 256-bit stores — at ek[pos][a·4 + b] (all 16 blocks: NS is not symmetric)
// and the residual entry (a, κ0 = b) at er[pos][a][b]; the element's 16 lanes write 2 KB contiguously.
constexpr int NSE_WARPS = 8;
// dst[i][c] = src[c][i] for c < ncomp, dst[i][c] = 0 for ncomp <= c < 4 (component-major -> node-major, 32 B/node)
__global__ void k_aos4(const double* __restrict__ src, double* __restrict__ dst, int64_t n, int ncomp) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < 4 * n; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = t >> 2;
    const int c = (int)(t & 3);
    dst[t] = c < ncomp ? __ldg(src + (int64_t)c * n + i) : 0.0;
  }
}
static int aos4(const double* src, double* dst, int64_t n, int ncomp, cudaStream_t s) {
  if (n <= 0) return 0;
  const int64_t blocks = std::min<int64_t>((4 * n + 255) / 256, 148 * 64);
  k_aos4<<<(unsigned)blocks, 256, 0, s>>>(src, dst, n, ncomp);
  FEM_CUDA_TRY(cudaGetLastError());
  return 0;
}
template <bool HAS_V, bool HAS_R>
__global__ void __launch_bounds__(32 * NSE_WARPS) k_ns_el(const double* __restrict__ xaos, const double* __restrict__ saos,
                                                         const int32_t* __restrict__ conn, int64_t N, int64_t E,
                                                         const int32_t* __restrict__ eperm, NsCoef cf,
                                                         double* __restrict__ ek, double* __restrict__ er, long long* err) {
  __shared__ double scr[NSE_WARPS][2][NS_SC];
  __shared__ double nd[NSE_WARPS][2][7 * 4];  // component-major point data of the half's element
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, h = lane >> 4, l16 = lane & 15;
  const int64_t n_half = (int64_t)gridDim.x * NSE_WARPS * 2;
  const int64_t first = ((int64_t)blockIdx.x * NSE_WARPS + warp) * 2 + h;
  double* sc = scr[warp][h];
  double* x = nd[warp][h];
  // the warp loops while either half has an element (ns_compute is warp-collective)
  for (int64_t base = first - h; base < E; base += n_half) {
    const int64_t pos = base + h;
    const bool valid = pos < E;
    const int64_t e = valid ? __ldg(eperm + pos) : 0;
    int node = 0;
    if (l16 < 4) node = valid ? __ldg(conn + (int64_t)l16 * E + e) : 0;
    {  // the element's 4 points, node-major copies: lane (w, n) < 8 loads 32 bytes (x y z - or u1 u2 u3 p)
      const int n = l16 & 3, wh = (l16 >> 2) & 1;
      const int nn = __shfl_sync(0xffffffffu, node, (lane & 16) | n);
      if (l16 < 8) {
        double v[4];
        if (valid) {
          st_ld4((wh ? saos : xaos) + (int64_t)nn * 4, v[0], v[1], v[2], v[3]);
        } else {  // (unit tet: det > 0)
#pragma unroll
          for (int i = 0; i < 4; i++) v[i] = wh ? 0.0 : (double)(n == i + 1);
        }
#pragma unroll
        for (int i = 0; i < 4; i++)
          if (wh || i < 3) x[(3 * wh + i) * 4 + n] = v[i];
      }
    }
    __syncwarp();
    double acc[4][4], res = 0.0;
    bool bad = false;
    const bool ok = ns_compute(cf, sc, valid, [&](int k, int n) { return x[k * 4 + n]; }, &bad, acc, res);
    if (!ok) {
      if (bad) atomicCAS((unsigned long long*)err, (unsigned long long)(-1LL), (unsigned long long)e);
      __syncwarp();
      continue;
    }
    if (valid) {
      if constexpr (HAS_V) {
        double* dst = ek + (pos * 16 + l16) * 16;
#pragma unroll
        for (int i = 0; i < 4; i++)
          st_st4(dst + 4 * i, cf.f0 * acc[i][0], cf.f0 * acc[i][1], cf.f0 * acc[i][2], cf.f0 * acc[i][3]);
      }
      if constexpr (HAS_R) er[pos * 16 + l16] = res;
    }
    __syncwarp();  // the scratch is rewritten by the next element
  }
}

// NS on P1 tets, 4-point rule, exactly one domain term NS_DOMAIN: the stored-mode element pass.
int launch_ns_el(const fem_mesh_s* m, const fem_problem* prob, const double* state, const int32_t* eperm,
                 double* ek, double* er, double* xaos, double* saos, cudaStream_t s, bool* handled) {
  *handled = false;
  if (m->etype != ET_TET || m->order != 1 || m->kh != 4 || m->physics != FEM_NS || prob->quad_order != 2) return 0;
  int n_dom = 0, t_dom = -1;
  for (int t = 0; t < prob->n_terms; t++)
    if (prob->terms[t].region < 0) { n_dom++; t_dom = t; }
  if (n_dom != 1 || prob->terms[t_dom].form != FEM_WF_NS_DOMAIN) return 0;
  *handled = true;
  if (m->E == 0) return 0;
  {  // node-major copies: coordinates once (padded to 4), the state per call
    const int rc = aos4(m->coords, xaos, m->N, 3, s);
    if (rc) return rc;
    const int rc2 = aos4(state, saos, m->N, 4, s);
    if (rc2) return rc2;
  }
  const FormArgs F = make_form_args(prob, prob->terms[t_dom]);
  NsCoef cf;
  cf.rho = F.p[0]; cf.mu = F.p[1]; cf.tm = F.p[2]; cf.tc = F.p[3]; cf.f0 = F.f0;
  int dev = 0, sms = 148, per_sm = 1;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  auto go = [&](auto kern) -> int {
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 32 * NSE_WARPS, 0);
    const int64_t grid = std::min<int64_t>((m->E + 2 * NSE_WARPS - 1) / (2 * NSE_WARPS), (int64_t)sms * std::max(per_sm, 1));
    kern<<<(unsigned)grid, 32 * NSE_WARPS, 0, s>>>(xaos, saos, m->conn, m->N, m->E, eperm, cf, ek, er, m->err);
    FEM_CUDA_TRY(cudaGetLastError());
    return 0;
  };
  if (ek && er) return go(k_ns_el<true, true>);
  if (ek) return go(k_ns_el<true, false>);
  return go(k_ns_el<false, true>);
}

}  // namespace fem
