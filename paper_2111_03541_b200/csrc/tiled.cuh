// tiled.cuh — shared pieces of the node-tile owner-gather kernels (tiled.cu, hex_tiled.cu).
#pragma once
#include <cstdint>

#include "blocks.cuh"
#include "elements.cuh"
#include "fem_internal.cuh"

namespace fem {

constexpr int TILE_MAX_NODES = 512;
constexpr int MAX_DOM_TERMS = 4;
constexpr int MAX_FAC_TERMS = 8;
constexpr int TILED_THREADS = 512;

// ------------------------------------------------------------------ device: the tiled kernel
struct TiledParams {
  int n_dom, n_fac, lean;
  FormArgs dom[MAX_DOM_TERMS];
  FormArgs fac[MAX_FAC_TERMS];
  VisitList dvis;
  VisitList fvis[MAX_FAC_TERMS];
  const int64_t* tile_noff;
  const int32_t* tile_node;
  int64_t N, E, own_lo, n_own, nnz_s;
  const double* coords;
  const int32_t* conn;
  const double* state;
  const int64_t* rowptr_s;
  const uint8_t* loc;
  double* values;
  double* rhs;
  long long* err;
  int nu_hat;
  int fac_set[MAX_FAC_TERMS];  // boundary set of each facet term
  int vmax;      // capacity of the per-tile visit arrays
  int rec_bytes; // bytes of one warp's point-record slot
  const int64_t* halo_off;  // per tile: sorted points of the visited elements
  const int32_t* halo_node;
  int hmax;      // capacity of the halo arrays (0: halo staging off)
  int hcomp;     // doubles per halo point: dim coords + κ̂·(ν̂+1) state values
  // record-driven (persistent) kernels
  const uint8_t* rec;
  const int64_t* rec_off;
  int64_t n_tiles;
  int rec_cap;   // bytes of one record buffer
  int hcap;      // doubles of one halo buffer
  int acc_cap;   // doubles of the accumulator (incl. residual rows)
  int turn_cap;  // ints of the per-row turn counters (ordered deterministic kernels), multiple of 4
  int spin_ns;   // back-off of a visit waiting for its turn (FEM_SPIN_NS, default 0 = spin)
  int fvmax;     // capacity of the facet visit arrays
  int fac_inline;  // hex elasticity: boundary terms integrated inside the owning element's visit
  const int64_t* seq_off;  // sweep schedules: record sequences (see TileSchedule)
  int64_t n_seq;
};

// Lean point record for elasticity-only domain visits: w, ∇N_a, and w·σ.
template <int DIM, int NL>
struct QPE {
  double w;
  double G[NL][DIM];
  double S[DIM][DIM];
};

template <int ET, int ORD, int KH, int Q>
struct TileCfg {
  using EL = Elem<ET, ORD>;
  static constexpr int DIM = EL::DIM, NL = EL::NL;
  static constexpr int NQV = EL::vol_nq(Q), NQF = EL::fac_nq(Q);
  using QPG = QPX<DIM, NL, KH>;
  using QPL = QPE<DIM, NL>;
  static constexpr size_t HEAD_BYTES = 20 * TILE_MAX_NODES + 16;
  static constexpr int WARPS = TILED_THREADS / 32;
};

// lanes per quadrature point in the cooperative geometry: largest power of two with NQ*NSUB <= 32
template <int NQ>
struct Sub {
  static constexpr int v = NQ >= 32 ? 1 : (NQ * 32 <= 32 ? 32 : (NQ * 16 <= 32 ? 16 : (NQ * 8 <= 32 ? 8 :
                           (NQ * 4 <= 32 ? 4 : (NQ * 2 <= 32 ? 2 : 1)))));
};

__device__ __forceinline__ int find_local(const int32_t* __restrict__ tnode, int T, int node) {
  int lo = 0, hi = T - 1;
  while (lo <= hi) {
    const int mid = (lo + hi) >> 1;
    const int v = tnode[mid];
    if (v == node) return mid;
    if (v < node) lo = mid + 1;
    else hi = mid - 1;
  }
  return -1;
}

template <int NSUB>
__device__ __forceinline__ double group_sum(double v) {
#pragma unroll
  for (int o = 1; o < NSUB; o <<= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

struct TileSmem {
  int32_t* tnode; int64_t* trps; int32_t* tdeg; int32_t* toff;
  int32_t* vid;    // [vmax] element id of each visit
  int8_t* vfac;    // [vmax] facet id
  int32_t* vnode;  // [vmax*NL]
  int16_t* vown;   // [vmax*NL] tile-local point index or -1
  unsigned char* qp;  // per-warp point-record slots
  int16_t* vhal;   // [vmax*NL] halo index of each visit point
  const uint8_t* vloc = nullptr;  // [vmax][NL][NL] local column offsets in shared memory (records)
  int32_t* hnode;  // [hmax]
  double* hdat;    // [hcomp][hmax] staged coordinates and state of the halo points
  int H;
  double* acc;
  double* racc;
  int T;
};

// One warp assembles one element (or facet) visit into the tile accumulator.
template <int ET, int ORD, int KH, int Q, bool FACET, bool LEAN>
__device__ __forceinline__ void warp_visit(const TiledParams& P, const FormArgs* forms, int nforms, const TileSmem& S,
                                           int v, unsigned char* slot, int fac_override = -1) {
  using C = TileCfg<ET, ORD, KH, Q>;
  using EL = typename C::EL;
  constexpr int DIM = C::DIM, NL = C::NL;
  constexpr int NQ = FACET ? C::NQF : C::NQV;
  constexpr int NSUB = Sub<NQ>::v;
  using QPG = typename C::QPG;
  using QPL = typename C::QPL;
  const int lane = threadIdx.x & 31;
  const int32_t* nd = S.vnode + v * NL;
  const int16_t* own = S.vown + v * NL;
  // ---- cooperative geometry: lane -> (point g, node group sub)
  const int g = lane / NSUB, sub = lane % NSUB;
  const bool gl = g < NQ;
  const int gq = gl ? g : 0;
  double xi[3] = {0, 0, 0}, wref, mref[3] = {0, 0, 0};
  if constexpr (FACET) EL::fac_qp(Q, fac_override >= 0 ? fac_override : S.vfac[v], gq, xi, wref, mref);
  else EL::vol_qp(Q, gq, xi, wref);
  double N[NL], dN[NL][DIM];
  EL::shape(xi, N, dN);
  double J[DIM][DIM], xp[DIM];
#pragma unroll
  for (int i = 0; i < DIM; i++) {
    xp[i] = 0.0;
#pragma unroll
    for (int j = 0; j < DIM; j++) J[i][j] = 0.0;
  }
#pragma unroll
  for (int a = 0; a < NL; a++)
    if (a % NSUB == sub) {
      double X[DIM];
#pragma unroll
      for (int d = 0; d < DIM; d++)
        X[d] = S.hdat ? S.hdat[d * S.H + (uint16_t)S.vhal[v * NL + a]] : __ldg(P.coords + (int64_t)d * P.N + nd[a]);
#pragma unroll
      for (int i = 0; i < DIM; i++) {
        xp[i] = fma(N[a], X[i], xp[i]);
#pragma unroll
        for (int j = 0; j < DIM; j++) J[i][j] = fma(X[i], dN[a][j], J[i][j]);
      }
    }
#pragma unroll
  for (int i = 0; i < DIM; i++) {
    xp[i] = group_sum<NSUB>(xp[i]);
#pragma unroll
    for (int j = 0; j < DIM; j++) J[i][j] = group_sum<NSUB>(J[i][j]);
  }
  double Ji[DIM][DIM], det;
  if constexpr (DIM == 2) {
    det = J[0][0] * J[1][1] - J[0][1] * J[1][0];
    const double rr = 1.0 / det;
    Ji[0][0] = J[1][1] * rr;  Ji[0][1] = -J[0][1] * rr;
    Ji[1][0] = -J[1][0] * rr; Ji[1][1] = J[0][0] * rr;
  } else {
    const double c00 = J[1][1] * J[2][2] - J[1][2] * J[2][1];
    const double c01 = J[1][2] * J[2][0] - J[1][0] * J[2][2];
    const double c02 = J[1][0] * J[2][1] - J[1][1] * J[2][0];
    det = J[0][0] * c00 + J[0][1] * c01 + J[0][2] * c02;
    const double rr = 1.0 / det;
    Ji[0][0] = c00 * rr; Ji[1][0] = c01 * rr; Ji[2][0] = c02 * rr;
    Ji[0][1] = (J[0][2] * J[2][1] - J[0][1] * J[2][2]) * rr;
    Ji[1][1] = (J[0][0] * J[2][2] - J[0][2] * J[2][0]) * rr;
    Ji[2][1] = (J[0][1] * J[2][0] - J[0][0] * J[2][1]) * rr;
    Ji[0][2] = (J[0][1] * J[1][2] - J[0][2] * J[1][1]) * rr;
    Ji[1][2] = (J[0][2] * J[1][0] - J[0][0] * J[1][2]) * rr;
    Ji[2][2] = (J[0][0] * J[1][1] - J[0][1] * J[1][0]) * rr;
  }
  const bool bad = __any_sync(0xffffffffu, gl && !(det > 0.0));
  if (bad) {
    if (lane == 0) atomicCAS((unsigned long long*)P.err, (unsigned long long)(-1LL), (unsigned long long)S.vid[v]);
    return;
  }
  double w, nrm[DIM];
  if constexpr (FACET) {  // Nanson: n dA = det(J) J^{-T} m̂ dÂ
    double nn = 0.0;
#pragma unroll
    for (int i = 0; i < DIM; i++) {
      double sacc = 0.0;
#pragma unroll
      for (int j = 0; j < DIM; j++) sacc = fma(Ji[j][i], mref[j], sacc);
      nrm[i] = det * sacc;
      nn = fma(nrm[i], nrm[i], nn);
    }
    const double dA = sqrt(nn);
#pragma unroll
    for (int i = 0; i < DIM; i++) nrm[i] /= dA;
    w = wref * dA;
  } else {
#pragma unroll
    for (int i = 0; i < DIM; i++) nrm[i] = 0.0;
    w = wref * det;
  }
  // gradients of this lane's nodes and partial operand fields
  double u0[KH], u1[KH], gu[KH][DIM];
#pragma unroll
  for (int k = 0; k < KH; k++) {
    u0[k] = 0.0;
    u1[k] = 0.0;
#pragma unroll
    for (int d = 0; d < DIM; d++) gu[k][d] = 0.0;
  }
  QPL* ql = reinterpret_cast<QPL*>(slot);
  QPG* qg = reinterpret_cast<QPG*>(slot);
#pragma unroll
  for (int a = 0; a < NL; a++)
    if (a % NSUB == sub) {
      double Ga[DIM];
#pragma unroll
      for (int i = 0; i < DIM; i++) {
        double sacc = 0.0;
#pragma unroll
        for (int j = 0; j < DIM; j++) sacc = fma(Ji[j][i], dN[a][j], sacc);
        Ga[i] = sacc;
      }
      if (gl) {
        if constexpr (LEAN) {
#pragma unroll
          for (int i = 0; i < DIM; i++) ql[gq].G[a][i] = Ga[i];
        } else {
          qg[gq].N[a] = N[a];
#pragma unroll
          for (int i = 0; i < DIM; i++) qg[gq].G[a][i] = Ga[i];
        }
      }
#pragma unroll
      for (int k = 0; k < KH; k++) {
        const int hi = S.hdat ? (uint16_t)S.vhal[v * NL + a] : 0;
        const double s0 = S.hdat ? S.hdat[(DIM + k) * S.H + hi] : __ldg(P.state + (int64_t)k * P.N + nd[a]);
        u0[k] = fma(N[a], s0, u0[k]);
        if (!LEAN && P.nu_hat >= 1)
          u1[k] = fma(N[a], S.hdat ? S.hdat[(DIM + KH + k) * S.H + hi] : __ldg(P.state + ((int64_t)KH + k) * P.N + nd[a]),
                      u1[k]);
#pragma unroll
        for (int d = 0; d < DIM; d++) gu[k][d] = fma(Ga[d], s0, gu[k][d]);
      }
    }
#pragma unroll
  for (int k = 0; k < KH; k++) {
    u0[k] = group_sum<NSUB>(u0[k]);
    if (!LEAN) u1[k] = group_sum<NSUB>(u1[k]);
#pragma unroll
    for (int d = 0; d < DIM; d++) gu[k][d] = group_sum<NSUB>(gu[k][d]);
  }
  if (gl && sub == 0) {
    if constexpr (LEAN) {
      ql[gq].w = w;
      double div = 0.0;
#pragma unroll
      for (int k = 0; k < DIM; k++) div += gu[k % KH][k];
      const double lw = forms[0].lam * w * div, mw = forms[0].mu * w;
#pragma unroll
      for (int i = 0; i < DIM; i++)
#pragma unroll
        for (int j = 0; j < DIM; j++) ql[gq].S[i][j] = (i == j ? lw : 0.0) + mw * (gu[i % KH][j] + gu[j % KH][i]);
    } else {
      QPG& q = qg[gq];
      q.w = w;
#pragma unroll
      for (int d = 0; d < DIM; d++) { q.x[d] = xp[d]; q.n[d] = nrm[d]; }
#pragma unroll
      for (int k = 0; k < KH; k++) {
        q.u[0][k] = u0[k];
        q.u[1][k] = u1[k];
#pragma unroll
        for (int d = 0; d < DIM; d++) q.gu[k][d] = gu[k][d];
      }
      if constexpr (KH == DIM + 1) {  // NS strong residuals at the point
        const double rho = forms[0].p[0];
        double rc = 0.0;
#pragma unroll
        for (int k = 0; k < DIM; k++) rc += gu[k][k];
        q.ext[DIM] = rc;
#pragma unroll
        for (int i = 0; i < DIM; i++) {
          double rm = gu[DIM][i];
#pragma unroll
          for (int k = 0; k < DIM; k++) rm = fma(rho * u0[k], gu[i][k], rm);
          q.ext[i] = rm;
        }
      }
      if constexpr (KH == DIM) {
        if (!FACET && forms[0].form == FEM_WF_ELAST_DOMAIN) {
          double div = 0.0;
#pragma unroll
          for (int k = 0; k < DIM; k++) div += gu[k][k];
          const double lw = forms[0].lam * w * div, mw = forms[0].mu * w;
#pragma unroll
          for (int i = 0; i < DIM; i++)
#pragma unroll
            for (int j = 0; j < DIM; j++) q.ext[i * DIM + j] = (i == j ? lw : 0.0) + mw * (gu[i][j] + gu[j][i]);
        }
      }
    }
  }
  __syncwarp();
  // ---- owned test nodes of this visit
  int owned_a[NL], n_owned = 0;
#pragma unroll
  for (int a = 0; a < NL; a++)
    if (own[a] >= 0) owned_a[n_owned++] = a;
  const int npair = P.values ? n_owned * NL : 0;
  const int nres = P.rhs ? n_owned : 0;
  const int e = S.vid[v];
  for (int t = lane; t < npair + nres; t += 32) {
    const bool is_mat = t < npair;
    const int ia = is_mat ? t / NL : t - npair;
    int a = 0;
#pragma unroll
    for (int k = 0; k < NL; k++)
      if (k == ia) a = owned_a[k];
    const int li = own[a];
    if (is_mat) {
      const int b = t % NL;
      const int pos = S.vloc ? (int)S.vloc[v * (NL * NL) + a * NL + b] : (int)__ldg(P.loc + (int64_t)e * (NL * NL) + a * NL + b);
      double K[KH][KH];
#pragma unroll
      for (int i = 0; i < KH; i++)
#pragma unroll
        for (int m = 0; m < KH; m++) K[i][m] = 0.0;
      if constexpr (LEAN) {
        double M[DIM][DIM];
#pragma unroll
        for (int j = 0; j < DIM; j++)
#pragma unroll
          for (int k = 0; k < DIM; k++) M[j][k] = 0.0;
#pragma unroll
        for (int gg = 0; gg < NQ; gg++) {
          double wa[DIM], gb[DIM];
          const double wq = ql[gg].w;
#pragma unroll
          for (int j = 0; j < DIM; j++) { wa[j] = wq * ql[gg].G[a][j]; gb[j] = ql[gg].G[b][j]; }
#pragma unroll
          for (int j = 0; j < DIM; j++)
#pragma unroll
            for (int k = 0; k < DIM; k++) M[j][k] = fma(wa[j], gb[k], M[j][k]);
        }
        for (int f = 0; f < nforms; f++) {  // every LEAN form is ELAST_DOMAIN
          const double lam = forms[f].lam, mu = forms[f].mu, f0 = forms[f].f0;
          double tr = 0.0;
#pragma unroll
          for (int j = 0; j < DIM; j++) tr += M[j][j];
#pragma unroll
          for (int i = 0; i < DIM; i++)
#pragma unroll
            for (int m = 0; m < DIM; m++)
              K[i % KH][m % KH] -= f0 * (lam * M[i][m] + mu * M[m][i] + (i == m ? mu * tr : 0.0));
        }
      } else {
        for (int f = 0; f < nforms; f++)
          if (forms[f].form != FEM_WF_ELAST_LOAD) pair_block<DIM, NL, KH, NQ>(forms[f], qg, a, b, K);
      }
      const int d = S.tdeg[li], sr = acc_row_stride(KH, d, P.nnz_s);
      double* rowb = S.acc + S.toff[li] + pos;
#pragma unroll
      for (int i = 0; i < KH; i++)
#pragma unroll
        for (int m = 0; m < KH; m++) atomicAdd(rowb + i * sr + m * d, K[i][m]);
    } else {
      double rr[KH];
#pragma unroll
      for (int i = 0; i < KH; i++) rr[i] = 0.0;
      if constexpr (LEAN) {
#pragma unroll
        for (int gg = 0; gg < NQ; gg++)
#pragma unroll
          for (int i = 0; i < DIM; i++) {
            double tt = 0.0;
#pragma unroll
            for (int j = 0; j < DIM; j++) tt = fma(ql[gg].S[i][j], ql[gg].G[a][j], tt);
            rr[i % KH] -= tt;
          }
      } else {
        for (int f = 0; f < nforms; f++) row_res<DIM, NL, KH, NQ>(forms[f], qg, a, rr, !FACET && f == 0);
      }
#pragma unroll
      for (int i = 0; i < KH; i++) atomicAdd(S.racc + i * S.T + li, rr[i]);
    }
  }
  __syncwarp();
}

// Stage the tile's halo points (coordinates + state levels) in shared memory.
template <int DIM>
__device__ __forceinline__ void load_halo(const TiledParams& P, TileSmem& S, int64_t tile) {
  const int64_t h0 = P.halo_off[tile];
  const int H = (int)(P.halo_off[tile + 1] - h0);
  S.H = H;
  for (int i = threadIdx.x; i < H; i += blockDim.x) S.hnode[i] = P.halo_node[h0 + i];
  __syncthreads();
  const int ns = P.hcomp - DIM;
  for (int t = threadIdx.x; t < H * P.hcomp; t += blockDim.x) {
    const int c = t / H, i = t % H, node = S.hnode[i];
    S.hdat[t] = c < DIM ? __ldg(P.coords + (int64_t)c * P.N + node) : __ldg(P.state + (int64_t)(c - DIM) * P.N + node);
  }
  (void)ns;
}

// Load the tile's visits of list V into shared memory; returns the count.
template <int NL, bool FACET>
__device__ __forceinline__ int load_visits(const TiledParams& P, const VisitList& V, int64_t tile, const TileSmem& S) {
  const int64_t vb = V.run[V.roff[tile]];
  const int nv = (int)(V.run[V.roff[tile + 1]] - vb);
  for (int t = threadIdx.x; t < nv; t += blockDim.x) {
    S.vid[t] = V.elem[vb + t];
    if constexpr (FACET) S.vfac[t] = V.facet[vb + t];
  }
  __syncthreads();
  for (int t = threadIdx.x; t < nv * NL; t += blockDim.x) {
    const int v = t / NL, a = t % NL;
    const int node = __ldg(P.conn + (int64_t)a * P.E + S.vid[v]);
    S.vnode[t] = node;
    S.vown[t] = (int16_t)find_local(S.tnode, S.T, node);
    if (P.hmax) S.vhal[t] = (int16_t)find_local(S.hnode, S.H, node);
  }
  __syncthreads();
  return nv;
}


// shared-memory carve-up: head (tile points) | per-warp point records | visit arrays | accumulator
template <int NL>
__device__ __forceinline__ TileSmem tile_smem_layout(unsigned char* smem, const TiledParams& P, int warps) {
  TileSmem S;
  S.trps = reinterpret_cast<int64_t*>(smem);
  S.tnode = reinterpret_cast<int32_t*>(S.trps + TILE_MAX_NODES);
  S.tdeg = S.tnode + TILE_MAX_NODES;
  S.toff = S.tdeg + TILE_MAX_NODES;  // [TILE_MAX_NODES + 4]
  unsigned char* p = smem + (20 * TILE_MAX_NODES + 16);
  // union: per-warp point records (facet phase) | staged halo points (domain phase of hex_tiled)
  S.qp = p;
  S.hnode = reinterpret_cast<int32_t*>(p);
  S.hdat = P.hmax ? reinterpret_cast<double*>(p + ((4 * (size_t)P.hmax + 15) / 16) * 16) : nullptr;
  const size_t halo_bytes = P.hmax ? ((4 * (size_t)P.hmax + 15) / 16) * 16 + 8 * (size_t)P.hmax * P.hcomp : 0;
  const size_t slot_bytes = (size_t)P.rec_bytes * warps;
  p += ((halo_bytes > slot_bytes ? halo_bytes : slot_bytes) + 15) / 16 * 16;
  S.vid = reinterpret_cast<int32_t*>(p);
  p += 4 * (size_t)P.vmax;
  S.vnode = reinterpret_cast<int32_t*>(p);
  p += 4 * (size_t)P.vmax * NL;
  S.vown = reinterpret_cast<int16_t*>(p);
  p += 2 * (size_t)P.vmax * NL;
  S.vhal = reinterpret_cast<int16_t*>(p);
  p += P.hmax ? 2 * (size_t)P.vmax * NL : 0;
  S.vfac = reinterpret_cast<int8_t*>(p);
  p += P.vmax;
  p = smem + (((size_t)(p - smem) + 15) / 16) * 16;
  S.acc = reinterpret_cast<double*>(p);
  S.H = 0;
  return S;
}

// tile points, their row offsets (prefix of κ̂²·deg) and a zeroed accumulator
template <int KH>
__device__ __forceinline__ void tile_prologue(const TiledParams& P, TileSmem& S, int64_t tile) {
  const int64_t n0 = P.tile_noff[tile];
  const int T = (int)(P.tile_noff[tile + 1] - n0);
  S.T = T;
  const int tid = threadIdx.x, nth = blockDim.x;
  for (int i = tid; i < T; i += nth) {
    const int node = P.tile_node[n0 + i];
    S.tnode[i] = node;
    const int64_t rr = P.rowptr_s[node - P.own_lo];
    S.trps[i] = rr;
    S.tdeg[i] = (int)(P.rowptr_s[node - P.own_lo + 1] - rr);
  }
  __syncthreads();
  if (tid < 32) {
    int carry = 0;
    for (int base = 0; base < T; base += 32) {
      const int i = base + tid;
      int v = (i < T) ? KH * acc_row_stride(KH, S.tdeg[i], P.nnz_s) : 0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int u = __shfl_up_sync(0xffffffffu, v, o);
        if (tid >= o) v += u;
      }
      if (i < T) S.toff[i + 1] = carry + v;
      carry += __shfl_sync(0xffffffffu, v, 31);
    }
    if (tid == 0) S.toff[0] = 0;
  }
  __syncthreads();
  const int acc_n = P.values ? S.toff[T] : 0;
  S.racc = S.acc + acc_n;
  for (int i = tid; i < acc_n + KH * T; i += nth) S.acc[i] = 0.0;
}

// boundary terms: every facet visit of the tile, warp per visit, atomic accumulation
template <int ET, int ORD, int KH, int Q, int NW = TILED_THREADS / 32>
__device__ __forceinline__ void tile_facets(const TiledParams& P, const TileSmem& S, int64_t tile, unsigned char* slot) {
  using C = TileCfg<ET, ORD, KH, Q>;
  const int warp = threadIdx.x >> 5;
  for (int f = 0; f < P.n_fac; f++) {
    __syncthreads();
    const int nv = load_visits<C::NL, true>(P, P.fvis[f], tile, S);
    if (warp < NW)
      for (int v = warp; v < nv; v += NW) warp_visit<ET, ORD, KH, Q, true, false>(P, &P.fac[f], 1, S, v, slot);
  }
}

// Dynamic work distribution inside a tile: a warp grabs `step` visits from a shared counter.
__device__ __forceinline__ int grab_visits(int* ctr, int step) {
  int v = 0;
  if ((threadIdx.x & 31) == 0) v = atomicAdd(ctr, step);
  return __shfl_sync(0xffffffffu, v, 0);
}

// Boundary terms from the tile record: facet visit i of set k is facet ffac[i] of domain visit fdv[i]
// (the domain view D carries the staged halo and the local column offsets).
template <int ET, int ORD, int KH, int Q, int NW, bool DET = false>
__device__ __forceinline__ void rec_facets(const TiledParams& P, const TileSmem& D, const uint8_t* rec,
                                           const RecLayout& L, unsigned char* slot) {
  const int32_t* fcnt = reinterpret_cast<const int32_t*>(rec + L.o_fcnt);
  const int16_t* fdv = reinterpret_cast<const int16_t*>(rec + L.o_fdv);
  const int8_t* ffac = reinterpret_cast<const int8_t*>(rec + L.o_ffac);
  const int warp = threadIdx.x >> 5;
  __syncthreads();  // per-warp slots may alias scratch used by the domain phase
  if constexpr (DET) {
    // segment by segment (node-disjoint facets, see rec_layout): each accumulator entry receives at
    // most one contribution per segment, from one lane, so the summation order is fixed
    const int32_t* segk = reinterpret_cast<const int32_t*>(rec + L.o_fseg);
    const int32_t* seg = segk + reinterpret_cast<const int32_t*>(rec)[6] + 1;
    for (int f = 0; f < P.n_fac; f++) {
      const int k = P.fac_set[f];
      for (int sg = segk[k]; sg < segk[k + 1]; sg++) {
        if (warp < NW)
          for (int i = seg[sg] + warp; i < seg[sg + 1]; i += NW)
            warp_visit<ET, ORD, KH, Q, true, false>(P, &P.fac[f], 1, D, fdv[i], slot, ffac[i]);
        __syncthreads();
      }
    }
    return;
  }
  if (warp >= NW) return;
  for (int f = 0; f < P.n_fac; f++) {
    const int k = P.fac_set[f];
    for (int i = fcnt[k] + warp; i < fcnt[k + 1]; i += NW)
      warp_visit<ET, ORD, KH, Q, true, false>(P, &P.fac[f], 1, D, fdv[i], slot, ffac[i]);
  }
}

// bulk (TMA) store shared -> global, completion tracked per thread by bulk groups
__device__ __forceinline__ void bulk_s2g(double* dst, const double* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst),
               "r"((uint32_t)__cvta_generic_to_shared(src)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read_all() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// Write every owned row once and the residual rows.  A row segment whose shared-memory copy has the
// 16-byte phase of its destination (the record layout arranges it, see acc_row_stride) leaves by one
// bulk store of its aligned middle plus at most two single doubles; other rows are copied element by
// element.  One thread per row (a tile has a few hundred rows): the bulk stores drain to HBM
// asynchronously; only their shared-memory reads are awaited (before the accumulator is reused).
template <int KH>
__device__ __forceinline__ void tile_epilogue(const TiledParams& P, const TileSmem& S) {
  fence_proxy_async_smem();  // generic-proxy accumulator writes -> async-proxy (bulk copy) reads
  __syncthreads();
  const int tid = threadIdx.x, nth = blockDim.x, T = S.T;
  if (P.values) {
    bool issued = false;
    for (int rr = tid; rr < T * KH; rr += nth) {
      const int li = rr / KH, k0 = rr - li * KH;
      const int d = S.tdeg[li];
      const int len = KH * d;
      const double* src = S.acc + S.toff[li] + k0 * acc_row_stride(KH, d, P.nnz_s);
      double* dst = P.values + (int64_t)k0 * KH * P.nnz_s + (int64_t)KH * S.trps[li];
      if ((((uintptr_t)src ^ (uintptr_t)dst) & 15) == 0 && len >= 4) {
        const int head = ((uintptr_t)dst & 15) ? 1 : 0;
        const int mid = (len - head) & ~1;
        bulk_s2g(dst + head, src + head, 8u * (uint32_t)mid);
        issued = true;
        if (head) dst[0] = src[0];
        if (head + mid < len) dst[len - 1] = src[len - 1];
      } else {
        for (int j = 0; j < len; j++) dst[j] = src[j];
      }
    }
    if (issued) {
      bulk_commit();
      bulk_wait_read_all();  // the accumulator may be zeroed for the next tile after the caller's barrier
    }
  }
  if (P.rhs)
    for (int t = tid; t < KH * T; t += nth) {
      const int k0 = t / T, li = t % T;
      P.rhs[(int64_t)k0 * P.n_own + (S.tnode[li] - P.own_lo)] = S.racc[t];
    }
}

// ---- async copy helpers: TMA bulk copies (cp.async.bulk + mbarrier) and LDGSTS gathers (cp.async)
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}\n" ::"r"(
          smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// mbarrier wait with a suspend-time hint: the waiting warp sleeps in the barrier unit instead of spinning
// on issue slots the other warps of the SM need
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAITS_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, 0x989680;\n @!p bra WAITS_%=;\n}\n" ::"r"(
          smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

int launch_hex_tiled(TiledParams& P, const TileSchedule& T, int kh, bool det, cudaStream_t s, bool* handled);
int launch_ns_tiled(TiledParams& P, const TileSchedule& T, bool det, cudaStream_t s, bool* handled);
int launch_p2_tiled(TiledParams& P, const TileSchedule& T, bool det, cudaStream_t s, bool* handled);

}  // namespace fem
