// tiled.cu — node-tile owner-gather assembly (FEM_SCATTER_TILED), the fast deterministic path.
//
// PAPER.md D-2/D-3 add every element's contribution into d and K "by the (atomic)
// increment".  On B200 an fp64 RED to L2 costs far more than the arithmetic (M0: 0.2-0.3 T RED/s
// vs 33 TF fp64), so instead each CTA OWNS a spatially compact tile of control points and gathers
// all contributions to their rows:
//   - the tile's rows (κ̂² · deg per point) live in a shared-memory accumulator;
//   - the CTA visits every element touching the tile (its own + one ghost layer), in colour runs
//     (elements of one colour share no point, so a run updates each accumulator entry at most once:
//     plain RMW, no atomics, fixed order => bit-exact run to run);
//   - per run batch: one thread per (element, quadrature point) computes J, det J, J^{-1}, ∇N_a, w and
//     the operand fields into shared memory; one thread per (element, owned test node a, trial node b)
//     computes the κ̂×κ̂ pair block (blocks.cuh) and adds it at the row offsets (slot map -> local
//     column offsets, uint8); one thread per (element, owned a) adds the residual row;
//   - finally every owned row is written ONCE to HBM with coalesced stores (no clear pass, no RMW).
// Only the element geometry of ghost-layer elements is recomputed; each (a,b) pair block is computed
// exactly once (by the tile owning a).
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <vector>

#include "blocks.cuh"
#include "elements.cuh"
#include "fem_internal.cuh"

namespace fem {

constexpr int TILE_MAX_NODES = 512;
constexpr int64_t ACC_BUDGET_MAX = 16384;  // doubles (128 KB): hard cap of the row accumulator
static int64_t acc_budget() {  // default 16384 doubles (128 KB): one 16-warp CTA per SM
  static int64_t v = [] {
    const char* s = getenv("FEM_TILE_ACC");
    int64_t x = s ? atoll(s) : 16384;
    return x < 256 ? 256 : (x > ACC_BUDGET_MAX ? ACC_BUDGET_MAX : x);
  }();
  return v;
}
constexpr int MAX_DOM_TERMS = 4;
constexpr int MAX_FAC_TERMS = 8;
constexpr int TILED_THREADS = 512;

// ------------------------------------------------------------------ host: tile schedule
static uint64_t spread_bits3(uint64_t x) {  // 21 bits -> every third bit
  x &= 0x1fffff;
  x = (x | x << 32) & 0x1f00000000ffffull;
  x = (x | x << 16) & 0x1f0000ff0000ffull;
  x = (x | x << 8) & 0x100f00f00f00f00full;
  x = (x | x << 4) & 0x10c30c30c30c30c3ull;
  x = (x | x << 2) & 0x1249249249249249ull;
  return x;
}
static uint64_t spread_bits2(uint64_t x) {  // 31 bits -> every second bit
  x &= 0x7fffffff;
  x = (x | x << 16) & 0x0000ffff0000ffffull;
  x = (x | x << 8) & 0x00ff00ff00ff00ffull;
  x = (x | x << 4) & 0x0f0f0f0f0f0f0f0full;
  x = (x | x << 2) & 0x3333333333333333ull;
  x = (x | x << 1) & 0x5555555555555555ull;
  return x;
}

__global__ void k_loc_table(const int32_t* __restrict__ slot, const int32_t* __restrict__ conn,
                            const int64_t* __restrict__ rowptr_s, int64_t E, int NL, int64_t lo, int64_t hi,
                            uint8_t* __restrict__ loc) {
  const int64_t total = E * NL * NL;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = t / (NL * NL);
    const int ab = (int)(t % (NL * NL)), a = ab / NL;
    const int64_t r = conn[(int64_t)a * E + e];
    uint8_t v = 255;
    if (r >= lo && r < hi) v = (uint8_t)(slot[(int64_t)ab * E + e] - rowptr_s[r - lo]);
    loc[t] = v;
  }
}

static void free_visits(VisitList& V) {
  cudaFree(V.roff); cudaFree(V.run); cudaFree(V.elem); cudaFree(V.facet);
  V = VisitList();
}

void tiles_free(TileSchedule& T) {
  cudaFree(T.tile_noff);
  cudaFree(T.tile_node);
  cudaFree(T.loc);
  free_visits(T.dom);
  for (auto& v : T.bnd) free_visits(v);
  T = TileSchedule();
}

// Sort the visits of every tile by (colour, item) and cut colour runs.
static int make_visits(int64_t n_tiles, const std::vector<int64_t>& voff, std::vector<int32_t>& items,
                       const std::vector<uint8_t>& colour_of_item, const int32_t* elem_of_item,
                       const int8_t* facet_of_item, VisitList& V) {
  std::vector<int64_t> roff(n_tiles + 1, 0), run;
  run.reserve(items.size() / 8 + n_tiles + 1);
  for (int64_t t = 0; t < n_tiles; t++) {
    auto b = items.begin() + voff[t], e = items.begin() + voff[t + 1];
    std::stable_sort(b, e, [&](int32_t x, int32_t y) { return colour_of_item[x] < colour_of_item[y]; });
    roff[t] = (int64_t)run.size();
    for (int64_t i = voff[t]; i < voff[t + 1]; i++)
      if (i == voff[t] || colour_of_item[items[i]] != colour_of_item[items[i - 1]]) run.push_back(i);
  }
  roff[n_tiles] = (int64_t)run.size();
  run.push_back((int64_t)items.size());
  for (int64_t t = 0; t < n_tiles; t++) V.max_per_tile = std::max<int64_t>(V.max_per_tile, voff[t + 1] - voff[t]);
  V.n_runs = (int64_t)run.size() - 1;
  V.n_visits = (int64_t)items.size();
  std::vector<int32_t> el(items.size());
  std::vector<int8_t> fa(facet_of_item ? items.size() : 0);
  for (size_t i = 0; i < items.size(); i++) {
    el[i] = elem_of_item ? elem_of_item[items[i]] : items[i];
    if (facet_of_item) fa[i] = facet_of_item[items[i]];
  }
  FEM_CUDA_TRY(cudaMalloc(&V.roff, sizeof(int64_t) * (n_tiles + 1)));
  FEM_CUDA_TRY(cudaMalloc(&V.run, sizeof(int64_t) * run.size()));
  FEM_CUDA_TRY(cudaMalloc(&V.elem, sizeof(int32_t) * (el.size() + 1)));
  FEM_CUDA_TRY(cudaMemcpy(V.roff, roff.data(), sizeof(int64_t) * (n_tiles + 1), cudaMemcpyHostToDevice));
  FEM_CUDA_TRY(cudaMemcpy(V.run, run.data(), sizeof(int64_t) * run.size(), cudaMemcpyHostToDevice));
  if (!el.empty()) FEM_CUDA_TRY(cudaMemcpy(V.elem, el.data(), sizeof(int32_t) * el.size(), cudaMemcpyHostToDevice));
  if (facet_of_item) {
    FEM_CUDA_TRY(cudaMalloc(&V.facet, sizeof(int8_t) * (fa.size() + 1)));
    if (!fa.empty()) FEM_CUDA_TRY(cudaMemcpy(V.facet, fa.data(), fa.size(), cudaMemcpyHostToDevice));
  }
  return 0;
}

int tiles_build(fem_mesh_s* m, fem_pattern_s* p, cudaStream_t s) {
  TileSchedule& T = p->tiles;
  const int NL = m->n_loc, KH = m->kh, dim = m->dim;
  const int64_t n_own = m->n_own, lo = m->own_lo, E = m->E, N = m->N;
  if (n_own == 0) return 0;
  std::vector<int64_t> rps(n_own + 1);
  FEM_CUDA_TRY(cudaMemcpyAsync(rps.data(), p->rowptr_s, sizeof(int64_t) * (n_own + 1), cudaMemcpyDeviceToHost, s));
  FEM_CUDA_TRY(cudaStreamSynchronize(s));
  std::vector<int64_t> sz(n_own);
  int64_t max_sz = 0;
  for (int64_t i = 0; i < n_own; i++) {
    const int64_t deg = rps[i + 1] - rps[i];
    if (deg > 255) { set_error("tiled schedule: a row has more than 255 scalar neighbours"); return FEM_E_UNSUPPORTED; }
    sz[i] = (int64_t)KH * KH * deg;
    max_sz = std::max(max_sz, sz[i]);
  }
  const int64_t ACC_BUDGET = acc_budget();
  if (max_sz > ACC_BUDGET) { set_error("tiled schedule: one row exceeds the shared accumulator"); return FEM_E_UNSUPPORTED; }
  // 1. Morton order of the owned points (spatial locality independent of the numbering)
  double bmin[3] = {1e300, 1e300, 1e300}, bmax[3] = {-1e300, -1e300, -1e300};
  for (int d = 0; d < dim; d++)
    for (int64_t i = 0; i < n_own; i++) {
      const double x = m->h_coords[(int64_t)d * N + lo + i];
      bmin[d] = std::min(bmin[d], x);
      bmax[d] = std::max(bmax[d], x);
    }
  // quantise on a cell size h ≈ (volume / points)^(1/dim), i.e. about one point per cell, so that a
  // Morton group of level L holds about 2^(dim·L) points (aligned bricks on structured meshes)
  double vol = 1.0;
  for (int d = 0; d < dim; d++) vol *= std::max(bmax[d] - bmin[d], 1e-300);
  const double h = std::pow(vol / (double)n_own, 1.0 / dim);
  const uint64_t qmax = dim == 3 ? (1ull << 21) - 1 : (1ull << 31) - 1;
  std::vector<std::pair<uint64_t, int32_t>> key(n_own);
  for (int64_t i = 0; i < n_own; i++) {
    uint64_t code = 0;
    for (int d = 0; d < dim; d++) {
      double f = (m->h_coords[(int64_t)d * N + lo + i] - bmin[d]) / h;
      f = f < 0 ? 0 : f;
      uint64_t q = (uint64_t)f;
      q = q > qmax ? qmax : q;
      code |= (dim == 3 ? spread_bits3(q) : spread_bits2(q)) << d;
    }
    key[i] = {code, (int32_t)i};
  }
  std::sort(key.begin(), key.end());
  // 2. level of Morton groups whose full group fits the accumulator, then greedy merge
  int L = 0;
  while (L < 7 && (int64_t(1) << (dim * (L + 1))) <= TILE_MAX_NODES &&
         (int64_t(1) << (dim * (L + 1))) * max_sz <= ACC_BUDGET)
    L++;
  std::vector<int64_t> tile_off{0};
  std::vector<int32_t> tile_nodes;
  tile_nodes.reserve(n_own);
  int64_t cur_n = 0, cur_acc = 0, acc_max = 0;
  int max_nodes = 0;
  auto close_tile = [&]() {
    if (cur_n == 0) return;
    std::sort(tile_nodes.end() - cur_n, tile_nodes.end());
    tile_off.push_back((int64_t)tile_nodes.size());
    acc_max = std::max(acc_max, cur_acc);
    max_nodes = std::max(max_nodes, (int)cur_n);
    cur_n = 0;
    cur_acc = 0;
  };
  for (int64_t g0 = 0; g0 < n_own;) {
    int64_t g1 = g0 + 1;
    const uint64_t gk = key[g0].first >> (dim * L);
    while (g1 < n_own && (key[g1].first >> (dim * L)) == gk) g1++;
    int64_t gacc = 0;
    for (int64_t i = g0; i < g1; i++) gacc += sz[key[i].second];
    if (cur_n + (g1 - g0) <= TILE_MAX_NODES && cur_acc + gacc <= ACC_BUDGET) {
      for (int64_t i = g0; i < g1; i++) tile_nodes.push_back((int32_t)(lo + key[i].second));
      cur_n += g1 - g0;
      cur_acc += gacc;
    } else {
      close_tile();
      for (int64_t i = g0; i < g1; i++) {  // group alone: add node by node
        const int64_t zi = sz[key[i].second];
        if (cur_n + 1 > TILE_MAX_NODES || cur_acc + zi > ACC_BUDGET) close_tile();
        tile_nodes.push_back((int32_t)(lo + key[i].second));
        cur_n++;
        cur_acc += zi;
      }
    }
    g0 = g1;
  }
  close_tile();
  const int64_t n_tiles = (int64_t)tile_off.size() - 1;
  T.n_tiles = n_tiles;
  T.max_tile_nodes = max_nodes;
  T.acc_max = acc_max;
  std::vector<int32_t> tile_of(n_own);
  for (int64_t t = 0; t < n_tiles; t++)
    for (int64_t i = tile_off[t]; i < tile_off[t + 1]; i++) tile_of[tile_nodes[i] - lo] = (int32_t)t;
  // 3. element visits: (tile, element) for every distinct tile among the element's owned points
  auto tiles_of_elem = [&](int64_t e, int32_t* out) {
    int n = 0;
    for (int a = 0; a < NL; a++) {
      const int64_t r = m->h_conn[(int64_t)a * E + e];
      if (r < lo || r >= m->own_hi) continue;
      const int32_t t = tile_of[r - lo];
      bool seen = false;
      for (int k = 0; k < n; k++) seen |= (out[k] == t);
      if (!seen) out[n++] = t;
    }
    return n;
  };
  {
    std::vector<int64_t> cnt(n_tiles + 1, 0);
    int32_t buf[16];
    for (int64_t e = 0; e < E; e++) {
      const int n = tiles_of_elem(e, buf);
      for (int k = 0; k < n; k++) cnt[buf[k] + 1]++;
    }
    for (int64_t t = 0; t < n_tiles; t++) cnt[t + 1] += cnt[t];
    std::vector<int32_t> items(cnt[n_tiles]);
    std::vector<int64_t> pos(cnt.begin(), cnt.end() - 1);
    for (int64_t e = 0; e < E; e++) {
      const int n = tiles_of_elem(e, buf);
      for (int k = 0; k < n; k++) items[pos[buf[k]]++] = (int32_t)e;
    }
    T.visits_total = (int64_t)items.size();
    int rc = make_visits(n_tiles, cnt, items, m->h_colour, nullptr, nullptr, T.dom);
    if (rc) return rc;
  }
  // 4. facet visits per boundary set
  T.bnd.resize(m->h_bset_elem.size());
  for (size_t k = 0; k < m->h_bset_elem.size(); k++) {
    const std::vector<int32_t>& be = m->h_bset_elem[k];
    std::vector<int64_t> cnt(n_tiles + 1, 0);
    int32_t buf[16];
    for (size_t j = 0; j < be.size(); j++) {
      const int n = tiles_of_elem(be[j], buf);
      for (int q = 0; q < n; q++) cnt[buf[q] + 1]++;
    }
    for (int64_t t = 0; t < n_tiles; t++) cnt[t + 1] += cnt[t];
    std::vector<int32_t> items(cnt[n_tiles]);
    std::vector<int64_t> pos(cnt.begin(), cnt.end() - 1);
    for (size_t j = 0; j < be.size(); j++) {
      const int n = tiles_of_elem(be[j], buf);
      for (int q = 0; q < n; q++) items[pos[buf[q]]++] = (int32_t)j;
    }
    int rc = make_visits(n_tiles, cnt, items, m->h_bset_colour[k], be.data(), m->h_bset_facet[k].data(), T.bnd[k]);
    if (rc) return rc;
  }
  // 5. device node lists + local column-offset table
  FEM_CUDA_TRY(cudaMalloc(&T.tile_noff, sizeof(int64_t) * (n_tiles + 1)));
  FEM_CUDA_TRY(cudaMalloc(&T.tile_node, sizeof(int32_t) * tile_nodes.size()));
  FEM_CUDA_TRY(cudaMemcpy(T.tile_noff, tile_off.data(), sizeof(int64_t) * (n_tiles + 1), cudaMemcpyHostToDevice));
  FEM_CUDA_TRY(cudaMemcpy(T.tile_node, tile_nodes.data(), sizeof(int32_t) * tile_nodes.size(), cudaMemcpyHostToDevice));
  const int64_t nloc_tot = E * NL * NL;
  FEM_CUDA_TRY(cudaMalloc(&T.loc, nloc_tot > 0 ? nloc_tot : 1));
  if (nloc_tot > 0) {
    int64_t blocks = std::min<int64_t>((nloc_tot + 255) / 256, 148 * 32);
    k_loc_table<<<(unsigned)blocks, 256, 0, s>>>(p->slot, m->conn, p->rowptr_s, E, NL, lo, m->own_hi, T.loc);
    FEM_CUDA_TRY(cudaGetLastError());
  }
  FEM_CUDA_TRY(cudaStreamSynchronize(s));
  return 0;
}

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
  int vmax;      // capacity of the per-tile visit arrays
  int rec_bytes; // bytes of one warp's point-record slot
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
  double* acc;
  double* racc;
  int T;
};

// One warp assembles one element (or facet) visit into the tile accumulator.
template <int ET, int ORD, int KH, int Q, bool FACET, bool LEAN>
__device__ __forceinline__ void warp_visit(const TiledParams& P, const FormArgs* forms, int nforms, const TileSmem& S,
                                           int v, unsigned char* slot) {
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
  if constexpr (FACET) EL::fac_qp(Q, S.vfac[v], gq, xi, wref, mref);
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
      for (int d = 0; d < DIM; d++) X[d] = __ldg(P.coords + (int64_t)d * P.N + nd[a]);
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
        const double s0 = __ldg(P.state + (int64_t)k * P.N + nd[a]);
        u0[k] = fma(N[a], s0, u0[k]);
        if (!LEAN && P.nu_hat >= 1) u1[k] = fma(N[a], __ldg(P.state + ((int64_t)KH + k) * P.N + nd[a]), u1[k]);
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
      const int pos = __ldg(P.loc + (int64_t)e * (NL * NL) + a * NL + b);
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
      const int d = S.tdeg[li];
      double* rowb = S.acc + S.toff[li] + pos;
#pragma unroll
      for (int i = 0; i < KH; i++)
#pragma unroll
        for (int m = 0; m < KH; m++) atomicAdd(rowb + (i * KH + m) * d, K[i][m]);
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
  }
  __syncthreads();
  return nv;
}

template <int ET, int ORD, int KH, int Q>
__global__ void __launch_bounds__(TILED_THREADS, 1) k_tiled(const __grid_constant__ TiledParams P) {
  using C = TileCfg<ET, ORD, KH, Q>;
  constexpr int NL = C::NL;
  extern __shared__ __align__(16) unsigned char smem[];
  TileSmem S;
  S.trps = reinterpret_cast<int64_t*>(smem);
  S.tnode = reinterpret_cast<int32_t*>(S.trps + TILE_MAX_NODES);
  S.tdeg = S.tnode + TILE_MAX_NODES;
  S.toff = S.tdeg + TILE_MAX_NODES;  // [TILE_MAX_NODES + 4]
  unsigned char* p = smem + C::HEAD_BYTES;
  S.qp = p;
  p += (size_t)P.rec_bytes * C::WARPS;
  S.vid = reinterpret_cast<int32_t*>(p);
  p += 4 * (size_t)P.vmax;
  S.vnode = reinterpret_cast<int32_t*>(p);
  p += 4 * (size_t)P.vmax * NL;
  S.vown = reinterpret_cast<int16_t*>(p);
  p += 2 * (size_t)P.vmax * NL;
  S.vfac = reinterpret_cast<int8_t*>(p);
  p += P.vmax;
  p = smem + (((size_t)(p - smem) + 15) / 16) * 16;
  S.acc = reinterpret_cast<double*>(p);
  const int64_t tile = blockIdx.x;
  const int64_t n0 = P.tile_noff[tile];
  const int T = (int)(P.tile_noff[tile + 1] - n0);
  S.T = T;
  const int tid = threadIdx.x, nth = blockDim.x, warp = tid >> 5;
  for (int i = tid; i < T; i += nth) {
    const int node = P.tile_node[n0 + i];
    S.tnode[i] = node;
    const int64_t rr = P.rowptr_s[node - P.own_lo];
    S.trps[i] = rr;
    S.tdeg[i] = (int)(P.rowptr_s[node - P.own_lo + 1] - rr);
  }
  __syncthreads();
  if (tid < 32) {  // prefix of the row-block sizes κ̂²·deg
    int carry = 0;
    for (int base = 0; base < T; base += 32) {
      const int i = base + tid;
      int v = (i < T) ? KH * KH * S.tdeg[i] : 0;
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
  unsigned char* slot = S.qp + (size_t)P.rec_bytes * warp;
  {
    const int nv = load_visits<NL, false>(P, P.dvis, tile, S);  // (its first barrier also covers the zeroing)
    if (P.lean)
      for (int v = warp; v < nv; v += C::WARPS) warp_visit<ET, ORD, KH, Q, false, true>(P, P.dom, P.n_dom, S, v, slot);
    else
      for (int v = warp; v < nv; v += C::WARPS) warp_visit<ET, ORD, KH, Q, false, false>(P, P.dom, P.n_dom, S, v, slot);
  }
  for (int f = 0; f < P.n_fac; f++) {
    __syncthreads();
    const int nv = load_visits<NL, true>(P, P.fvis[f], tile, S);
    for (int v = warp; v < nv; v += C::WARPS) warp_visit<ET, ORD, KH, Q, true, false>(P, &P.fac[f], 1, S, v, slot);
  }
  __syncthreads();
  // write every owned row once (coalesced, one warp per row)
  if (P.values) {
    const int lane = tid & 31, nw = nth >> 5;
    for (int rr = warp; rr < T * KH; rr += nw) {
      const int li = rr / KH, k0 = rr % KH;
      const int len = KH * S.tdeg[li];
      const double* src = S.acc + S.toff[li] + k0 * len;
      double* dst = P.values + (int64_t)k0 * KH * P.nnz_s + (int64_t)KH * S.trps[li];
      for (int j = lane; j < len; j += 32) dst[j] = src[j];
    }
  }
  if (P.rhs)
    for (int t = tid; t < KH * T; t += nth) {
      const int k0 = t / T, li = t % T;
      P.rhs[(int64_t)k0 * P.n_own + (S.tnode[li] - P.own_lo)] = S.racc[t];
    }
}

template <int ET, int ORD, int KH, int Q>
static int run_tiled(TiledParams& P, const TileSchedule& T, cudaStream_t s) {
  using C = TileCfg<ET, ORD, KH, Q>;
  constexpr int NL = C::NL;
  const size_t rec_dom = (P.lean ? sizeof(typename C::QPL) : sizeof(typename C::QPG)) * C::NQV;
  const size_t rec_fac = sizeof(typename C::QPG) * C::NQF;
  P.rec_bytes = (int)((std::max(rec_dom, rec_fac) + 15) / 16 * 16);
  int vmax = (int)T.dom.max_per_tile;
  for (int f = 0; f < P.n_fac; f++) vmax = std::max<int>(vmax, (int)P.fvis[f].max_per_tile);
  vmax = std::max(vmax, 1);
  P.vmax = vmax;
  const size_t vis_bytes = (size_t)vmax * (4 + 1) + (size_t)vmax * NL * (4 + 2) + 16;
  const size_t smem = C::HEAD_BYTES + (size_t)P.rec_bytes * C::WARPS + vis_bytes + 16 +
                      sizeof(double) * ((P.values ? T.acc_max : 0) + (size_t)KH * T.max_tile_nodes);
  if (smem > 227 * 1024) {
    set_error("tiled kernel: shared memory request too large (" + std::to_string(smem) + " B)");
    return FEM_E_UNSUPPORTED;
  }
  FEM_CUDA_TRY(cudaFuncSetAttribute(k_tiled<ET, ORD, KH, Q>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  if (T.n_tiles <= 0) return 0;
  k_tiled<ET, ORD, KH, Q><<<(unsigned)T.n_tiles, TILED_THREADS, smem, s>>>(P);
  FEM_CUDA_TRY(cudaGetLastError());
  return 0;
}

template <int ET, int ORD, int KH>
static int run_tiled_q(int q, TiledParams& P, const TileSchedule& T, cudaStream_t s) {
  if (q == 1) return run_tiled<ET, ORD, KH, 1>(P, T, s);
  if (q == 2) return run_tiled<ET, ORD, KH, 2>(P, T, s);
  if constexpr (ET == ET_HEX) {
    if (q == 3) return run_tiled<ET, ORD, KH, 3>(P, T, s);
  }
  set_error("tiled: unsupported quadrature order");
  return FEM_E_UNSUPPORTED;
}

int launch_tiled(const fem_mesh_s* m, const fem_pattern_s* pat, const fem_problem* prob, const double* state,
                 double* values, double* rhs, cudaStream_t s) {
  const TileSchedule& T = pat->tiles;
  TiledParams P;
  memset(&P, 0, sizeof(P));
  bool lean = m->physics == FEM_ELASTICITY;
  for (int t = 0; t < prob->n_terms; t++) {
    const fem_term& term = prob->terms[t];
    if (term.region < 0) {
      if (P.n_dom == MAX_DOM_TERMS) { set_error("tiled: too many domain terms"); return FEM_E_UNSUPPORTED; }
      P.dom[P.n_dom++] = make_form_args(prob, term);
      lean &= term.form == FEM_WF_ELAST_DOMAIN;
    } else {
      if (P.n_fac == MAX_FAC_TERMS) { set_error("tiled: too many boundary terms"); return FEM_E_UNSUPPORTED; }
      P.fvis[P.n_fac] = T.bnd[term.region];
      P.fac[P.n_fac++] = make_form_args(prob, term);
    }
  }
  // (NS point records use ρ = params[0] of the batch's first form; every NS form stores ρ first)
  P.lean = lean && P.n_dom > 0;
  P.dvis = T.dom;
  P.tile_noff = T.tile_noff;
  P.tile_node = T.tile_node;
  P.N = m->N; P.E = m->E; P.own_lo = m->own_lo; P.n_own = m->n_own; P.nnz_s = pat->nnz_s;
  P.coords = m->coords; P.conn = m->conn; P.state = state;
  P.rowptr_s = pat->rowptr_s; P.loc = T.loc;
  P.values = values; P.rhs = rhs; P.err = m->err;
  P.nu_hat = prob->time.kind == FEM_TIME_GENALPHA ? prob->time.nu_hat : 0;
  const int et = m->etype, o = m->order, kh = m->kh, q = prob->quad_order;
  if (et == ET_TRI && o == 1) {
    if (kh == 1) return run_tiled_q<ET_TRI, 1, 1>(q, P, T, s);
    if (kh == 2) return run_tiled_q<ET_TRI, 1, 2>(q, P, T, s);
  }
  if (et == ET_HEX && o == 1) {
    if (kh == 1) return run_tiled_q<ET_HEX, 1, 1>(q, P, T, s);
    if (kh == 3) return run_tiled_q<ET_HEX, 1, 3>(q, P, T, s);
  }
  if (et == ET_TET && o == 1) {
    if (kh == 1) return run_tiled_q<ET_TET, 1, 1>(q, P, T, s);
    if (kh == 3) return run_tiled_q<ET_TET, 1, 3>(q, P, T, s);
    if (kh == 4) return run_tiled_q<ET_TET, 1, 4>(q, P, T, s);
  }
  if (et == ET_TET && o == 2) {
    if (kh == 1) return run_tiled_q<ET_TET, 2, 1>(q, P, T, s);
    if (kh == 3) return run_tiled_q<ET_TET, 2, 3>(q, P, T, s);
  }
  set_error("tiled: unsupported element/physics combination");
  return FEM_E_UNSUPPORTED;
}

}  // namespace fem
