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

#include "tiled.cuh"

namespace fem {

constexpr int64_t ACC_BUDGET_MAX = 16384;  // doubles (128 KB): hard cap of the row accumulator
static int64_t acc_budget() {  // default 16384 doubles (128 KB): one 16-warp CTA per SM
  static int64_t v = [] {
    const char* s = getenv("FEM_TILE_ACC");
    int64_t x = s ? atoll(s) : 16384;
    return x < 256 ? 256 : (x > ACC_BUDGET_MAX ? ACC_BUDGET_MAX : x);
  }();
  return v;
}

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
  cudaFree(T.halo_off);
  cudaFree(T.halo_node);
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
    // halo: the sorted unique points of the elements each tile visits (staged in shared memory)
    std::vector<int64_t> hoff(n_tiles + 1, 0);
    std::vector<int32_t> hnode;
    hnode.reserve(items.size() * 2);
    std::vector<int32_t> tmp;
    for (int64_t t = 0; t < n_tiles; t++) {
      tmp.clear();
      for (int64_t i = cnt[t]; i < cnt[t + 1]; i++)
        for (int a = 0; a < NL; a++) tmp.push_back(m->h_conn[(int64_t)a * E + items[i]]);
      std::sort(tmp.begin(), tmp.end());
      tmp.erase(std::unique(tmp.begin(), tmp.end()), tmp.end());
      hnode.insert(hnode.end(), tmp.begin(), tmp.end());
      hoff[t + 1] = (int64_t)hnode.size();
      T.max_halo = std::max<int64_t>(T.max_halo, (int64_t)tmp.size());
    }
    FEM_CUDA_TRY(cudaMalloc(&T.halo_off, sizeof(int64_t) * (n_tiles + 1)));
    FEM_CUDA_TRY(cudaMalloc(&T.halo_node, sizeof(int32_t) * (hnode.size() + 1)));
    FEM_CUDA_TRY(cudaMemcpy(T.halo_off, hoff.data(), sizeof(int64_t) * (n_tiles + 1), cudaMemcpyHostToDevice));
    if (!hnode.empty())
      FEM_CUDA_TRY(cudaMemcpy(T.halo_node, hnode.data(), sizeof(int32_t) * hnode.size(), cudaMemcpyHostToDevice));
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

template <int ET, int ORD, int KH, int Q>
__global__ void __launch_bounds__(TILED_THREADS, 1) k_tiled(const __grid_constant__ TiledParams P) {
  using C = TileCfg<ET, ORD, KH, Q>;
  constexpr int NL = C::NL;
  extern __shared__ __align__(16) unsigned char smem[];
  TileSmem S = tile_smem_layout<NL>(smem, P, C::WARPS);
  const int64_t tile = blockIdx.x;
  tile_prologue<KH>(P, S, tile);
  const int warp = threadIdx.x >> 5;
  unsigned char* slot = S.qp + (size_t)P.rec_bytes * warp;
  {
    const int nv = load_visits<NL, false>(P, P.dvis, tile, S);  // (its first barrier also covers the zeroing)
    if (P.lean)
      for (int v = warp; v < nv; v += C::WARPS) warp_visit<ET, ORD, KH, Q, false, true>(P, P.dom, P.n_dom, S, v, slot);
    else
      for (int v = warp; v < nv; v += C::WARPS) warp_visit<ET, ORD, KH, Q, false, false>(P, P.dom, P.n_dom, S, v, slot);
  }
  tile_facets<ET, ORD, KH, Q>(P, S, tile, slot);
  tile_epilogue<KH>(P, S);
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
  const size_t vis_bytes = (size_t)vmax * (4 + 1) + (size_t)vmax * NL * (4 + 2) + 32;
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
  if (et == ET_HEX && o == 1 && q == 2 && !getenv("FEM_NO_HEX_MMA")) {
    bool handled = false;
    const int rc = launch_hex_tiled(P, T, kh, getenv("FEM_TILED_DET") != nullptr, s, &handled);
    if (handled) return rc;
  }
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
