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
#include <tuple>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <vector>

#include "tiled.cuh"

namespace fem {

constexpr int64_t ACC_BUDGET_MAX = 16384;  // doubles (128 KB): hard cap of the row accumulator
// Cap on element visits per tile (bounds the packed record, double-buffered in shared memory).
static int64_t tile_visit_cap(int NL) { return NL == 8 ? 144 : (NL == 10 ? 240 : 640); }
// Cap on halo points per tile (bounds the staged coordinates/state, double-buffered).
static int64_t tile_halo_cap(int NL) { return NL == 8 ? 300 : (NL == 10 ? 480 : 640); }

// Accumulator budget (doubles).  κ̂ = 1 rows are short, so a tile would hold hundreds of points and
// its packed record (double-buffered in shared memory) would not fit: cap it at 4096 doubles.
static int64_t acc_budget(int kh, int nl) {
  // P2 tets: 144 B of visit data per element, so the double-buffered records need room too
  int64_t x = kh == 1 ? 4096 : (nl == 10 ? 8192 : 16384);
  return x < 256 ? 256 : (x > ACC_BUDGET_MAX ? ACC_BUDGET_MAX : x);
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
  cudaFree(T.seq_off);
  cudaFree(T.sw_lperm);
  cudaFree(T.sw_pcoords);
  cudaFree(T.sw_pstate);
  cudaFree(T.rec);
  cudaFree(T.rec_off);
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
                       const int8_t* facet_of_item, VisitList& V, std::vector<int64_t>* roff_out = nullptr,
                       std::vector<int64_t>* run_out = nullptr) {
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
  if (roff_out) *roff_out = std::move(roff);
  if (run_out) *run_out = std::move(run);
  return 0;
}

// Local column offsets of every (visit, a, b) written straight into the tile records.
__global__ void k_fill_rec_loc(uint8_t* __restrict__ rec, const int64_t* __restrict__ vis_loc_off,
                               const int32_t* __restrict__ vis_elem, int64_t n_vis, const int32_t* __restrict__ slot,
                               const int32_t* __restrict__ conn, const int64_t* __restrict__ rowptr_s, int64_t E,
                               int NL, int64_t lo, int64_t hi) {
  const int64_t total = n_vis * NL * NL;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t v = t / (NL * NL);
    const int ab = (int)(t % (NL * NL)), a = ab / NL;
    const int64_t e = vis_elem[v];
    const int64_t r = conn[(int64_t)a * E + e];
    uint8_t val = 255;
    if (r >= lo && r < hi) val = (uint8_t)(slot[(int64_t)ab * E + e] - rowptr_s[r - lo]);
    rec[vis_loc_off[v] + ab] = val;
  }
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
    sz[i] = (int64_t)KH * acc_row_stride(KH, (int)deg, p->nnz_s) + 1;  // + phase pad
    max_sz = std::max(max_sz, sz[i]);
  }
  const int64_t ACC_BUDGET = acc_budget(KH, NL);
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
  // point -> element adjacency, to bound the number of element visits of a tile (its record size)
  std::vector<int64_t> adj_off(n_own + 1, 0);
  for (int64_t i = 0; i < (int64_t)NL * E; i++) {
    const int64_t r = m->h_conn[i];
    if (r >= lo && r < m->own_hi) adj_off[r - lo + 1]++;
  }
  for (int64_t i = 0; i < n_own; i++) adj_off[i + 1] += adj_off[i];
  std::vector<int32_t> adj(adj_off[n_own]);
  {
    std::vector<int64_t> pos(adj_off.begin(), adj_off.end() - 1);
    for (int64_t e = 0; e < E; e++)
      for (int a = 0; a < NL; a++) {
        const int64_t r = m->h_conn[(int64_t)a * E + e];
        if (r >= lo && r < m->own_hi) adj[pos[r - lo]++] = (int32_t)e;
      }
  }
  std::vector<int64_t> stamp(E, -1);  // element -> id of the last tile (or probe) that counted it
  std::vector<int64_t> nstamp(N, -1); // point -> id of the last tile that counted it in its halo
  int64_t stamp_id = 0;
  const int64_t VISIT_CAP = tile_visit_cap(NL), HALO_CAP = tile_halo_cap(NL);
  int64_t cur_n = 0, cur_acc = 0, cur_vis = 0, cur_halo = 0, acc_max = 0;
  int max_nodes = 0;
  auto close_tile = [&]() {
    if (cur_n == 0) return;
    std::sort(tile_nodes.end() - cur_n, tile_nodes.end());
    tile_off.push_back((int64_t)tile_nodes.size());
    acc_max = std::max(acc_max, cur_acc);
    max_nodes = std::max(max_nodes, (int)cur_n);
    cur_n = 0;
    cur_acc = 0;
    cur_vis = 0;
    cur_halo = 0;
    stamp_id++;
  };
  // new elements a set of points would add to the current tile (without committing)
  std::vector<int32_t> newe, newn;
  int64_t probe_halo = 0;
  auto probe = [&](int64_t g0, int64_t g1) {
    newe.clear();
    newn.clear();
    for (int64_t i = g0; i < g1; i++) {
      const int64_t li = key[i].second;
      for (int64_t k = adj_off[li]; k < adj_off[li + 1]; k++)
        if (stamp[adj[k]] != stamp_id) newe.push_back(adj[k]);
    }
    std::sort(newe.begin(), newe.end());
    newe.erase(std::unique(newe.begin(), newe.end()), newe.end());
    for (int32_t e : newe)
      for (int a = 0; a < NL; a++) {
        const int32_t r = m->h_conn[(int64_t)a * E + e];
        if (nstamp[r] != stamp_id) newn.push_back(r);
      }
    std::sort(newn.begin(), newn.end());
    newn.erase(std::unique(newn.begin(), newn.end()), newn.end());
    probe_halo = (int64_t)newn.size();
    return (int64_t)newe.size();
  };
  auto commit = [&](int64_t g0, int64_t g1, int64_t gacc) {
    for (int64_t i = g0; i < g1; i++) tile_nodes.push_back((int32_t)(lo + key[i].second));
    for (int32_t e : newe) stamp[e] = stamp_id;
    for (int32_t r : newn) nstamp[r] = stamp_id;
    cur_n += g1 - g0;
    cur_acc += gacc;
    cur_vis += (int64_t)newe.size();
    cur_halo += probe_halo;
  };
  for (int64_t g0 = 0; g0 < n_own;) {
    int64_t g1 = g0 + 1;
    const uint64_t gk = key[g0].first >> (dim * L);
    while (g1 < n_own && (key[g1].first >> (dim * L)) == gk) g1++;
    int64_t gacc = 0;
    for (int64_t i = g0; i < g1; i++) gacc += sz[key[i].second];
    const int64_t gvis = probe(g0, g1);
    if (cur_n + (g1 - g0) <= TILE_MAX_NODES && cur_acc + gacc <= ACC_BUDGET && cur_vis + gvis <= VISIT_CAP &&
        cur_halo + probe_halo <= HALO_CAP) {
      commit(g0, g1, gacc);
    } else {
      close_tile();
      for (int64_t i = g0; i < g1; i++) {  // group alone: add point by point
        const int64_t zi = sz[key[i].second];
        int64_t vi = probe(i, i + 1);
        if (cur_n + 1 > TILE_MAX_NODES || cur_acc + zi > ACC_BUDGET ||
            (cur_n > 0 && (cur_vis + vi > VISIT_CAP || cur_halo + probe_halo > HALO_CAP))) {
          close_tile();
          vi = probe(i, i + 1);
        }
        commit(i, i + 1, zi);
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
  std::vector<int32_t> dom_items;
  std::vector<int64_t> dom_cnt, dom_roff, dom_run;
  std::vector<uint32_t> fac_mask(n_tiles, 0);
  std::vector<std::vector<int64_t>> fac_cnt;   // per boundary set: facet-visit offsets per tile
  std::vector<std::vector<int32_t>> fac_items; // per boundary set: facet entries, tile-major
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
    std::vector<int64_t> roff, run;
    int rc = make_visits(n_tiles, cnt, items, m->h_colour, nullptr, nullptr, T.dom, &roff, &run);
    if (rc) return rc;
    dom_items = std::move(items);
    dom_cnt = std::move(cnt);
    dom_roff = std::move(roff);
    dom_run = std::move(run);
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
    for (int64_t t = 0; t < n_tiles; t++)
      if (cnt[t + 1] > cnt[t] && k < 32) fac_mask[t] |= 1u << k;
    fac_cnt.push_back(std::move(cnt));
    fac_items.push_back(std::move(items));
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
  // 6. packed per-tile records (one bulk copy per tile in the record-driven kernels)
  {
    std::vector<int64_t> roff(n_tiles + 1, 0);
    std::vector<int32_t> halo;
    std::vector<int64_t> hoff(n_tiles + 1, 0);
    std::vector<int32_t> tmp;
    // facet visits of tile t: per set, ordered by (rank of the facet among its element's facets in the set,
    // domain visit, facet id), cut into segments of strictly increasing visits of one colour
    std::vector<int16_t> f_dv;
    std::vector<int8_t> f_fac;
    std::vector<int32_t> f_cnt, f_segk, f_seg;
    auto tile_facet_lists = [&](int64_t t) {
      const int nv = (int)(dom_cnt[t + 1] - dom_cnt[t]);
      const int nb = (int)fac_cnt.size();
      f_dv.clear(); f_fac.clear(); f_cnt.assign(1, 0); f_segk.assign(1, 0); f_seg.clear();
      if (nb == 0) { f_seg.push_back(0); return; }
      std::vector<std::pair<int32_t, int16_t>> ev(nv);
      for (int v = 0; v < nv; v++) ev[v] = {dom_items[dom_cnt[t] + v], (int16_t)v};
      std::sort(ev.begin(), ev.end());
      const int64_t r0 = dom_roff[t], nruns = dom_roff[t + 1] - r0;
      auto colour_of = [&](int v) {  // run index of visit v
        int r = 0;
        while (r + 1 < nruns && dom_run[r0 + r + 1] - dom_cnt[t] <= v) r++;
        return r;
      };
      std::vector<std::tuple<int, int16_t, int8_t>> items;
      std::vector<int> seen(nv, 0);
      for (int k = 0; k < nb; k++) {
        items.clear();
        for (int64_t j = fac_cnt[k][t]; j < fac_cnt[k][t + 1]; j++) {
          const int32_t entry = fac_items[k][j];
          const int32_t e = m->h_bset_elem[k][entry];
          auto f = std::lower_bound(ev.begin(), ev.end(), std::make_pair(e, (int16_t)-32768));
          items.emplace_back(seen[f->second]++, f->second, m->h_bset_facet[k][entry]);
        }
        for (auto& it : items) seen[std::get<1>(it)] = 0;
        std::sort(items.begin(), items.end());
        int prev_v = -1, prev_c = -1;
        for (auto& it : items) {
          const int v = std::get<1>(it), c = colour_of(v);
          if (v <= prev_v || c != prev_c) f_seg.push_back((int32_t)f_dv.size());
          prev_v = v; prev_c = c;
          f_dv.push_back((int16_t)v);
          f_fac.push_back(std::get<2>(it));
        }
        f_cnt.push_back((int32_t)f_dv.size());
        f_segk.push_back((int32_t)f_seg.size());
      }
      f_seg.push_back((int32_t)f_dv.size());
    };
    for (int64_t t = 0; t < n_tiles; t++) {
      const int64_t nvt = dom_cnt[t + 1] - dom_cnt[t];
      tmp.clear();
      for (int64_t i = dom_cnt[t]; i < dom_cnt[t + 1]; i++)
        for (int a = 0; a < NL; a++) tmp.push_back(m->h_conn[(int64_t)a * E + dom_items[i]]);
      std::sort(tmp.begin(), tmp.end());
      tmp.erase(std::unique(tmp.begin(), tmp.end()), tmp.end());
      halo.insert(halo.end(), tmp.begin(), tmp.end());
      hoff[t + 1] = (int64_t)halo.size();
      const int nruns = (int)(dom_roff[t + 1] - dom_roff[t]);
      tile_facet_lists(t);
      const RecLayout L = rec_layout(NL, (int)(tile_off[t + 1] - tile_off[t]), (int)tmp.size(), (int)nvt, nruns,
                                     (int)fac_cnt.size(), (int)f_dv.size(), (int)f_seg.size() - 1);
      roff[t + 1] = roff[t] + L.size;
      T.rec_max = std::max<int64_t>(T.rec_max, L.size);
    }
    std::vector<uint8_t> buf((size_t)roff[n_tiles], 0);
    std::vector<int64_t> vis_loc(dom_items.size());
    int max_turns_all = 0;
    for (int64_t t = 0; t < n_tiles; t++) {
      const int Tn = (int)(tile_off[t + 1] - tile_off[t]);
      const int H = (int)(hoff[t + 1] - hoff[t]);
      const int nv = (int)(dom_cnt[t + 1] - dom_cnt[t]);
      const int nruns = (int)(dom_roff[t + 1] - dom_roff[t]);
      const int nb = (int)fac_cnt.size();
      tile_facet_lists(t);
      const int nf = (int)f_dv.size(), ns = (int)f_seg.size() - 1;
      const RecLayout L = rec_layout(NL, Tn, H, nv, nruns, nb, nf, ns);
      uint8_t* r = buf.data() + roff[t];
      int32_t* hdr = reinterpret_cast<int32_t*>(r);
      const int32_t* tn = tile_nodes.data() + tile_off[t];
      const int32_t* hn = halo.data() + hoff[t];
      int32_t* o_tnode = reinterpret_cast<int32_t*>(r + L.o_tnode);
      int32_t* o_tdeg = reinterpret_cast<int32_t*>(r + L.o_tdeg);
      int32_t* o_toff = reinterpret_cast<int32_t*>(r + L.o_toff);
      int64_t* o_trps = reinterpret_cast<int64_t*>(r + L.o_trps);
      int acc = 0;
      for (int i = 0; i < Tn; i++) {
        const int64_t li = tn[i] - lo;
        o_tnode[i] = tn[i];
        o_trps[i] = rps[li];
        o_tdeg[i] = (int32_t)(rps[li + 1] - rps[li]);
        if ((acc ^ (int)((KH * rps[li]) & 1)) & 1) acc++;  // 16-byte phase of the destination rows
        o_toff[i] = acc;
        acc += KH * acc_row_stride(KH, o_tdeg[i], p->nnz_s);
      }
      o_toff[Tn] = acc;
      hdr[0] = Tn; hdr[1] = H; hdr[2] = nv; hdr[3] = nruns; hdr[4] = acc; hdr[5] = (int32_t)fac_mask[t];
      hdr[6] = nb; hdr[7] = nf; hdr[8] = ns;
      if (nb > 0) {  // facet visits: (domain visit of the facet's element, facet id) + segments
        memcpy(r + L.o_fcnt, f_cnt.data(), sizeof(int32_t) * f_cnt.size());
        memcpy(r + L.o_fdv, f_dv.data(), sizeof(int16_t) * f_dv.size());
        memcpy(r + L.o_ffac, f_fac.data(), f_fac.size());
        memcpy(r + L.o_fseg, f_segk.data(), sizeof(int32_t) * f_segk.size());
        memcpy(r + L.o_fseg + 4 * (nb + 1), f_seg.data(), sizeof(int32_t) * f_seg.size());
      }
      memcpy(r + L.o_hnode, hn, sizeof(int32_t) * H);
      int32_t* o_run = reinterpret_cast<int32_t*>(r + L.o_run);
      for (int k = 0; k <= nruns; k++) o_run[k] = (int32_t)(dom_run[dom_roff[t] + k] - dom_cnt[t]);
      int32_t* o_velem = reinterpret_cast<int32_t*>(r + L.o_velem);
      uint16_t* o_vhal = reinterpret_cast<uint16_t*>(r + L.o_vhal);
      int16_t* o_vown = reinterpret_cast<int16_t*>(r + L.o_vown);
      uint8_t* o_vseq = r + L.o_vseq;
      std::vector<int> turn(Tn, 0);
      for (int v = 0; v < nv; v++) {
        const int64_t gi = dom_cnt[t] + v;
        const int32_t e = dom_items[gi];
        o_velem[v] = e;
        for (int a = 0; a < NL; a++) {
          const int32_t node = m->h_conn[(int64_t)a * E + e];
          o_vhal[v * NL + a] = (uint16_t)(std::lower_bound(hn, hn + H, node) - hn);
          const int32_t* f = std::lower_bound(tn, tn + Tn, node);
          o_vown[v * NL + a] = (f != tn + Tn && *f == node) ? (int16_t)(f - tn) : (int16_t)-1;
          o_vseq[v * NL + a] = o_vown[v * NL + a] >= 0 ? (uint8_t)std::min(turn[f - tn]++, 255) : (uint8_t)0;
        }
        vis_loc[gi] = roff[t] + L.o_vloc + (int64_t)v * NL * NL;
      }
      for (int i = 0; i < Tn; i++) max_turns_all = std::max(max_turns_all, turn[i]);
    }
    T.max_turns = max_turns_all;
    FEM_CUDA_TRY(cudaMalloc(&T.rec, buf.size() + 16));
    FEM_CUDA_TRY(cudaMalloc(&T.rec_off, sizeof(int64_t) * (n_tiles + 1)));
    FEM_CUDA_TRY(cudaMemcpy(T.rec, buf.data(), buf.size(), cudaMemcpyHostToDevice));
    FEM_CUDA_TRY(cudaMemcpy(T.rec_off, roff.data(), sizeof(int64_t) * (n_tiles + 1), cudaMemcpyHostToDevice));
    T.rec_bytes_total = (int64_t)buf.size();
    int64_t* d_vloc = nullptr;
    FEM_CUDA_TRY(cudaMalloc(&d_vloc, sizeof(int64_t) * (vis_loc.size() + 1)));
    FEM_CUDA_TRY(cudaMemcpy(d_vloc, vis_loc.data(), sizeof(int64_t) * vis_loc.size(), cudaMemcpyHostToDevice));
    const int64_t tot = (int64_t)vis_loc.size() * NL * NL;
    if (tot > 0) {
      const int64_t blocks = std::min<int64_t>((tot + 255) / 256, 148 * 32);
      k_fill_rec_loc<<<(unsigned)blocks, 256, 0, s>>>(T.rec, d_vloc, T.dom.elem, (int64_t)vis_loc.size(), p->slot,
                                                       m->conn, p->rowptr_s, E, NL, lo, m->own_hi);
      FEM_CUDA_TRY(cudaGetLastError());
    }
    FEM_CUDA_TRY(cudaStreamSynchronize(s));
    cudaFree(d_vloc);
  }
  return 0;
}

// ---- persistent record-driven generic kernel (tets, triangles, hex with other forms): the next tile's
// packed record arrives by one TMA bulk copy while the current tile computes; the tile's halo points
// (coordinates + state) are staged in shared memory once per tile; warps take element visits freely
// and accumulate with shared-memory fp64 atomics.
template <int NL, int DIM>
__device__ __forceinline__ void gather_halo_gen(const TiledParams& P, const uint8_t* rec, double* hbuf) {
  const int32_t* hdr = reinterpret_cast<const int32_t*>(rec);
  const int H = hdr[1];
  const RecLayout L = rec_layout_hdr(NL, hdr);
  const int32_t* hn = reinterpret_cast<const int32_t*>(rec + L.o_hnode);
  for (int t = threadIdx.x; t < H * P.hcomp; t += blockDim.x) {
    const int c = t / H, i = t % H, node = hn[i];
    const double* src = c < DIM ? P.coords + (int64_t)c * P.N + node : P.state + (int64_t)(c - DIM) * P.N + node;
    cp_async8(hbuf + t, src);
  }
  cp_async_commit();
}

// DET: the visits of a colour run share no point, so within a run every accumulator entry receives at most
// one contribution; runs are separated by block barriers and boundary facets go by node-disjoint segments
// (rec_facets): the sums have a fixed order, bit-identical run to run.  !DET: warps grab visits freely and
// shared-memory fp64 atomics resolve the conflicts (FEM_SCATTER_TILED_UNORDERED).
template <int ET, int ORD, int KH, int Q, bool DET>
__global__ void __launch_bounds__(TILED_THREADS, 1) k_gen_rec(const __grid_constant__ TiledParams P) {
  using C = TileCfg<ET, ORD, KH, Q>;
  constexpr int NL = C::NL, DIM = C::DIM;
  extern __shared__ __align__(16) unsigned char smem[];
  uint64_t* mbar = reinterpret_cast<uint64_t*>(smem);
  int* ctr = reinterpret_cast<int*>(smem + 64);
  unsigned char* rbuf[2] = {smem + 128, smem + 128 + P.rec_cap};
  double* hbuf = reinterpret_cast<double*>(smem + 128 + 2 * (size_t)P.rec_cap);
  double* acc = hbuf + P.hcap;
  TileSmem S;
  unsigned char* fp = reinterpret_cast<unsigned char*>(acc + P.acc_cap);
  S.qp = fp;
  fp += (size_t)P.rec_bytes * C::WARPS;
  S.vid = reinterpret_cast<int32_t*>(fp);  // facet-phase visit arrays
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
  const int tid = threadIdx.x, warp = tid >> 5;
  unsigned char* slot = S.qp + (size_t)P.rec_bytes * warp;
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
    if (tid == 0 && next < P.n_tiles) {  // prefetch the next record
      const uint32_t bytes = (uint32_t)(P.rec_off[next + 1] - P.rec_off[next]);
      mbar_expect_tx(&mbar[oth], bytes);
      bulk_g2s(rbuf[oth], P.rec + P.rec_off[next], bytes, &mbar[oth]);
    }
    const uint8_t* rec = rbuf[cur];
    gather_halo_gen<NL, DIM>(P, rec, hbuf);
    const int32_t* hdr = reinterpret_cast<const int32_t*>(rec);
    const int T = hdr[0], H = hdr[1], nv = hdr[2], nr = hdr[3], acc_n = P.values ? hdr[4] : 0;
    const uint32_t fmask = (uint32_t)hdr[5];
    const RecLayout L = rec_layout_hdr(NL, hdr);
    TileSmem D = S;  // domain view: everything from the record + the staged halo
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
    for (int i = tid; i < acc_n + KH * T; i += blockDim.x) acc[i] = 0.0;
    if (tid == 0) *ctr = 0;
    cp_async_wait_all();
    __syncthreads();
    if constexpr (DET) {
      const int32_t* run = reinterpret_cast<const int32_t*>(rec + L.o_run);
      for (int r = 0; r < nr; r++) {
        if (P.lean)
          for (int v = run[r] + warp; v < run[r + 1]; v += C::WARPS)
            warp_visit<ET, ORD, KH, Q, false, true>(P, P.dom, P.n_dom, D, v, slot);
        else
          for (int v = run[r] + warp; v < run[r + 1]; v += C::WARPS)
            warp_visit<ET, ORD, KH, Q, false, false>(P, P.dom, P.n_dom, D, v, slot);
        __syncthreads();
      }
    } else {
      if (P.lean)
        for (int v = grab_visits(ctr, 1); v < nv; v = grab_visits(ctr, 1))
          warp_visit<ET, ORD, KH, Q, false, true>(P, P.dom, P.n_dom, D, v, slot);
      else
        for (int v = grab_visits(ctr, 1); v < nv; v = grab_visits(ctr, 1))
          warp_visit<ET, ORD, KH, Q, false, false>(P, P.dom, P.n_dom, D, v, slot);
    }
    if (fmask) rec_facets<ET, ORD, KH, Q, C::WARPS, DET>(P, D, rec, L, slot);
    tile_epilogue<KH>(P, D);
    __syncthreads();
  }
}

template <int ET, int ORD, int KH, int Q, bool DET>
static int run_gen_rec(TiledParams& P, const TileSchedule& T, cudaStream_t s) {
  using C = TileCfg<ET, ORD, KH, Q>;
  constexpr int NL = C::NL, DIM = C::DIM;
  const size_t rec_dom = (P.lean ? sizeof(typename C::QPL) : sizeof(typename C::QPG)) * C::NQV;
  const size_t rec_fac = sizeof(typename C::QPG) * C::NQF;
  P.rec_bytes = (int)((std::max(rec_dom, rec_fac) + 15) / 16 * 16);
  int fv = 1;
  for (int f = 0; f < P.n_fac; f++) fv = std::max<int>(fv, (int)P.fvis[f].max_per_tile);
  P.fvmax = fv;
  P.vmax = fv;
  P.hmax = 0;
  P.hcomp = DIM + KH * (P.nu_hat >= 1 ? 2 : 1);
  P.rec = T.rec;
  P.rec_off = T.rec_off;
  P.n_tiles = T.n_tiles;
  P.rec_cap = (int)((T.rec_max + 15) / 16 * 16);
  P.hcap = (int)(((T.max_halo * P.hcomp) + 1) / 2 * 2);
  P.acc_cap = (int)((P.values ? T.acc_max : 0) + (int64_t)KH * T.max_tile_nodes);
  P.acc_cap = (P.acc_cap + 1) / 2 * 2;
  const size_t fac_bytes = (size_t)P.rec_bytes * C::WARPS + (size_t)fv * (4 + NL * 6 + 1) + 16;
  const size_t smem = 128 + 2 * (size_t)P.rec_cap + 8 * (size_t)P.hcap + 8 * (size_t)P.acc_cap + fac_bytes;
  if (smem > 227 * 1024) {
    set_error("record kernel: shared memory request too large (" + std::to_string(smem) + " B)");
    return FEM_E_UNSUPPORTED;
  }
  FEM_CUDA_TRY(cudaFuncSetAttribute(k_gen_rec<ET, ORD, KH, Q, DET>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  if (T.n_tiles <= 0) return 0;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t grid = std::min<int64_t>(T.n_tiles, sms);
  k_gen_rec<ET, ORD, KH, Q, DET><<<(unsigned)grid, TILED_THREADS, smem, s>>>(P);
  FEM_CUDA_TRY(cudaGetLastError());
  return 0;
}

template <int ET, int ORD, int KH, bool DET>
static int run_tiled_q(int q, TiledParams& P, const TileSchedule& T, cudaStream_t s) {
  if (!T.rec) {
    set_error("tiled: no tile records");
    return FEM_E_UNSUPPORTED;
  }
  if (q == 1) return run_gen_rec<ET, ORD, KH, 1, DET>(P, T, s);
  if (q == 2) return run_gen_rec<ET, ORD, KH, 2, DET>(P, T, s);
  if constexpr (ET == ET_HEX) {
    if (q == 3) return run_gen_rec<ET, ORD, KH, 3, DET>(P, T, s);
  }
  set_error("tiled: unsupported quadrature order");
  return FEM_E_UNSUPPORTED;
}

int launch_tiled(const fem_mesh_s* m, const fem_pattern_s* pat, const fem_problem* prob, const double* state,
                 double* values, double* rhs, bool det, cudaStream_t s) {
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
      P.fac_set[P.n_fac] = term.region;
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
  // det (FEM_SCATTER_TILED): bit-identical run to run — ordered per-row turns (hex, NS) or colour runs
  // (generic); !det (FEM_SCATTER_TILED_UNORDERED): shared-memory fp64 atomics where a kernel has them
  if (et == ET_HEX && o == 1 && q == 2) {
    bool handled = false;
    const int rc = launch_hex_tiled(P, T, kh, det, s, &handled);
    if (handled) return rc;
  }
  if (et == ET_TET && o == 1 && kh == 4 && q == 2) {
    bool handled = false;
    // ordered turns cost ~25% on c4 (24 elements per vertex: consecutive visits share rows)
    const int rc = launch_ns_tiled(P, T, det, s, &handled);
    if (handled) return rc;
  }
  if (et == ET_TET && o == 2 && kh == 3 && q == 2) {  // P2 elasticity (c3)
    bool handled = false;
    const int rc = launch_p2_tiled(P, T, det, s, &handled);
    if (handled) return rc;
  }
#define FEM_GEN(ET_, ORD_, KH_) \
  return det ? run_tiled_q<ET_, ORD_, KH_, true>(q, P, T, s) : run_tiled_q<ET_, ORD_, KH_, false>(q, P, T, s)
  if (et == ET_TRI && o == 1) {
    if (kh == 1) FEM_GEN(ET_TRI, 1, 1);
    if (kh == 2) FEM_GEN(ET_TRI, 1, 2);
  }
  if (et == ET_HEX && o == 1) {
    if (kh == 1) FEM_GEN(ET_HEX, 1, 1);
    if (kh == 3) FEM_GEN(ET_HEX, 1, 3);
  }
  if (et == ET_TET && o == 1) {
    if (kh == 1) FEM_GEN(ET_TET, 1, 1);
    if (kh == 3) FEM_GEN(ET_TET, 1, 3);
    if (kh == 4) FEM_GEN(ET_TET, 1, 4);
  }
  if (et == ET_TET && o == 2) {
    if (kh == 1) FEM_GEN(ET_TET, 2, 1);
    if (kh == 3) FEM_GEN(ET_TET, 2, 3);
  }
#undef FEM_GEN
  set_error("tiled: unsupported element/physics combination");
  return FEM_E_UNSUPPORTED;
}

}  // namespace fem
