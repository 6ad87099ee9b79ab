// sweep.cu — the z-sweep schedule of the Q1-hex owner-gather path (FEM_SCATTER_TILED on c5-like meshes).
//
// PAPER.md D-2/D-3 add every element's contribution into d and K.  The node-tile schedule of
// tiled.cu gives each CTA a 4x4x4 tile of control points and recomputes the ghost layer around it: 125
// element visits for 64 points, 1.95 visits per element on c5.  Here a CTA owns a COLUMN of the node
// lattice (CX x CY points in x/y, a chunk of planes in z) and sweeps it plane by plane:
//   step l visits the element layer l (between node planes l and l+1, plus the one-element ring around
//   the column in x/y), which contributes to the rows of planes l and l+1 of the column;
//   after step l plane l is complete (it has seen layers l-1 and l) and leaves to HBM, while plane l+1 is
//   carried to step l+1 in a shared-memory ring of two planes.
// Every element is visited once per column it touches: (CX+1)(CY+1)/(CX·CY) visits per element (1.36 for
// 6x6) plus one ghost layer per z-chunk.  Rows keep their ring position for their whole life, so the
// per-row turn counters of the ordered (deterministic) accumulation carry over between steps.
//
// The schedule applies to hexahedral meshes whose nodes sit on a lattice (structured, or perturbed by less
// than h/2 and renumbered at random — the c5 variants): lattice indices are recovered by rounding the
// coordinates on the mean element edge length per axis and validated element by element; any mesh that
// fails the check keeps the node-tile schedule.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <vector>

#include "tiled.cuh"

namespace fem {

// Local column offsets (slot - rowptr_s of the row's point) of every (visit, a, b), written into the records.
// Bit 7 marks the first contribution to the 3x3 block of this life of the ring row (the visit stores
// instead of adding, so no accumulator zeroing pass is needed): from the record's first-contribution masks.
__global__ void k_sweep_loc(uint8_t* __restrict__ rec, const int64_t* __restrict__ vis_loc_off,
                            const int64_t* __restrict__ vis_fst_off, const int32_t* __restrict__ vis_elem,
                            int64_t n_vis, const int32_t* __restrict__ slot, const int32_t* __restrict__ conn,
                            const int64_t* __restrict__ rowptr_s, int64_t E, int64_t lo, int64_t hi) {
  const int64_t total = n_vis * 64;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t v = t >> 6;
    const int ab = (int)(t & 63), a = ab >> 3;
    const int64_t e = vis_elem[v];
    const int64_t r = conn[(int64_t)a * E + e];
    uint8_t val = 255;
    if (r >= lo && r < hi) {
      val = (uint8_t)(slot[(int64_t)ab * E + e] - rowptr_s[r - lo]);
      const uint64_t fst = *reinterpret_cast<const uint64_t*>(rec + vis_fst_off[v]);
      if ((fst >> ab) & 1ull) val |= 0x80;
    }
    rec[vis_loc_off[v] + ab] = val;
  }
}

namespace {
// VTK hex corner a -> lattice offset (0/1 per axis): x - + + - - + + -, y - - + + - - + +, z - - - - + + + +
inline int corner_off(int a, int d) {
  if (d == 0) return ((a & 3) == 1 || (a & 3) == 2) ? 1 : 0;
  if (d == 1) return (a & 3) >= 2 ? 1 : 0;
  return a >= 4 ? 1 : 0;
}
}  // namespace

// Column footprint (points) per plane: the ring holds two planes of CX·CY rows in shared memory.
static void sweep_column_dims(int KH, int* cx, int* cy) {
  if (KH == 3) { *cx = 6; *cy = 6; }  // 2 x 36 rows x 3 x (81 + pad) doubles = 141 KB
  else { *cx = 12; *cy = 12; }
}
constexpr int SWEEP_CHUNK = 64;  // node planes per sequence (one ghost layer each): load balance over 148 SMs

int sweep_build(fem_mesh_s* m, fem_pattern_s* p, cudaStream_t s) {
  TileSchedule& T = p->tiles;
  const int NL = m->n_loc, KH = m->kh;
  if (m->etype != FEM_HEX || m->order != 1 || m->dim != 3 || KH != 3) return FEM_E_UNSUPPORTED;
  const int64_t E = m->E, N = m->N, lo = m->own_lo, hi = m->own_hi, n_own = m->n_own;
  if (n_own == 0 || E == 0) return FEM_E_UNSUPPORTED;
  const int32_t* conn = m->h_conn.data();
  const double* X = m->h_coords.data();
  // ---- 1. lattice indices: round on the mean element edge length per axis, validate every element
  double h[3] = {0, 0, 0}, xmin[3] = {1e300, 1e300, 1e300};
  const int edge_to[3] = {1, 3, 4};  // VTK edges (0,1) along ξ, (0,3) along η, (0,4) along ζ
  for (int64_t e = 0; e < E; e++)
    for (int d = 0; d < 3; d++) h[d] += std::fabs(X[d * N + conn[edge_to[d] * E + e]] - X[d * N + conn[e]]);
  for (int d = 0; d < 3; d++) {
    h[d] /= (double)E;
    if (!(h[d] > 0.0)) return FEM_E_UNSUPPORTED;
    for (int64_t i = 0; i < N; i++) xmin[d] = std::min(xmin[d], X[d * N + i]);
  }
  std::vector<int32_t> lat(3 * N);
  int64_t nlat[3] = {0, 0, 0};
  for (int d = 0; d < 3; d++)
    for (int64_t i = 0; i < N; i++) {
      const long long q = std::llround((X[d * N + i] - xmin[d]) / h[d]);
      if (q < 0 || q > (1 << 20)) return FEM_E_UNSUPPORTED;
      lat[3 * i + d] = (int32_t)q;
      nlat[d] = std::max<int64_t>(nlat[d], q + 1);
    }
  if (nlat[0] * nlat[1] * nlat[2] > ((int64_t)1 << 31)) return FEM_E_UNSUPPORTED;
  auto lid = [&](int64_t x, int64_t y, int64_t z) { return x + nlat[0] * (y + nlat[1] * z); };
  std::vector<int32_t> node_at(nlat[0] * nlat[1] * nlat[2], -1), elem_at(nlat[0] * nlat[1] * nlat[2], -1);
  for (int64_t i = 0; i < N; i++) {
    int32_t& slot = node_at[lid(lat[3 * i], lat[3 * i + 1], lat[3 * i + 2])];
    if (slot >= 0) return FEM_E_UNSUPPORTED;  // two points on one lattice site
    slot = (int32_t)i;
  }
  for (int64_t e = 0; e < E; e++) {
    const int32_t* b = &lat[3 * (int64_t)conn[e]];
    for (int a = 1; a < 8; a++)
      for (int d = 0; d < 3; d++)
        if (lat[3 * (int64_t)conn[a * E + e] + d] != b[d] + corner_off(a, d)) return FEM_E_UNSUPPORTED;
    int32_t& slot = elem_at[lid(b[0], b[1], b[2])];
    if (slot >= 0) return FEM_E_UNSUPPORTED;
    slot = (int32_t)e;
  }
  // lattice rank of every point: renumbered meshes stage their halo from lattice-ordered copies
  std::vector<int32_t> lpos(N), lperm;
  bool lat_ident = true;
  {
    int32_t k = 0;
    for (size_t q = 0; q < node_at.size(); q++)
      if (node_at[q] >= 0) lpos[node_at[q]] = k++;
    for (int64_t i = 0; i < N && lat_ident; i++) lat_ident = lpos[i] == i;
    if (!lat_ident) {
      lperm.resize(N);
      for (int64_t i = 0; i < N; i++) lperm[lpos[i]] = (int32_t)i;
    }
  }
  // ---- 2. pattern rows (degrees, row starts) and boundary facets per element
  std::vector<int64_t> rps(n_own + 1);
  FEM_CUDA_TRY(cudaMemcpyAsync(rps.data(), p->rowptr_s, sizeof(int64_t) * (n_own + 1), cudaMemcpyDeviceToHost, s));
  FEM_CUDA_TRY(cudaStreamSynchronize(s));
  for (int64_t i = 0; i < n_own; i++)
    if (rps[i + 1] - rps[i] > 255) return FEM_E_UNSUPPORTED;
  const int nb = (int)m->h_bset_elem.size();
  std::vector<std::vector<std::pair<int32_t, int8_t>>> efac(nb);  // per set: (element, face) sorted
  for (int k = 0; k < nb; k++) {
    for (size_t j = 0; j < m->h_bset_elem[k].size(); j++) efac[k].emplace_back(m->h_bset_elem[k][j], m->h_bset_facet[k][j]);
    std::sort(efac[k].begin(), efac[k].end());
  }
  int CX, CY;
  sweep_column_dims(KH, &CX, &CY);
  const int PMAX = CX * CY, TR = 2 * PMAX;  // ring rows
  // every ring position owns a fixed region (even size, one pad double for the 16-byte phase of its row's
  // destination): the lives of a position follow each other in turn order, but lives of DIFFERENT
  // positions are not ordered, so their rows must never share memory
  // fixed 27-column row layout (hex_visit_el2 SWSR): sub-row stride SR = 3·27 + (1 if nnz_s is even), so that
  // SR ≡ 3·nnz_s (mod 2) and every sub-row keeps the 16-byte phase of its destination
  const int SR = 81 + ((p->nnz_s & 1) ? 0 : 1);
  const int row_reg = (KH * SR + 2) / 2 * 2;
  const int64_t SLOT = (int64_t)PMAX * row_reg;  // doubles per ring plane
  // owned lattice range
  int64_t ob[3][2] = {{1 << 30, -1}, {1 << 30, -1}, {1 << 30, -1}};
  for (int64_t i = lo; i < hi; i++)
    for (int d = 0; d < 3; d++) {
      ob[d][0] = std::min<int64_t>(ob[d][0], lat[3 * i + d]);
      ob[d][1] = std::max<int64_t>(ob[d][1], lat[3 * i + d]);
    }
  const int64_t ncx = (ob[0][1] - ob[0][0]) / CX + 1, ncy = (ob[1][1] - ob[1][0]) / CY + 1;
  const int64_t nz_planes = ob[2][1] - ob[2][0] + 1;
  const int64_t nchunk = (nz_planes + SWEEP_CHUNK - 1) / SWEEP_CHUNK;
  const int64_t zc = (nz_planes + nchunk - 1) / nchunk;  // planes per chunk, evened out
  // ---- 3. steps of every sequence (column chunk)
  std::vector<int64_t> seq_off{0};
  std::vector<uint8_t> buf;
  std::vector<int64_t> roff{0};
  std::vector<int32_t> all_vis;       // visit elements in record order
  std::vector<int64_t> vis_loc;       // byte offset of each visit's local-column table
  std::vector<int64_t> vis_fst;       // byte offset of each visit's first-contribution mask
  int64_t rec_max = 0, max_halo = 0, max_vis = 0, max_fac = 0;
  int max_turns = 0;
  std::vector<int32_t> turn(TR, 0);
  std::vector<std::vector<int32_t>> seen_cols(TR);  // column points of the current life of each ring row
  std::vector<int32_t> row_first(n_own, -1), row_last(n_own, -1);  // step of the first / last touch (in its chunk)
  std::vector<int32_t> r_node(TR), r_deg(TR), r_off(TR);
  std::vector<int64_t> r_rps(TR);
  std::vector<int32_t> halo;
  std::vector<int32_t> vis;
  for (int64_t cyi = 0; cyi < ncy; cyi++)
    for (int64_t cxi = 0; cxi < ncx; cxi++)
      for (int64_t ch = 0; ch < nchunk; ch++) {
        const int64_t x0 = ob[0][0] + cxi * CX, x1 = std::min<int64_t>(x0 + CX, ob[0][1] + 1);
        const int64_t y0 = ob[1][0] + cyi * CY, y1 = std::min<int64_t>(y0 + CY, ob[1][1] + 1);
        const int64_t z0 = ob[2][0] + ch * zc, z1 = std::min<int64_t>(z0 + zc, ob[2][1] + 1);
        // owned point at (x, y, z) of this chunk, or -1
        auto own_at = [&](int64_t x, int64_t y, int64_t z) -> int32_t {
          if (x < x0 || x >= x1 || y < y0 || y >= y1 || z < z0 || z >= z1) return -1;
          const int32_t n = node_at[lid(x, y, z)];
          return (n >= lo && n < hi) ? n : -1;
        };
        auto rp_of = [&](int64_t x, int64_t y, int64_t z) { return (int)((z & 1) * PMAX + (x - x0) + CX * (y - y0)); };
        // layers: l = z0-1 .. z1-1 (element layer l joins planes l, l+1)
        int64_t first_step = -1, nsteps = 0;
        std::vector<std::vector<int32_t>> layer_vis;
        std::vector<int64_t> layers;
        for (int64_t l = z0 - 1; l <= z1 - 1; l++) {
          if (l < 0 || l + 1 >= nlat[2]) continue;
          vis.clear();
          for (int64_t j = y0 - 1; j < y1; j++)
            for (int64_t i = x0 - 1; i < x1; i++) {
              if (i < 0 || j < 0 || i + 1 >= nlat[0] || j + 1 >= nlat[1]) continue;
              const int32_t e = elem_at[lid(i, j, l)];
              if (e < 0) continue;
              bool touches = false;
              for (int a = 0; a < 8 && !touches; a++)
                touches = own_at(i + corner_off(a, 0), j + corner_off(a, 1), l + corner_off(a, 2)) >= 0;
              if (touches) vis.push_back(e);
            }
          if (vis.empty()) continue;
          if (first_step < 0) first_step = l;
          layer_vis.push_back(vis);
          layers.push_back(l);
          nsteps++;
        }
        if (nsteps == 0) continue;
        // first / last step touching each owned row (per point: ragged meshes may leave a row untouched by
        // some step that touches its plane)
        for (int64_t k = 0; k < nsteps; k++)
          for (int32_t e : layer_vis[k]) {
            const int32_t* b = &lat[3 * (int64_t)conn[e]];
            for (int a = 0; a < NL; a++) {
              const int32_t on = own_at(b[0] + corner_off(a, 0), b[1] + corner_off(a, 1), b[2] + corner_off(a, 2));
              if (on < 0) continue;
              if (row_first[on - lo] < 0) row_first[on - lo] = (int32_t)k;
              row_last[on - lo] = (int32_t)k;
            }
          }
        std::fill(turn.begin(), turn.end(), 0);
        for (int64_t k = 0; k < nsteps; k++) {
          const int64_t l = layers[k];
          std::vector<int32_t>& V = layer_vis[k];
          // visit order = turn order, sorted by the lattice parity class (i mod 2, j mod 2) of the element: the
          // four classes of a layer share no point, so the visits the consumer warps take at the same time
          // rarely wait for each other (measured: natural lattice order 2.6x slower, classes interleaved
          // 1.7x; the mesh's greedy colouring of a renumbered mesh has 17 colours and costs 1.45x)
          auto cls = [&](int32_t e) {
            const int32_t* bb = &lat[3 * (int64_t)conn[e]];
            return (bb[0] & 1) + 2 * (bb[1] & 1);
          };
          std::stable_sort(V.begin(), V.end(), [&](int32_t a, int32_t b) { return cls(a) < cls(b); });
          std::vector<int32_t> run{0};
          for (size_t v = 1; v < V.size(); v++)
            if (cls(V[v]) != cls(V[v - 1])) run.push_back((int32_t)v);
          run.push_back((int32_t)V.size());
          // rows of planes l, l+1 (ring positions), zero / write lists
          std::vector<int16_t> zrow, wrow;
          for (int64_t z = l; z <= l + 1; z++) {
            if (z < z0 || z >= z1) continue;
            for (int64_t y = y0; y < y1; y++)
              for (int64_t x = x0; x < x1; x++) {
                const int32_t n = own_at(x, y, z);
                if (n < 0) continue;
                const int rp = rp_of(x, y, z);
                const int64_t li = n - lo;
                r_node[rp] = n;
                r_rps[rp] = rps[li];
                r_deg[rp] = (int32_t)(rps[li + 1] - rps[li]);
                if (r_deg[rp] > 27) {
                  set_error("sweep schedule: a row has more than 27 scalar columns");
                  return FEM_E_UNSUPPORTED;
                }
                int64_t acc = (int64_t)rp * row_reg;                   // even: rp's fixed region
                if ((acc ^ (int64_t)((KH * rps[li]) & 1)) & 1) acc++;  // 16-byte phase of the destination row
                r_off[rp] = (int32_t)acc;
                if (row_first[li] == k) { zrow.push_back((int16_t)rp); seen_cols[rp].clear(); }
                if (row_last[li] == k) wrow.push_back((int16_t)rp);
              }
          }
          // halo points
          halo.clear();
          for (int32_t e : V)
            for (int a = 0; a < NL; a++) halo.push_back(conn[(int64_t)a * E + e]);
          std::sort(halo.begin(), halo.end());
          halo.erase(std::unique(halo.begin(), halo.end()), halo.end());
          // facets of the visited elements (sets < 5: 6 face bits each in the kernel's 32-bit mask)
          std::vector<int32_t> f_cnt{0};
          std::vector<int16_t> f_dv;
          std::vector<int8_t> f_fac;
          for (int kk = 0; kk < nb; kk++) {
            for (size_t v = 0; v < V.size(); v++) {
              auto it = std::lower_bound(efac[kk].begin(), efac[kk].end(), std::make_pair(V[v], (int8_t)-128));
              for (; it != efac[kk].end() && it->first == V[v]; ++it) {
                f_dv.push_back((int16_t)v);
                f_fac.push_back(it->second);
              }
            }
            f_cnt.push_back((int32_t)f_dv.size());
          }
          const int nv = (int)V.size(), H = (int)halo.size(), nf = (int)f_dv.size();
          const RecLayout L = rec_layout(NL, TR, H, nv, (int)run.size() - 1, nb, nf, 0, (int)zrow.size(),
                                         (int)wrow.size(), 1);
          const size_t base = buf.size();
          buf.resize(base + L.size, 0);
          uint8_t* r = buf.data() + base;
          int32_t* hdr = reinterpret_cast<int32_t*>(r);
          hdr[0] = TR; hdr[1] = H; hdr[2] = nv; hdr[3] = (int)run.size() - 1; hdr[4] = (int32_t)(2 * SLOT);
          hdr[5] = 0;
          for (int kk = 0; kk < nb && kk < 32; kk++)
            if (f_cnt[kk + 1] > f_cnt[kk]) hdr[5] |= 1 << kk;
          hdr[6] = nb; hdr[7] = nf; hdr[8] = 0; hdr[9] = (int32_t)zrow.size(); hdr[10] = (int32_t)wrow.size();
          hdr[11] = 1;
          int32_t* o_tnode = reinterpret_cast<int32_t*>(r + L.o_tnode);
          int32_t* o_tdeg = reinterpret_cast<int32_t*>(r + L.o_tdeg);
          int32_t* o_toff = reinterpret_cast<int32_t*>(r + L.o_toff);
          int64_t* o_trps = reinterpret_cast<int64_t*>(r + L.o_trps);
          for (int z = 0; z < 2; z++) {
            const int64_t zz = l + z;
            if (zz < z0 || zz >= z1) continue;
            for (int64_t y = y0; y < y1; y++)
              for (int64_t x = x0; x < x1; x++) {
                if (own_at(x, y, zz) < 0) continue;
                const int rp = rp_of(x, y, zz);
                o_tnode[rp] = r_node[rp]; o_tdeg[rp] = r_deg[rp]; o_toff[rp] = r_off[rp]; o_trps[rp] = r_rps[rp];
              }
          }
          o_toff[TR] = (int32_t)(2 * SLOT);
          if (lat_ident) {
            memcpy(r + L.o_hnode, halo.data(), sizeof(int32_t) * H);
          } else {
            int32_t* hn = reinterpret_cast<int32_t*>(r + L.o_hnode);
            for (int i = 0; i < H; i++) hn[i] = lpos[halo[i]];
          }
          memcpy(r + L.o_run, run.data(), sizeof(int32_t) * run.size());
          int32_t* o_velem = reinterpret_cast<int32_t*>(r + L.o_velem);
          uint16_t* o_vhal = reinterpret_cast<uint16_t*>(r + L.o_vhal);
          int16_t* o_vown = reinterpret_cast<int16_t*>(r + L.o_vown);
          uint8_t* o_vseq = r + L.o_vseq;
          uint16_t* o_vsw = reinterpret_cast<uint16_t*>(r + L.o_vsw);
          uint32_t* o_vfm = reinterpret_cast<uint32_t*>(r + L.o_vfm);
          uint64_t* o_vfst = reinterpret_cast<uint64_t*>(r + L.o_vfst);
          // the last visit of this step touching each row the step completes (its writer)
          std::vector<int> last_v(TR, -1);
          for (int v = 0; v < nv; v++) {
            const int32_t* b = &lat[3 * (int64_t)conn[V[v]]];
            for (int a = 0; a < NL; a++) {
              const int64_t xa = b[0] + corner_off(a, 0), ya = b[1] + corner_off(a, 1), za = b[2] + corner_off(a, 2);
              if (own_at(xa, ya, za) >= 0) last_v[rp_of(xa, ya, za)] = v;
            }
          }
          std::vector<uint8_t> is_w(TR, 0), is_z(TR, 0);
          for (int16_t rp : wrow) is_w[rp] = 1;
          for (int16_t rp : zrow) is_z[rp] = 1;
          std::vector<uint8_t> started(TR, 0);
          for (int v = 0; v < nv; v++) {
            const int32_t e = V[v];
            o_velem[v] = e;
            const int32_t* b = &lat[3 * (int64_t)conn[e]];
            uint64_t fst = 0;
            int16_t rps_v[8];
            for (int a = 0; a < NL; a++) {
              const int32_t node = conn[(int64_t)a * E + e];
              o_vhal[v * NL + a] = (uint16_t)(std::lower_bound(halo.begin(), halo.end(), node) - halo.begin());
              const int64_t xa = b[0] + corner_off(a, 0), ya = b[1] + corner_off(a, 1), za = b[2] + corner_off(a, 2);
              const int32_t on = own_at(xa, ya, za);
              rps_v[a] = -1;
              if (on >= 0) {
                const int rp = rp_of(xa, ya, za);
                rps_v[a] = (int16_t)rp;
                o_vown[v * NL + a] = (int16_t)rp;
                uint16_t w = (uint16_t)turn[rp]++;
                if (is_z[rp] && !started[rp]) { w |= 1u << 14; started[rp] = 1; }
                if (is_w[rp] && last_v[rp] == v) w |= 1u << 15;
                o_vsw[v * NL + a] = w;
                o_vseq[v * NL + a] = (uint8_t)std::min(turn[rp] - 1, 255);
                max_turns = std::max(max_turns, turn[rp]);
              } else {
                o_vown[v * NL + a] = -1;
                o_vseq[v * NL + a] = 0;
                o_vsw[v * NL + a] = 0;
              }
            }
            for (int a = 0; a < NL; a++) {  // first contribution of this life to block (row a, column point b)
              if (rps_v[a] < 0) continue;
              std::vector<int32_t>& sc = seen_cols[rps_v[a]];
              for (int bb = 0; bb < NL; bb++) {
                const int32_t col = conn[(int64_t)bb * E + e];
                if (std::find(sc.begin(), sc.end(), col) == sc.end()) {
                  sc.push_back(col);
                  fst |= 1ull << (a * 8 + bb);
                }
              }
            }
            o_vfst[v] = fst;
            uint32_t fm = 0;
            for (int kk = 0; kk < nb && kk < 5; kk++)
              for (int32_t i = f_cnt[kk]; i < f_cnt[kk + 1]; i++)
                if (f_dv[i] == v) fm |= 1u << (6 * kk + f_fac[i]);
            o_vfm[v] = fm;
            vis_loc.push_back((int64_t)base + L.o_vloc + (int64_t)v * NL * NL);
            vis_fst.push_back((int64_t)base + L.o_vfst + (int64_t)v * 8);
            all_vis.push_back(e);
          }
          if (nb > 0) {
            memcpy(r + L.o_fcnt, f_cnt.data(), sizeof(int32_t) * f_cnt.size());
            memcpy(r + L.o_fdv, f_dv.data(), sizeof(int16_t) * f_dv.size());
            memcpy(r + L.o_ffac, f_fac.data(), f_fac.size());
          }
          memcpy(r + L.o_zrow, zrow.data(), sizeof(int16_t) * zrow.size());
          memcpy(r + L.o_wrow, wrow.data(), sizeof(int16_t) * wrow.size());
          roff.push_back((int64_t)buf.size());
          rec_max = std::max<int64_t>(rec_max, L.size);
          max_halo = std::max<int64_t>(max_halo, H);
          max_vis = std::max<int64_t>(max_vis, nv);
          max_fac = std::max<int64_t>(max_fac, nf);
        }
        seq_off.push_back((int64_t)roff.size() - 1);
      }
  // every owned point must have been written exactly once
  {
    std::vector<uint8_t> seen(n_own, 0);
    for (size_t t = 0; t + 1 < roff.size(); t++) {
      const int32_t* hdr = reinterpret_cast<const int32_t*>(buf.data() + roff[t]);
      const RecLayout L = rec_layout_hdr(NL, hdr);
      const int16_t* w = reinterpret_cast<const int16_t*>(buf.data() + roff[t] + L.o_wrow);
      const int32_t* tn = reinterpret_cast<const int32_t*>(buf.data() + roff[t] + L.o_tnode);
      for (int i = 0; i < hdr[10]; i++) seen[tn[w[i]] - lo]++;
    }
    for (int64_t i = 0; i < n_own; i++)
      if (seen[i] != 1) { set_error("sweep schedule: an owned point is not written exactly once"); return FEM_E_UNSUPPORTED; }
  }
  if (max_vis > 255 || max_turns >= (1 << 14)) return FEM_E_UNSUPPORTED;
  // ---- 4. device copies
  const int64_t n_tiles = (int64_t)roff.size() - 1;
  T.sweep = true;
  T.sweep_sr = SR;
  T.n_tiles = n_tiles;
  T.n_seq = (int64_t)seq_off.size() - 1;
  T.max_tile_nodes = TR;
  T.acc_max = 2 * SLOT;
  T.max_halo = max_halo;
  T.rec_max = rec_max;
  T.rec_bytes_total = (int64_t)buf.size();
  T.max_turns = max_turns;
  T.visits_total = (int64_t)all_vis.size();
  T.dom.max_per_tile = max_vis;
  T.dom.n_visits = (int64_t)all_vis.size();
  T.bnd.assign(nb, VisitList());
  for (int kk = 0; kk < nb; kk++) T.bnd[kk].max_per_tile = max_fac;
  FEM_CUDA_TRY(cudaMalloc(&T.rec, buf.size() + 16));
  FEM_CUDA_TRY(cudaMalloc(&T.rec_off, sizeof(int64_t) * roff.size()));
  FEM_CUDA_TRY(cudaMalloc(&T.seq_off, sizeof(int64_t) * seq_off.size()));
  FEM_CUDA_TRY(cudaMemcpy(T.rec, buf.data(), buf.size(), cudaMemcpyHostToDevice));
  FEM_CUDA_TRY(cudaMemcpy(T.rec_off, roff.data(), sizeof(int64_t) * roff.size(), cudaMemcpyHostToDevice));
  FEM_CUDA_TRY(cudaMemcpy(T.seq_off, seq_off.data(), sizeof(int64_t) * seq_off.size(), cudaMemcpyHostToDevice));
  int32_t* d_vis = nullptr;
  int64_t *d_vloc = nullptr, *d_vfst = nullptr;
  FEM_CUDA_TRY(cudaMalloc(&d_vis, sizeof(int32_t) * (all_vis.size() + 1)));
  FEM_CUDA_TRY(cudaMalloc(&d_vloc, sizeof(int64_t) * (vis_loc.size() + 1)));
  FEM_CUDA_TRY(cudaMalloc(&d_vfst, sizeof(int64_t) * (vis_fst.size() + 1)));
  FEM_CUDA_TRY(cudaMemcpy(d_vis, all_vis.data(), sizeof(int32_t) * all_vis.size(), cudaMemcpyHostToDevice));
  FEM_CUDA_TRY(cudaMemcpy(d_vloc, vis_loc.data(), sizeof(int64_t) * vis_loc.size(), cudaMemcpyHostToDevice));
  FEM_CUDA_TRY(cudaMemcpy(d_vfst, vis_fst.data(), sizeof(int64_t) * vis_fst.size(), cudaMemcpyHostToDevice));
  const int64_t tot = (int64_t)all_vis.size() * 64;
  if (tot > 0) {
    const int64_t blocks = std::min<int64_t>((tot + 255) / 256, 148 * 32);
    k_sweep_loc<<<(unsigned)blocks, 256, 0, s>>>(T.rec, d_vloc, d_vfst, d_vis, (int64_t)all_vis.size(), p->slot,
                                                 m->conn, p->rowptr_s, E, lo, hi);
    FEM_CUDA_TRY(cudaGetLastError());
  }
  if (!lat_ident) {  // lattice-ordered copies: coordinates once, the state buffer for the per-call gather
    T.sw_pstate_comps = 2 * KH;  // d (and ḋ with ν̂ >= 1)
    FEM_CUDA_TRY(cudaMalloc(&T.sw_lperm, sizeof(int32_t) * N));
    FEM_CUDA_TRY(cudaMalloc(&T.sw_pcoords, sizeof(double) * 3 * N));
    FEM_CUDA_TRY(cudaMalloc(&T.sw_pstate, sizeof(double) * T.sw_pstate_comps * N));
    FEM_CUDA_TRY(cudaMemcpy(T.sw_lperm, lperm.data(), sizeof(int32_t) * N, cudaMemcpyHostToDevice));
    const int rc = perm_gather(m->coords, T.sw_pcoords, T.sw_lperm, N, 3, s);
    if (rc) return rc;
  }
  FEM_CUDA_TRY(cudaStreamSynchronize(s));
  cudaFree(d_vis);
  cudaFree(d_vloc);
  cudaFree(d_vfst);
  return 0;
}

// dst[c][k] = src[c][perm[k]] for c < ncomp (component-major arrays of n points)
__global__ void k_perm_gather(const double* __restrict__ src, double* __restrict__ dst, const int32_t* __restrict__ perm,
                              int64_t n, int ncomp) {
  const int64_t tot = n * ncomp;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < tot; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = t / n, k = t - c * n;
    dst[t] = __ldg(src + c * n + __ldg(perm + k));
  }
}
int perm_gather(const double* src, double* dst, const int32_t* perm, int64_t n, int ncomp, cudaStream_t s) {
  const int64_t tot = n * ncomp;
  if (tot <= 0) return 0;
  const int64_t blocks = std::min<int64_t>((tot + 255) / 256, 148 * 64);
  k_perm_gather<<<(unsigned)blocks, 256, 0, s>>>(src, dst, perm, n, ncomp);
  FEM_CUDA_TRY(cudaGetLastError());
  return 0;
}

}  // namespace fem
