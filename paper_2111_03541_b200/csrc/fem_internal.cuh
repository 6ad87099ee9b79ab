// fem_internal.cuh — library-internal structures shared by the host driver and the kernels.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <vector>

#include "../../include/libfem.h"
#include "physics.cuh"

namespace fem {

void set_error(const std::string& msg);

#define FEM_CUDA_TRY(call)                                                                   \
  do {                                                                                       \
    cudaError_t e_ = (call);                                                                 \
    if (e_ != cudaSuccess) {                                                                 \
      ::fem::set_error(std::string("CUDA error ") + cudaGetErrorString(e_) + " at " +       \
                       __FILE__ + ":" + std::to_string(__LINE__) + ": " #call);              \
      return e_ == cudaErrorMemoryAllocation ? FEM_E_OOM : FEM_E_CUDA;                       \
    }                                                                                        \
  } while (0)

// A list of assembly tasks: elements (domain terms) or (element, facet) pairs (boundary terms),
// grouped by colour: tasks [col_off[c], col_off[c+1]) share no control point.
struct TaskList {
  int64_t n = 0;
  int32_t* elem = nullptr;  // device
  int8_t* facet = nullptr;  // device (boundary sets only)
  std::vector<int64_t> col_off;  // host, size n_colours+1
};

// Visits of one tile schedule: for tile t, runs [roff[t], roff[t+1]); run r covers visits
// [run[r], run[r+1]) which all have the same colour (no two share a control point).
struct VisitList {
  int64_t n_runs = 0, n_visits = 0, max_per_tile = 0;
  int64_t* roff = nullptr;   // device [n_tiles+1]
  int64_t* run = nullptr;    // device [n_runs+1]
  int32_t* elem = nullptr;   // device [n_visits]
  int8_t* facet = nullptr;   // device [n_visits] (boundary sets only)
};

// Node-tile schedule (FEM_SCATTER_TILED): owned points split into spatially compact tiles whose
// rows fit the shared-memory accumulator; each tile visits every element touching it.
struct TileSchedule {
  int64_t n_tiles = 0;
  int max_tile_nodes = 0;
  int64_t acc_max = 0;           // largest accumulator (doubles) of any tile
  int64_t* tile_noff = nullptr;  // device [n_tiles+1] offsets into tile_node
  int32_t* tile_node = nullptr;  // device: owned points of each tile (ascending)
  VisitList dom;                 // element visits
  std::vector<VisitList> bnd;    // facet visits per boundary set
  uint8_t* loc = nullptr;        // device [E][n_loc][n_loc]: slot - rowptr_s[α(e,a)] (255: not owned)
  int64_t visits_total = 0;
  int64_t* halo_off = nullptr;   // device [n_tiles+1]: points of the elements a tile visits
  int32_t* halo_node = nullptr;  // device: sorted per tile
  int64_t max_halo = 0;
  uint8_t* rec = nullptr;        // device: packed per-tile records (layout rec_layout)
  int64_t* rec_off = nullptr;    // device [n_tiles+1] byte offsets
  int64_t rec_max = 0, rec_bytes_total = 0;
  int max_turns = 0;              // most visits of one tile touching one owned point (ordered kernels need <= 255)
  // z-sweep schedule (hex meshes on a lattice, sweep.cu): records are the steps of sequences; a CTA walks
  // one sequence (a column chunk) step by step, carrying accumulator rows in a ring of two node planes.
  // Row tables of a step record are indexed by ring position; zrow/wrow list the rows to zero at the
  // step's start and to write at its end.  Plain node tiles are sequences of one record.
  bool sweep = false;
  int sweep_sr = 0;                // ring sub-row stride (81 or 82: fixed 27-column layout, parity of 3·nnz_s)
  int64_t n_seq = 0;
  int64_t* seq_off = nullptr;     // device [n_seq+1]: records of sequence q are [seq_off[q], seq_off[q+1])
  // renumbered meshes (points not in lattice order): the sweep stages its halo from copies of the point data
  // in lattice order, so the gathers of a step are contiguous; sw_lperm[k] = the point at lattice rank k,
  // sw_pcoords = coordinates in that order (built once), sw_pstate = the state, permuted per call
  int32_t* sw_lperm = nullptr;
  double* sw_pcoords = nullptr;
  double* sw_pstate = nullptr;
  int sw_pstate_comps = 0;
};

// Packed per-tile record: header int32 {T, H, nv, nruns, acc_n, fac_mask, 0, 0} followed by
// 16-byte aligned sections (see rec_layout).  Built on the host at pattern time (loc on the device).
struct RecLayout {
  int o_tnode, o_tdeg, o_toff, o_trps, o_hnode, o_run, o_velem, o_vhal, o_vown, o_vloc, o_vseq, o_fcnt, o_fdv, o_ffac,
      o_fseg, o_zrow, o_wrow, o_vsw, o_vfm, o_vfst, size;
};
// header[6] = number of boundary sets nb, header[7] = facet visits nf; facet visit i of set k
// (fcnt[k] <= i < fcnt[k+1]) is facet ffac[i] of the tile's domain visit fdv[i].
// vseq[v][a] = number of earlier visits of the record that touch node a (u8, saturating at 255): the
// turn of visit v on the accumulator row of a in the ordered deterministic kernels.
// header[8] = facet segments ns: fseg = int32 [nb+1] first segment of each set, then int32 [ns+1]
// segment starts; the facets of one segment belong to distinct elements of one colour (node-disjoint),
// so a deterministic kernel may run a segment's facets concurrently with plain adds.
__host__ __device__ inline RecLayout rec_layout(int NL, int T, int H, int nv, int nruns, int nb = 0, int nf = 0,
                                                int ns = 0, int nzr = 0, int nwr = 0, int sweep = 0) {
  RecLayout L;
  int o = 48;
  auto al = [](int x) { return (x + 15) & ~15; };
  L.o_tnode = o; o = al(o + 4 * T);
  L.o_tdeg = o;  o = al(o + 4 * T);
  L.o_toff = o;  o = al(o + 4 * (T + 1));
  L.o_trps = o;  o = al(o + 8 * T);
  L.o_hnode = o; o = al(o + 4 * H);
  L.o_run = o;   o = al(o + 4 * (nruns + 1));
  L.o_velem = o; o = al(o + 4 * nv);
  L.o_vhal = o;  o = al(o + 2 * nv * NL);
  L.o_vown = o;  o = al(o + 2 * nv * NL);
  L.o_vloc = o;  o = al(o + nv * NL * NL);
  L.o_vseq = o;  o = al(o + nv * NL);
  L.o_fcnt = o;  o = al(o + 4 * (nb + 1));
  L.o_fdv = o;   o = al(o + 2 * nf);
  L.o_ffac = o;  o = al(o + nf);
  L.o_fseg = o;  o = al(o + 4 * (nb + 1) + 4 * (ns + 1));
  L.o_zrow = o;  o = al(o + 2 * nzr);
  L.o_wrow = o;  o = al(o + 2 * nwr);
  // sweep records (header[11] = 1): per (visit, node) uint16 turn | first-touch << 14 | last-touch << 15,
  // per visit the 32-bit boundary-face mask (6 bits per set) and the 64-bit first-contribution mask (a, b)
  L.o_vsw = o;   o = al(o + (sweep ? 2 * nv * NL : 0));
  L.o_vfm = o;   o = al(o + (sweep ? 4 * nv : 0));
  L.o_vfst = o;  o = al(o + (sweep ? 8 * nv : 0));
  L.size = o;
  return L;
}
// Accumulator row stride of a tile point with d block columns: entry (i, m, col) of its KH x KH blocks
// sits at toff + i*stride + m*d + col.  One pad double when needed makes stride ≡ KH*nnz_s (mod 2), so
// that with toff ≡ KH*rowptr_s (mod 2) every row segment has the 16-byte phase of its destination in
// `values` and can leave by one bulk (TMA) store.
__host__ __device__ inline int acc_row_stride(int KH, int d, int64_t nnz_s) {
  return KH == 1 ? d : KH * d + ((KH * (d + (int)(nnz_s & 1))) & 1);
}
// header[9] / [10] = number of zrow / wrow entries (sweep steps; 0 for plain tiles)
__host__ __device__ inline RecLayout rec_layout_hdr(int NL, const int32_t* h) {
  return rec_layout(NL, h[0], h[1], h[2], h[3], h[6], h[7], h[8], h[9], h[10], h[11]);
}

}  // namespace fem

struct fem_mesh_s {
  int dim = 0, etype = 0, order = 0, physics = 0, n_loc = 0, kh = 0;
  int64_t N = 0, E = 0, own_lo = 0, own_hi = 0, n_own = 0;
  double* coords = nullptr;  // device [dim][N]
  int32_t* conn = nullptr;   // device [n_loc][E]
  fem::TaskList dom;         // element tasks, coloured
  std::vector<fem::TaskList> bnd;  // boundary set tasks, coloured
  std::vector<int64_t> bset_len;
  std::vector<int32_t*> bset_elem_dev;  // original order (device)
  std::vector<int8_t*> bset_facet_dev;
  // host copies kept for the tile schedule (built at pattern time, needs row degrees)
  std::vector<int32_t> h_conn;
  std::vector<double> h_coords;
  std::vector<uint8_t> h_colour;
  std::vector<std::vector<int32_t>> h_bset_elem;
  std::vector<std::vector<int8_t>> h_bset_facet;
  std::vector<std::vector<uint8_t>> h_bset_colour;
  long long* err = nullptr;     // device error word: an offending element id or -1
  // fixed-order residual norms: per-block partials (Σd², max|d|) + the last-block ticket; sized for
  // norm_blocks = 4 × the device's SM count (queried at create), so the reduction order is fixed per device
  double* norm_partials = nullptr;
  unsigned int* norm_ticket = nullptr;
  int norm_blocks = 0;
  double* scratch_state = nullptr;  // e2e staging buffer (lazily allocated)
  size_t scratch_state_bytes = 0;
  // pipelined e2e (fem_linearize_host_async): two staging buffers, a copy stream and their events
  double* async_state[2] = {nullptr, nullptr};
  size_t async_bytes = 0;
  cudaStream_t copy_stream = nullptr;
  cudaEvent_t ev_copied[2] = {nullptr, nullptr}, ev_used[2] = {nullptr, nullptr};
  int64_t async_calls = 0;
  int n_colours = 0;
  int64_t last_n_tiles = 0;
};

struct fem_pattern_s {
  fem_mesh_s* mesh = nullptr;
  fem::TileSchedule tiles;
  int64_t n_rows = 0, nnz = 0, nnz_s = 0;
  int64_t* rowptr_s = nullptr;  // device [n_own+1]
  int32_t* colidx_s = nullptr;  // device [nnz_s]
  int32_t* slot = nullptr;      // device [n_loc²][E]
  int64_t* rowptr = nullptr;    // device [n_rows+1]
  int32_t* colidx = nullptr;    // device [nnz]
  int tiles_rc = 0;             // != 0: no tile schedule for this mesh (tiled calls return it)
  std::string tiles_msg;
  // FEM_SCATTER_STORED (stored.cu, fem_pattern_stored_prepare).  Elements are stored in the Morton order of
  // their centroids (position pos, eperm[pos] = e, epos[e] = pos).  Per scalar slot s its contributions
  // (pos, a, b) at ent[off[s] .. off[s+1]), encoded (pos·NB + blk) << 1 | transposed; per owned row its
  // residual contributions pos·NL + a at rent[roff[li] .. roff[li+1]).
  uint32_t* st_ent = nullptr;
  uint32_t* st_off = nullptr;
  uint32_t* st_rent = nullptr;
  uint32_t* st_roff = nullptr;
  int32_t* st_epos = nullptr;
  int32_t* st_eperm = nullptr;
  int32_t* st_rows = nullptr;  // owned rows in gather order (Morton order of their points)
  double* st_ek = nullptr;     // [E][NB][KH][KH] (only with with_matrix)
  double* st_er = nullptr;     // [E][NL][KH]
  int64_t st_n_ent = 0;
  int st_nb = 0;               // blocks stored per element: NL(NL+1)/2 (symmetric physics, a <= b) or NL²
  // boundary sets re-grouped for the stored mode: facets only conflict when they belong to the same element
  // (each element owns its storage), so group g of a set holds each element's g-th facet (≤ 6 groups)
  std::vector<fem::TaskList> st_bnd;
  double* st_xaos = nullptr;   // P1-tet NS: node-major coordinates / state (32 bytes per point) for k_ns_el
  double* st_saos = nullptr;
};

namespace fem {

// Arguments of one assembly launch.
struct AsmArgs {
  const fem_mesh_s* m;
  const fem_pattern_s* pat;  // may be null for residual-only
  FormArgs F;
  int quad_order;
  const double* state;
  double* values;  // null: no matrix
  double* rhs;     // null: no residual
  int plain;       // 1: plain RMW (coloured), 0: atomics
  const int32_t* task_elem;  // null: identity 0..n-1
  const int8_t* task_facet;  // null for domain terms
  int64_t task_begin, task_count;
  cudaStream_t stream;
  double* ek = nullptr;  // FEM_SCATTER_STORED element blocks / residuals (stored.cu); values/rhs unused then
  double* er = nullptr;
  int ek_add = 0;
  const int32_t* ek_map = nullptr;  // element -> storage index (null: identity)
};

int launch_generic(const AsmArgs& A, bool facet);
// FEM_SCATTER_STORED: element pass into the pattern's element scratch, then the per-slot gathers (stored.cu)
int launch_stored(const fem_mesh_s* m, const fem_pattern_s* p, const fem_problem* prob, const double* state,
                  double* values, double* rhs, cudaStream_t s);
void stored_free(fem_pattern_s* p);
// quadratic-cube elasticity domain term on the fp64 tensor cores (hex2_el.cu); *handled = 0: not applicable
int launch_q2_elast(const AsmArgs& A, int* handled);
// z-sweep schedule for Q1-hex elasticity on lattice meshes (sweep.cu); FEM_E_UNSUPPORTED: not applicable
int sweep_build(fem_mesh_s* m, fem_pattern_s* p, cudaStream_t s);
// dst[c][k] = src[c][perm[k]] (sweep.cu)
int perm_gather(const double* src, double* dst, const int32_t* perm, int64_t n, int ncomp, cudaStream_t s);
int launch_tiled(const fem_mesh_s* m, const fem_pattern_s* pat, const fem_problem* prob,
                 const double* state, double* values, double* rhs, bool det, cudaStream_t stream);
int pattern_build(fem_mesh_s* m, cudaStream_t stream, fem_pattern_s* p);
int tiles_build(fem_mesh_s* m, fem_pattern_s* p, cudaStream_t stream);
void tiles_free(TileSchedule& T);
int residual_norms(const fem_mesh_s* m, const double* rhs, double* norms, cudaStream_t stream);
FormArgs make_form_args(const fem_problem* prob, const fem_term& t);

}  // namespace fem
