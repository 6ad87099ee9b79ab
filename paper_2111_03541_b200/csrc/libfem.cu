// libfem.cu — host side of the C ABI (include/libfem.h): validation, device copies, element
// colouring, node-tile schedule, dispatch of the assembly kernels.  PAPER.md Blocks B and D
// (P:343-465); readings in DESIGN.md §4.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <string>
#include <vector>

#include "fem_internal.cuh"

namespace fem {

static thread_local std::string g_last_error;
void set_error(const std::string& msg) { g_last_error = msg; }

static int n_loc_of(int et, int order) {
  if (et == FEM_TRI && order == 1) return 3;
  if (et == FEM_TET && order == 1) return 4;
  if (et == FEM_TET && order == 2) return 10;
  if (et == FEM_HEX && order == 1) return 8;
  if (et == FEM_HEX && order == 2) return 27;              // Lagrange cube of order 2 (NEXT-2)
  if (et == FEM_HEX_SERENDIPITY && order == 2) return 20;  // serendipity cube of order 2
  return -1;
}

static int kappa_hat_of(int physics, int dim) {
  if (physics == FEM_THERMAL) return 1;
  if (physics == FEM_ELASTICITY) return dim;
  if (physics == FEM_NS) return dim + 1;
  return -1;
}

static bool form_in_physics(int physics, int form) {
  if (physics == FEM_THERMAL) return form >= FEM_WF_THERMAL_DOMAIN && form <= FEM_WF_THERMAL_FIX;
  if (physics == FEM_ELASTICITY) return form >= FEM_WF_ELAST_DOMAIN && form <= FEM_WF_ELAST_LOAD;
  if (physics == FEM_NS) return form >= FEM_WF_NS_DOMAIN && form <= FEM_WF_NS_BND_FIX;
  return false;
}

FormArgs make_form_args(const fem_problem* prob, const fem_term& t) {
  FormArgs F;
  F.form = t.form;
  const bool ga = prob->time.kind == FEM_TIME_GENALPHA;
  F.nu_hat = ga ? prob->time.nu_hat : 0;
  // Eq. gen_alpha: f_0 = c1, f_1 = c2 / (b1 Δt); static: f_0 = 1 (reading L12)
  F.f0 = ga ? prob->time.c1 : 1.0;
  F.f1 = ga ? prob->time.c2 / (prob->time.b1 * prob->time.dt) : 0.0;
  for (int i = 0; i < FEM_MAX_PARAMS; i++) F.p[i] = t.params[i];
  F.lam = F.mu = 0.0;
  if (t.form == FEM_WF_ELAST_DOMAIN) {
    const double E = t.params[0], nu = t.params[1];
    F.lam = E * nu / ((1.0 + nu) * (1.0 - 2.0 * nu));
    F.mu = E / (2.0 * (1.0 + nu));
  }
  return F;
}

// Greedy colouring: item i touches control points nodes(i); colours so that no two items of a colour
// share a point.  Returns the permutation sorted by colour and the colour offsets.
template <class NodesOf>
static int greedy_colour(int64_t n_items, int64_t n_nodes, int nl, NodesOf nodes_of, std::vector<int32_t>& order,
                         std::vector<int64_t>& off) {
  std::vector<uint64_t> used(n_nodes, 0);
  std::vector<uint8_t> col(n_items);
  int ncol = 0;
  for (int64_t i = 0; i < n_items; i++) {
    uint64_t m = 0;
    for (int a = 0; a < nl; a++) m |= used[nodes_of(i, a)];
    if (m == ~0ull) return -1;
    int c = __builtin_ctzll(~m);
    col[i] = (uint8_t)c;
    ncol = std::max(ncol, c + 1);
    for (int a = 0; a < nl; a++) used[nodes_of(i, a)] |= (1ull << c);
  }
  off.assign(ncol + 1, 0);
  for (int64_t i = 0; i < n_items; i++) off[col[i] + 1]++;
  for (int c = 0; c < ncol; c++) off[c + 1] += off[c];
  std::vector<int64_t> pos(off.begin(), off.end() - 1);
  order.resize(n_items);
  for (int64_t i = 0; i < n_items; i++) order[pos[col[i]]++] = (int32_t)i;
  return ncol;
}

}  // namespace fem

using namespace fem;

extern "C" {

const char* fem_last_error(void) { return g_last_error.c_str(); }
int fem_version(void) { return 1; }

static void free_tasks(TaskList& t) {
  if (t.elem) cudaFree(t.elem);
  if (t.facet) cudaFree(t.facet);
  t.elem = nullptr;
  t.facet = nullptr;
}

void fem_mesh_destroy(fem_mesh_t m) {
  if (!m) return;
  cudaFree(m->coords);
  cudaFree(m->conn);
  free_tasks(m->dom);
  for (auto& t : m->bnd) free_tasks(t);
  for (auto p : m->bset_elem_dev) cudaFree(p);
  for (auto p : m->bset_facet_dev) cudaFree(p);
  cudaFree(m->err);
  cudaFree(m->norm_partials);
  cudaFree(m->norm_ticket);
  if (m->scratch_state) cudaFree(m->scratch_state);
  for (int b = 0; b < 2; b++) {
    if (m->async_state[b]) cudaFree(m->async_state[b]);
    if (m->ev_copied[b]) cudaEventDestroy(m->ev_copied[b]);
    if (m->ev_used[b]) cudaEventDestroy(m->ev_used[b]);
  }
  if (m->copy_stream) cudaStreamDestroy(m->copy_stream);
  delete m;
}

int fem_mesh_create(const fem_problem* prob, int dim, int64_t n_nodes, const double* coords, int64_t n_elems,
                    const int32_t* conn, int n_bsets, const int64_t* bset_len, const int32_t* const* bset_elem,
                    const int8_t* const* bset_facet, int64_t own_lo, int64_t own_hi, void* stream,
                    fem_mesh_t* out) {
  if (!out) { set_error("fem_mesh_create: out is NULL"); return FEM_E_INVALID_ARG; }
  *out = nullptr;
  if (!prob || !coords || !conn || n_nodes <= 0 || n_elems < 0 || (dim != 2 && dim != 3) || n_bsets < 0 ||
      (n_bsets > 0 && (!bset_len || !bset_elem || !bset_facet))) {
    set_error("fem_mesh_create: invalid argument");
    return FEM_E_INVALID_ARG;
  }
  const int nl = n_loc_of(prob->etype, prob->order);
  const int kh = kappa_hat_of(prob->physics, dim);
  if (nl < 0 || kh < 0 || (prob->etype == FEM_TRI) != (dim == 2) || (prob->physics == FEM_NS && dim != 3)) {
    set_error("fem_mesh_create: unsupported element/order/physics/dimension combination");
    return FEM_E_UNSUPPORTED;
  }
  if (own_lo < 0 || own_hi > n_nodes || own_lo > own_hi) {
    set_error("fem_mesh_create: owned range outside [0, n_nodes]");
    return FEM_E_INVALID_ARG;
  }
  if (n_nodes >= ((int64_t)1 << 31) || n_elems >= ((int64_t)1 << 31)) {
    set_error("fem_mesh_create: node/element ids must fit int32");
    return FEM_E_INDEX_OVERFLOW;
  }
  for (int64_t i = 0; i < (int64_t)nl * n_elems; i++)
    if (conn[i] < 0 || conn[i] >= n_nodes) {
      set_error("fem_mesh_create: connectivity entry out of range");
      return FEM_E_INVALID_ARG;
    }
  const int nfac = prob->etype == FEM_TRI ? 3 : (prob->etype == FEM_TET ? 4 : 6);
  for (int k = 0; k < n_bsets; k++)
    for (int64_t j = 0; j < bset_len[k]; j++)
      if (bset_elem[k][j] < 0 || bset_elem[k][j] >= n_elems || bset_facet[k][j] < 0 || bset_facet[k][j] >= nfac) {
        set_error("fem_mesh_create: boundary facet entry out of range");
        return FEM_E_INVALID_ARG;
      }
  cudaStream_t s = (cudaStream_t)stream;
  fem_mesh_s* m = new fem_mesh_s();
  m->dim = dim; m->etype = prob->etype; m->order = prob->order; m->physics = prob->physics;
  m->n_loc = nl; m->kh = kh; m->N = n_nodes; m->E = n_elems;
  m->own_lo = own_lo; m->own_hi = own_hi; m->n_own = own_hi - own_lo;
  auto fail = [&](int code) { fem_mesh_destroy(m); return code; };
#define MTRY(call)                         \
  do {                                     \
    cudaError_t e_ = (call);               \
    if (e_ != cudaSuccess) {               \
      set_error(std::string("fem_mesh_create: ") + cudaGetErrorString(e_)); \
      return fail(e_ == cudaErrorMemoryAllocation ? FEM_E_OOM : FEM_E_CUDA); \
    }                                      \
  } while (0)
  MTRY(cudaMalloc(&m->coords, sizeof(double) * dim * n_nodes));
  MTRY(cudaMalloc(&m->conn, sizeof(int32_t) * nl * (n_elems > 0 ? n_elems : 1)));
  MTRY(cudaMalloc(&m->err, sizeof(long long)));
  {
    int dev = 0, sms = 0;
    MTRY(cudaGetDevice(&dev));
    MTRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    m->norm_blocks = 4 * (sms > 0 ? sms : 1);
  }
  MTRY(cudaMalloc(&m->norm_partials, sizeof(double) * 2 * m->norm_blocks));
  MTRY(cudaMalloc(&m->norm_ticket, sizeof(unsigned int)));
  MTRY(cudaMemsetAsync(m->norm_ticket, 0, sizeof(unsigned int), s));
  MTRY(cudaMemcpyAsync(m->coords, coords, sizeof(double) * dim * n_nodes, cudaMemcpyHostToDevice, s));
  if (n_elems > 0) MTRY(cudaMemcpyAsync(m->conn, conn, sizeof(int32_t) * nl * n_elems, cudaMemcpyHostToDevice, s));
  MTRY(cudaMemsetAsync(m->err, 0xff, sizeof(long long), s));
  // deterministic element colouring (domain terms)
  {
    std::vector<int32_t> order;
    int nc = greedy_colour(n_elems, n_nodes, nl, [&](int64_t e, int a) { return conn[(int64_t)a * n_elems + e]; },
                           order, m->dom.col_off);
    if (nc < 0) { set_error("fem_mesh_create: colouring needs more than 64 colours"); return fail(FEM_E_UNSUPPORTED); }
    m->n_colours = nc;
    m->h_colour.resize(n_elems);
    for (int c = 0; c < nc; c++)
      for (int64_t j = m->dom.col_off[c]; j < m->dom.col_off[c + 1]; j++) m->h_colour[order[j]] = (uint8_t)c;
    m->h_conn.assign(conn, conn + (int64_t)nl * n_elems);
    m->h_coords.assign(coords, coords + (int64_t)dim * n_nodes);
    m->dom.n = n_elems;
    MTRY(cudaMalloc(&m->dom.elem, sizeof(int32_t) * (n_elems > 0 ? n_elems : 1)));
    if (n_elems > 0) MTRY(cudaMemcpyAsync(m->dom.elem, order.data(), sizeof(int32_t) * n_elems, cudaMemcpyHostToDevice, s));
    MTRY(cudaStreamSynchronize(s));
  }
  // boundary sets: original order + coloured task lists
  m->bnd.resize(n_bsets);
  for (int k = 0; k < n_bsets; k++) {
    const int64_t L = bset_len[k];
    m->bset_len.push_back(L);
    int32_t* de = nullptr;
    int8_t* df = nullptr;
    MTRY(cudaMalloc(&de, sizeof(int32_t) * (L > 0 ? L : 1)));
    MTRY(cudaMalloc(&df, sizeof(int8_t) * (L > 0 ? L : 1)));
    m->bset_elem_dev.push_back(de);
    m->bset_facet_dev.push_back(df);
    if (L > 0) {
      MTRY(cudaMemcpyAsync(de, bset_elem[k], sizeof(int32_t) * L, cudaMemcpyHostToDevice, s));
      MTRY(cudaMemcpyAsync(df, bset_facet[k], sizeof(int8_t) * L, cudaMemcpyHostToDevice, s));
    }
    std::vector<int32_t> order;
    TaskList& T = m->bnd[k];
    int nc = greedy_colour(L, n_nodes, nl, [&](int64_t j, int a) { return conn[(int64_t)a * n_elems + bset_elem[k][j]]; },
                           order, T.col_off);
    if (nc < 0) { set_error("fem_mesh_create: facet colouring needs more than 64 colours"); return fail(FEM_E_UNSUPPORTED); }
    m->h_bset_elem.emplace_back(bset_elem[k], bset_elem[k] + L);
    m->h_bset_facet.emplace_back(bset_facet[k], bset_facet[k] + L);
    m->h_bset_colour.emplace_back(L);
    for (int c = 0; c + 1 < (int)T.col_off.size(); c++)
      for (int64_t j = T.col_off[c]; j < T.col_off[c + 1]; j++) m->h_bset_colour[k][order[j]] = (uint8_t)c;
    std::vector<int32_t> te(L);
    std::vector<int8_t> tf(L);
    for (int64_t j = 0; j < L; j++) { te[j] = bset_elem[k][order[j]]; tf[j] = bset_facet[k][order[j]]; }
    T.n = L;
    MTRY(cudaMalloc(&T.elem, sizeof(int32_t) * (L > 0 ? L : 1)));
    MTRY(cudaMalloc(&T.facet, sizeof(int8_t) * (L > 0 ? L : 1)));
    if (L > 0) {
      MTRY(cudaMemcpyAsync(T.elem, te.data(), sizeof(int32_t) * L, cudaMemcpyHostToDevice, s));
      MTRY(cudaMemcpyAsync(T.facet, tf.data(), sizeof(int8_t) * L, cudaMemcpyHostToDevice, s));
    }
    MTRY(cudaStreamSynchronize(s));
  }
  MTRY(cudaStreamSynchronize(s));
#undef MTRY
  *out = m;
  return 0;
}

int fem_mesh_info(fem_mesh_t m, int* n_loc, int* kappa_hat, int* n_colours, int64_t* n_tiles) {
  if (!m) { set_error("fem_mesh_info: NULL mesh"); return FEM_E_INVALID_ARG; }
  if (n_loc) *n_loc = m->n_loc;
  if (kappa_hat) *kappa_hat = m->kh;
  if (n_colours) *n_colours = m->n_colours;
  if (n_tiles) *n_tiles = m->last_n_tiles;
  return 0;
}

void fem_pattern_destroy(fem_pattern_t p) {
  if (!p) return;
  tiles_free(p->tiles);
  stored_free(p);
  cudaFree(p->rowptr_s); cudaFree(p->colidx_s); cudaFree(p->slot); cudaFree(p->rowptr); cudaFree(p->colidx);
  delete p;
}

int fem_pattern_build(fem_mesh_t m, void* stream, fem_pattern_t* out, int64_t* n_rows, int64_t* nnz) {
  if (!m || !out) { set_error("fem_pattern_build: NULL argument"); return FEM_E_INVALID_ARG; }
  *out = nullptr;
  fem_pattern_s* p = new fem_pattern_s();
  p->mesh = m;
  int rc = pattern_build(m, (cudaStream_t)stream, p);
  if (rc != 0) { fem_pattern_destroy(p); return rc; }
  // The node-tile schedule of FEM_SCATTER_TILED is built with the pattern (one-time).  When the mesh
  // does not fit it (an element type without a tile kernel, a row wider than the 8-bit local offsets, a
  // row larger than the shared accumulator) the pattern is still valid for the atomic and coloured scatters;
  // tiled calls then fail with FEM_E_UNSUPPORTED and this reason.
  if (m->order == 2 && (m->etype == FEM_HEX || m->etype == FEM_HEX_SERENDIPITY)) {
    p->tiles_rc = FEM_E_UNSUPPORTED;
    p->tiles_msg = "tiled scatter: no tile kernel for quadratic cubes (use FEM_SCATTER_COLOURED or _ATOMIC)";
  } else {
    // Q1-hex elasticity on a node lattice (c5 and its perturbed variant): the z-sweep schedule (sweep.cu),
    // 1.36 element visits per element instead of the node tiles' 1.95; other meshes: node tiles
    int trc = FEM_E_UNSUPPORTED;
    if (m->etype == FEM_HEX && m->order == 1 && m->kh == 3)
      trc = sweep_build(m, p, (cudaStream_t)stream);
    if (trc == FEM_E_OOM || trc == FEM_E_CUDA) { fem_pattern_destroy(p); return trc; }
    if (trc != 0) {
      tiles_free(p->tiles);
      trc = tiles_build(m, p, (cudaStream_t)stream);
    }
    if (trc == FEM_E_OOM || trc == FEM_E_CUDA) { fem_pattern_destroy(p); return trc; }
    if (trc != 0) {
      p->tiles_rc = trc;
      p->tiles_msg = fem_last_error();
      tiles_free(p->tiles);
    }
  }
  m->last_n_tiles = p->tiles.n_tiles;
  if (n_rows) *n_rows = p->n_rows;
  if (nnz) *nnz = p->nnz;
  *out = p;
  return 0;
}

int64_t fem_pattern_nnz_s(fem_pattern_t p) { return p ? p->nnz_s : -1; }

int fem_pattern_info(fem_pattern_t p, int64_t* out) {
  if (!p || !out) { set_error("fem_pattern_info: NULL argument"); return FEM_E_INVALID_ARG; }
  const TileSchedule& T = p->tiles;
  out[0] = T.n_tiles; out[1] = T.max_tile_nodes; out[2] = T.acc_max; out[3] = T.rec_max;
  out[4] = T.max_halo; out[5] = T.visits_total; out[6] = T.dom.max_per_tile; out[7] = T.rec_bytes_total;
  out[8] = p->tiles_rc ? -1 : (T.sweep ? 1 : 0);
  return 0;
}

int fem_pattern_export(fem_pattern_t p, int64_t* rowptr, int32_t* colidx, int32_t* slot_s, int64_t* rowptr_s,
                       int32_t* colidx_s, void* stream) {
  if (!p) { set_error("fem_pattern_export: NULL pattern"); return FEM_E_INVALID_ARG; }
  cudaStream_t s = (cudaStream_t)stream;
  const fem_mesh_s* m = p->mesh;
  if (rowptr) FEM_CUDA_TRY(cudaMemcpyAsync(rowptr, p->rowptr, sizeof(int64_t) * (p->n_rows + 1), cudaMemcpyDeviceToDevice, s));
  if (colidx) FEM_CUDA_TRY(cudaMemcpyAsync(colidx, p->colidx, sizeof(int32_t) * p->nnz, cudaMemcpyDeviceToDevice, s));
  if (slot_s) FEM_CUDA_TRY(cudaMemcpyAsync(slot_s, p->slot, sizeof(int32_t) * m->n_loc * m->n_loc * m->E, cudaMemcpyDeviceToDevice, s));
  if (rowptr_s) FEM_CUDA_TRY(cudaMemcpyAsync(rowptr_s, p->rowptr_s, sizeof(int64_t) * (m->n_own + 1), cudaMemcpyDeviceToDevice, s));
  if (colidx_s) FEM_CUDA_TRY(cudaMemcpyAsync(colidx_s, p->colidx_s, sizeof(int32_t) * p->nnz_s, cudaMemcpyDeviceToDevice, s));
  return 0;
}

int fem_pattern_csr(fem_pattern_t p, const int64_t** rowptr, const int32_t** colidx, int64_t* col_offset) {
  if (!p || !rowptr || !colidx) { set_error("fem_pattern_csr: NULL argument"); return FEM_E_INVALID_ARG; }
  *rowptr = p->rowptr;
  *colidx = p->colidx;
  if (col_offset) *col_offset = p->mesh->own_lo;
  return 0;
}

static int check_problem(const fem_mesh_s* m, const fem_problem* prob) {
  if (!prob) { set_error("NULL problem"); return FEM_E_INVALID_ARG; }
  if (prob->etype != m->etype || prob->order != m->order || prob->physics != m->physics) {
    set_error("problem element/physics does not match the mesh");
    return FEM_E_INVALID_ARG;
  }
  if (prob->n_terms < 0 || prob->n_terms > FEM_MAX_TERMS) { set_error("bad n_terms"); return FEM_E_INVALID_ARG; }
  for (int t = 0; t < prob->n_terms; t++) {
    const fem_term& T = prob->terms[t];
    if (!form_in_physics(prob->physics, T.form)) { set_error("weak form not in this physics"); return FEM_E_UNSUPPORTED; }
    if (T.region < -1 || T.region >= (int)m->bnd.size()) { set_error("term region out of range"); return FEM_E_INVALID_ARG; }
  }
  if (prob->time.kind == FEM_TIME_GENALPHA && (prob->time.nu_hat < 0 || prob->time.nu_hat > 1)) {
    set_error("only nu_hat <= 1 operands are used by the built forms");
    return FEM_E_UNSUPPORTED;
  }
  return 0;
}

static int assemble(fem_mesh_t m, fem_pattern_t p, const fem_problem* prob, const double* state, double* values,
                    double* rhs, int accumulate, int scatter, void* stream) {
  if (!m || !state || (!values && !rhs)) { set_error("assemble: NULL argument"); return FEM_E_INVALID_ARG; }
  if (values && !p) { set_error("assemble: matrix requested without a pattern"); return FEM_E_INVALID_ARG; }
  if (p && p->mesh != m) { set_error("assemble: pattern belongs to another mesh"); return FEM_E_INVALID_ARG; }
  int rc = check_problem(m, prob);
  if (rc) return rc;
  cudaStream_t s = (cudaStream_t)stream;
  bool bnd_only = false;  // tiled NS: domain terms in the tile kernel, boundary terms coloured afterwards
  if (scatter == FEM_SCATTER_STORED) {
    if (accumulate) { set_error("stored scatter writes complete rows; accumulate must be 0"); return FEM_E_INVALID_ARG; }
    if (!p) { set_error("stored scatter needs the pattern"); return FEM_E_INVALID_ARG; }
    return launch_stored(m, p, prob, state, values, rhs, s);
  }
  const bool tiled = scatter == FEM_SCATTER_TILED || scatter == FEM_SCATTER_TILED_UNORDERED;
  if (tiled && accumulate) { set_error("tiled scatter writes complete rows; accumulate must be 0"); return FEM_E_INVALID_ARG; }
  if (tiled && !values && m->etype == FEM_TET) {
    // residual-only calls on tetrahedra: the tile kernels visit each element ~3x (24 elements per vertex)
    // for rows that are cheap to scatter, so these calls take the element pass instead (documented in
    // libfem.h): coloured (deterministic) for FEM_SCATTER_TILED, atomic for _UNORDERED (c3 3.0 -> 0.9 ms)
    scatter = scatter == FEM_SCATTER_TILED ? FEM_SCATTER_COLOURED : FEM_SCATTER_ATOMIC;
  } else if (tiled) {
    if (!p) { set_error("tiled scatter needs the pattern"); return FEM_E_INVALID_ARG; }
    if (p->tiles_rc) { set_error(p->tiles_msg); return p->tiles_rc; }
    const bool det = scatter == FEM_SCATTER_TILED;
    // NS on P1 tets: the generic boundary terms (1% of the visits) would stall the whole tile
    // behind a facet phase run by a few warps (22% of c4); they run instead as the deterministic coloured
    // facet pass over the rows the tile kernel has written
    const bool ns_split = m->etype == FEM_TET && m->order == 1 && m->physics == FEM_NS;
    if (!ns_split) return launch_tiled(m, p, prob, state, values, rhs, det, s);
    fem_problem dom = *prob;
    dom.n_terms = 0;
    bool any_bnd = false;
    for (int t = 0; t < prob->n_terms; t++) {
      if (prob->terms[t].region < 0) dom.terms[dom.n_terms++] = prob->terms[t];
      else any_bnd = true;
    }
    rc = launch_tiled(m, p, &dom, state, values, rhs, det, s);
    if (rc || !any_bnd) return rc;
    bnd_only = true;
    scatter = FEM_SCATTER_COLOURED;
  }
  if (!tiled || scatter == FEM_SCATTER_COLOURED || scatter == FEM_SCATTER_ATOMIC) {
    if (scatter != FEM_SCATTER_ATOMIC && scatter != FEM_SCATTER_COLOURED) {
      set_error("bad scatter mode");
      return FEM_E_INVALID_ARG;
    }
    if (!accumulate && !bnd_only) {  // "cleared first" (D-2 P:426, D-3 P:441)
      if (values) FEM_CUDA_TRY(cudaMemsetAsync(values, 0, sizeof(double) * p->nnz, s));
      if (rhs) FEM_CUDA_TRY(cudaMemsetAsync(rhs, 0, sizeof(double) * m->kh * m->n_own, s));
    }
  }
  for (int t = 0; t < prob->n_terms; t++) {
    const fem_term& T = prob->terms[t];
    if (bnd_only && T.region < 0) continue;
    AsmArgs A;
    A.m = m; A.pat = p; A.F = make_form_args(prob, T); A.quad_order = prob->quad_order; A.state = state;
    A.values = (T.form == FEM_WF_ELAST_LOAD) ? nullptr : values;
    A.rhs = rhs;
    if (!A.values && !A.rhs) continue;
    A.plain = (scatter == FEM_SCATTER_COLOURED);
    A.stream = s;
    const TaskList& L = (T.region < 0) ? m->dom : m->bnd[T.region];
    A.task_elem = L.elem;
    A.task_facet = (T.region < 0) ? nullptr : L.facet;
    // element kernel: quadratic-cube elasticity on the fp64 tensor cores, else the generic batch kernel
    auto launch_el = [&](const AsmArgs& a) {
      if (T.region < 0) {
        int handled = 0;
        const int r = launch_q2_elast(a, &handled);
        if (handled) return r;
      }
      return launch_generic(a, T.region >= 0);
    };
    if (scatter == FEM_SCATTER_ATOMIC) {
      A.task_begin = 0; A.task_count = L.n;
      if (T.region < 0) A.task_elem = nullptr;  // natural element order
      rc = launch_el(A);
      if (rc) return rc;
    } else {
      for (size_t c = 0; c + 1 < L.col_off.size(); c++) {
        A.task_begin = L.col_off[c];
        A.task_count = L.col_off[c + 1] - L.col_off[c];
        rc = launch_el(A);
        if (rc) return rc;
      }
    }
  }
  return 0;
}

int fem_assemble_matrix(fem_mesh_t m, fem_pattern_t p, const fem_problem* prob, const double* state, double* values,
                        int accumulate, int scatter, void* stream) {
  if (!values) { set_error("fem_assemble_matrix: values is NULL"); return FEM_E_INVALID_ARG; }
  return assemble(m, p, prob, state, values, nullptr, accumulate, scatter, stream);
}

int fem_assemble_residual(fem_mesh_t m, fem_pattern_t p, const fem_problem* prob, const double* state, double* rhs,
                          int accumulate, int scatter, void* stream) {
  if (!rhs) { set_error("fem_assemble_residual: rhs is NULL"); return FEM_E_INVALID_ARG; }
  return assemble(m, p, prob, state, nullptr, rhs, accumulate, scatter, stream);
}

int fem_assemble_system(fem_mesh_t m, fem_pattern_t p, const fem_problem* prob, const double* state, double* values,
                        double* rhs, int accumulate, int scatter, void* stream) {
  if (!values || !rhs) { set_error("fem_assemble_system: NULL output"); return FEM_E_INVALID_ARG; }
  return assemble(m, p, prob, state, values, rhs, accumulate, scatter, stream);
}

int fem_residual_norms(fem_mesh_t m, const double* rhs, double* norms_dev, void* stream) {
  if (!m || !rhs || !norms_dev) { set_error("fem_residual_norms: NULL argument"); return FEM_E_INVALID_ARG; }
  return residual_norms(m, rhs, norms_dev, (cudaStream_t)stream);
}

int fem_linearize_host(fem_mesh_t m, fem_pattern_t p, const fem_problem* prob, const double* state_host,
                       double* values, double* rhs, double* norms_host, int scatter, void* stream) {
  if (!m || !p || !prob || !state_host || !values || !rhs || !norms_host) {
    set_error("fem_linearize_host: NULL argument");
    return FEM_E_INVALID_ARG;
  }
  cudaStream_t s = (cudaStream_t)stream;
  const int levels = (prob->time.kind == FEM_TIME_GENALPHA ? prob->time.nu_hat : 0) + 1;
  const size_t bytes = sizeof(double) * levels * m->kh * m->N;
  if (m->scratch_state_bytes < bytes + 2 * sizeof(double)) {
    if (m->scratch_state) cudaFree(m->scratch_state);
    m->scratch_state = nullptr;
    m->scratch_state_bytes = 0;
    FEM_CUDA_TRY(cudaMalloc(&m->scratch_state, bytes + 2 * sizeof(double)));
    m->scratch_state_bytes = bytes + 2 * sizeof(double);
  }
  FEM_CUDA_TRY(cudaMemcpyAsync(m->scratch_state, state_host, bytes, cudaMemcpyHostToDevice, s));
  int rc = assemble(m, p, prob, m->scratch_state, values, rhs, 0, scatter, stream);
  if (rc) return rc;
  double* nd = m->scratch_state + levels * m->kh * m->N;
  rc = residual_norms(m, rhs, nd, s);
  if (rc) return rc;
  FEM_CUDA_TRY(cudaMemcpyAsync(norms_host, nd, 2 * sizeof(double), cudaMemcpyDeviceToHost, s));
  FEM_CUDA_TRY(cudaStreamSynchronize(s));
  return 0;
}

int fem_linearize_host_async(fem_mesh_t m, fem_pattern_t p, const fem_problem* prob, const double* state_host,
                             double* values, double* rhs, double* norms_host, int scatter, void* stream) {
  if (!m || !p || !prob || !state_host || !values || !rhs || !norms_host) {
    set_error("fem_linearize_host_async: NULL argument");
    return FEM_E_INVALID_ARG;
  }
  cudaStream_t s = (cudaStream_t)stream;
  const int levels = (prob->time.kind == FEM_TIME_GENALPHA ? prob->time.nu_hat : 0) + 1;
  const size_t bytes = sizeof(double) * levels * m->kh * m->N;
  if (!m->copy_stream) {
    FEM_CUDA_TRY(cudaStreamCreateWithFlags(&m->copy_stream, cudaStreamNonBlocking));
    for (int b = 0; b < 2; b++) {
      FEM_CUDA_TRY(cudaEventCreateWithFlags(&m->ev_copied[b], cudaEventDisableTiming));
      FEM_CUDA_TRY(cudaEventCreateWithFlags(&m->ev_used[b], cudaEventDisableTiming));
    }
  }
  if (m->async_bytes < bytes + 2 * sizeof(double)) {
    FEM_CUDA_TRY(cudaStreamSynchronize(s));
    FEM_CUDA_TRY(cudaStreamSynchronize(m->copy_stream));
    for (int b = 0; b < 2; b++) {
      if (m->async_state[b]) cudaFree(m->async_state[b]);
      m->async_state[b] = nullptr;
    }
    m->async_bytes = 0;
    for (int b = 0; b < 2; b++) FEM_CUDA_TRY(cudaMalloc(&m->async_state[b], bytes + 2 * sizeof(double)));
    m->async_bytes = bytes + 2 * sizeof(double);
    m->async_calls = 0;
  }
  const int b = (int)(m->async_calls & 1);
  // the staging buffer b was last read by the assembly of call k-2: the copy waits for it, then this
  // call's H2D runs on the copy stream while the previous call's assembly runs on `stream`
  if (m->async_calls >= 2) FEM_CUDA_TRY(cudaStreamWaitEvent(m->copy_stream, m->ev_used[b], 0));
  FEM_CUDA_TRY(cudaMemcpyAsync(m->async_state[b], state_host, bytes, cudaMemcpyHostToDevice, m->copy_stream));
  FEM_CUDA_TRY(cudaEventRecord(m->ev_copied[b], m->copy_stream));
  FEM_CUDA_TRY(cudaStreamWaitEvent(s, m->ev_copied[b], 0));
  int rc = assemble(m, p, prob, m->async_state[b], values, rhs, 0, scatter, stream);
  if (rc) return rc;
  double* nd = m->async_state[b] + levels * m->kh * m->N;
  rc = residual_norms(m, rhs, nd, s);
  if (rc) return rc;
  FEM_CUDA_TRY(cudaMemcpyAsync(norms_host, nd, 2 * sizeof(double), cudaMemcpyDeviceToHost, s));
  FEM_CUDA_TRY(cudaEventRecord(m->ev_used[b], s));
  m->async_calls++;
  return 0;
}

int fem_get_status(fem_mesh_t m, void* stream, int64_t* bad_elem) {
  if (!m) { set_error("fem_get_status: NULL mesh"); return FEM_E_INVALID_ARG; }
  cudaStream_t s = (cudaStream_t)stream;
  long long h = -1;
  FEM_CUDA_TRY(cudaMemcpyAsync(&h, m->err, sizeof(long long), cudaMemcpyDeviceToHost, s));
  FEM_CUDA_TRY(cudaStreamSynchronize(s));
  FEM_CUDA_TRY(cudaMemsetAsync(m->err, 0xff, sizeof(long long), s));
  if (bad_elem) *bad_elem = h;
  if (h >= 0) { set_error("inverted element (det J <= 0)"); return FEM_E_INVERTED_ELEMENT; }
  return 0;
}

}  // extern "C"
