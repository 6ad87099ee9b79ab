// stored.cu — FEM_SCATTER_STORED: element-stored assembly with a deterministic per-slot gather.
//
// D-2 / D-3 add every element's local residual and local stiffness block into d and K.  The
// paper increments a COO array atomically; the owner-gather tiles of tiled.cu sum inside shared memory.
// This mode splits the sum into two halves joined through a scratch in HBM:
//   element  every element computes its whole local block K^e_(a,κ),(b,λ) (symmetric physics: the blocks
//            a <= b) and residual d^e_(a,κ) and stores them at its position in the Morton order of element
//            centroids — no conflicts, each element owns its storage (P2-tet elasticity: k_p2_el on the
//            tensor cores, tet2_el.cu; Q1-hex elasticity: k_hex_el, hex_tiled.cu; P1-tet NS: k_ns_el,
//            tet1_ns.cu; everything else: the generic element kernel); boundary terms add
//            into the owning element's storage;
//   gather   every scalar CSR slot s = (row point, column point) sums the blocks of the elements that
//            contain both points, in a fixed list order (built once by a stable radix sort of the slot map),
//            and writes its κ̂² values; every owned row sums its elements' residual rows.
// No atomics and a fixed summation order: bit-identical run to run, complete rows written.
#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>
#include <string>
#include <utility>
#include <vector>

#include "assemble_generic.cuh"
#include "stored.cuh"

namespace fem {

static int grid_of(int64_t n, int threads = 256) {
  int64_t b = (n + threads - 1) / threads;
  return (int)std::min<int64_t>(std::max<int64_t>(b, 1), 148 * 64);
}

// packed index of block (a, b), a <= b, of a symmetric element matrix stored row by row
__host__ __device__ inline int st_ublk(int a, int b, int NL) { return a * NL - a * (a - 1) / 2 + (b - a); }

// keys: the slot of (pos, a, b) for owned rows, nnz_s (sorted past every slot) otherwise; values: the block's
// storage index (pos·NB + blk) << 1 | transposed (sym: a block a > b is read as the transpose of (b, a));
// generated in position-major order, so the stable sort leaves every slot's list in position order
__global__ void k_st_keys(const int32_t* __restrict__ slot, const int32_t* __restrict__ conn,
                          const int32_t* __restrict__ eperm, int64_t E, int NL, int64_t lo, int64_t hi, uint32_t nnz_s,
                          int sym, uint32_t* __restrict__ key, uint32_t* __restrict__ val) {
  const int64_t n = E * NL * NL;
  const int NB = sym ? NL * (NL + 1) / 2 : NL * NL;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t pos = t / (NL * NL);
    const int ab = (int)(t - pos * NL * NL), a = ab / NL, b = ab - a * NL;
    const int64_t e = eperm[pos];
    const int64_t r = conn[(int64_t)a * E + e];
    key[t] = (r >= lo && r < hi) ? (uint32_t)slot[(int64_t)ab * E + e] : nnz_s;
    const int blk = !sym ? ab : (a <= b ? st_ublk(a, b, NL) : st_ublk(b, a, NL));
    val[t] = (uint32_t)(((pos * NB + blk) << 1) | (sym && a > b ? 1 : 0));
  }
}

// off[s] = first position of slot s in the sorted keys; off[nnz_s] = number of owned entries
__global__ void k_st_off(const uint32_t* __restrict__ key, int64_t n, uint32_t nnz_s, uint32_t* __restrict__ off) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t k = key[i], kp = i ? key[i - 1] : 0xffffffffu;
    if (k != kp && k <= nnz_s) off[k] = (uint32_t)i;  // k == nnz_s: the first non-owned entry (list end)
    if (i == n - 1 && k < nnz_s) off[nnz_s] = (uint32_t)n;
  }
}

// residual lists: the elements of owned row r are the entries of its diagonal slot (a = b, one per element)
__global__ void k_st_diag(const int32_t* __restrict__ slot, const int32_t* __restrict__ conn, int64_t E, int NL,
                          int64_t lo, int64_t hi, int64_t* __restrict__ diag) {
  const int64_t n = E * NL;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = t / NL;
    const int a = (int)(t - e * NL);
    const int64_t r = conn[(int64_t)a * E + e];
    if (r >= lo && r < hi) diag[r - lo] = slot[((int64_t)a * NL + a) * E + e];  // every writer agrees
  }
}
__global__ void k_st_rcount(const int64_t* __restrict__ diag, const uint32_t* __restrict__ off, int64_t n_own,
                            uint32_t* __restrict__ cnt) {
  for (int64_t li = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; li < n_own; li += (int64_t)gridDim.x * blockDim.x)
    cnt[li] = off[diag[li] + 1] - off[diag[li]];
}
__global__ void k_st_rfill(const int64_t* __restrict__ diag, const uint32_t* __restrict__ off,
                           const uint32_t* __restrict__ ent, const uint32_t* __restrict__ roff, int64_t n_own, int NL,
                           int sym, uint32_t* __restrict__ rent) {
  const int NB = sym ? NL * (NL + 1) / 2 : NL * NL;
  for (int64_t li = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; li < n_own; li += (int64_t)gridDim.x * blockDim.x) {
    const int64_t s = diag[li];
    for (uint32_t j = off[s]; j < off[s + 1]; j++) {
      const uint32_t x = ent[j] >> 1;
      const uint32_t pos = x / (uint32_t)NB, blk = x - pos * (uint32_t)NB;
      int a = 0;
      if (sym) { while (st_ublk(a, a, NL) != (int)blk) a++; }
      else a = (int)blk / (NL + 1);
      rent[roff[li] + (j - off[s])] = pos * (uint32_t)NL + (uint32_t)a;
    }
  }
}

// ---- two-phase path, gather: warp per owned row in the gather order
template <int KH, bool RES_ONLY>
__global__ void __launch_bounds__(256) k_st_gather(const int64_t* __restrict__ rowptr_s, int64_t n_own, int64_t nnz_s,
                                                   const int32_t* __restrict__ rows, const uint32_t* __restrict__ off,
                                                   const uint32_t* __restrict__ ent, const double* __restrict__ ek,
                                                   double* __restrict__ values, const uint32_t* __restrict__ roff,
                                                   const uint32_t* __restrict__ rent, const double* __restrict__ er,
                                                   double* __restrict__ rhs) {
  // κ̂ = 4 (P1-tet NS rows: ≤ 15 slots): four rows per warp, 8 lanes each (c4: 32 lanes 33.0, 16 lanes
  // 27.2, 8 lanes 25.6, 4 lanes 27.2 ms); κ̂ = 3 keeps a warp per row (c3: 8 lanes 5.2 vs 4.9 ms)
  // residual-only calls: a row has one entry per element (8-24), 8 lanes per row
  constexpr int W = (KH == 4 || RES_ONLY) ? 8 : 32, RPW = 32 / W;
  const int sub = (threadIdx.x & 31) / W;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t w0 = (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5) * RPW; w0 < n_own; w0 += nw * RPW) {
    const int64_t w = w0 + sub;
    const int64_t li = w < n_own ? (int64_t)__ldg(rows + w) : -1;
    if (values && li >= 0) st_gather_row<KH, W>(li, rowptr_s, nnz_s, off, ent, ek, values);
    if (rhs) st_res_row<KH, W>(li, n_own, roff, rent, er, rhs);
  }
}

void stored_free(fem_pattern_s* p) {
  void* ptrs[] = {p->st_ent, p->st_off, p->st_rent, p->st_roff, p->st_epos, p->st_eperm, p->st_rows, p->st_ek, p->st_er,
                  p->st_xaos, p->st_saos};
  for (void* q : ptrs) cudaFree(q);
  p->st_ent = p->st_off = p->st_rent = p->st_roff = nullptr;
  p->st_epos = p->st_eperm = p->st_rows = nullptr;
  p->st_ek = p->st_er = p->st_xaos = p->st_saos = nullptr;
  p->st_n_ent = 0;
  p->st_nb = 0;
  for (auto& L : p->st_bnd) { cudaFree(L.elem); cudaFree(L.facet); }
  p->st_bnd.clear();
}

// P2-tet elasticity element pass on the tensor cores (tet2_el.cu): *handled = false when the problem has
// other domain forms or another quadrature order
int launch_p2_el(const fem_mesh_s* m, const fem_problem* prob, const double* state, const int32_t* eperm,
                 double* ek, double* er, cudaStream_t s, bool* handled);
// Q1-hex elasticity element pass (hex_tiled.cu), same contract
int launch_hex_el(const fem_mesh_s* m, const fem_problem* prob, const double* state, const int32_t* eperm,
                  double* ek, double* er, cudaStream_t s, bool* handled);
// P1-tet NS (SUPG/PSPG) element pass (tet1_ns.cu), same contract
int launch_ns_el(const fem_mesh_s* m, const fem_problem* prob, const double* state, const int32_t* eperm,
                 double* ek, double* er, double* xaos, double* saos, cudaStream_t s, bool* handled);

// Morton code of quantised coordinates (about one point per cell)
struct MortonQ {
  int dim;
  double bmin[3], h;
  uint64_t code(const double* x) const {
    const int bits = dim == 3 ? 21 : 31;
    uint64_t q[3] = {0, 0, 0}, c = 0;
    for (int d = 0; d < dim; d++) {
      double f = (x[d] - bmin[d]) / h;
      f = f < 0 ? 0 : f;
      q[d] = std::min<uint64_t>((uint64_t)f, ((uint64_t)1 << bits) - 1);
    }
    for (int b = 0; b < bits; b++)
      for (int d = 0; d < dim; d++) c |= ((q[d] >> b) & 1ull) << (b * dim + d);
    return c;
  }
};
static MortonQ morton_q(const fem_mesh_s* m, int64_t n_cells) {
  MortonQ Q;
  Q.dim = m->dim;
  double bmax[3] = {-1e300, -1e300, -1e300};
  for (int d = 0; d < 3; d++) Q.bmin[d] = 1e300;
  for (int d = 0; d < m->dim; d++)
    for (int64_t i = 0; i < m->N; i++) {
      const double x = m->h_coords[(int64_t)d * m->N + i];
      Q.bmin[d] = std::min(Q.bmin[d], x);
      bmax[d] = std::max(bmax[d], x);
    }
  double vol = 1.0;
  for (int d = 0; d < m->dim; d++) vol *= std::max(bmax[d] - Q.bmin[d], 1e-300);
  Q.h = std::pow(vol / (double)std::max<int64_t>(n_cells, 1), 1.0 / m->dim);
  return Q;
}

template <class T>
static int upload(T** dst, const std::vector<T>& v, cudaStream_t s) {
  if (cudaMalloc(dst, sizeof(T) * std::max<size_t>(v.size(), 1))) { *dst = nullptr; return FEM_E_OOM; }
  if (!v.empty()) FEM_CUDA_TRY(cudaMemcpyAsync(*dst, v.data(), sizeof(T) * v.size(), cudaMemcpyHostToDevice, s));
  return 0;
}

}  // namespace fem

using namespace fem;

int fem_pattern_stored_prepare(fem_pattern_t p, int with_matrix, void* stream) {
  if (!p) { set_error("fem_pattern_stored_prepare: NULL pattern"); return FEM_E_INVALID_ARG; }
  const fem_mesh_s* m = p->mesh;
  cudaStream_t s = (cudaStream_t)stream;
  const int NL = m->n_loc, KH = m->kh, dim = m->dim;
  // elasticity: every form's tangent is symmetric, so only the blocks a <= b are stored
  const int sym = m->physics == FEM_ELASTICITY ? 1 : 0;
  const int NB = sym ? NL * (NL + 1) / 2 : NL * NL;
  const int64_t E = m->E, n = E * NL * NL, n_own = m->n_own, lo = m->own_lo, hi = m->own_hi;
  if (2 * E * NB >= ((int64_t)1 << 32) || p->nnz_s >= ((int64_t)1 << 32) - 1 || n >= ((int64_t)1 << 31)) {
    set_error("fem_pattern_stored_prepare: the element blocks do not fit the 32-bit contribution lists");
    return FEM_E_INDEX_OVERFLOW;
  }
  auto fail = [&](int rc, const std::string& what) {
    stored_free(p);
    set_error("fem_pattern_stored_prepare: " + what);
    return rc;
  };
  if (!p->st_ent) {
    // 1. element order: Morton order of the centroids (host, one-time)
    std::vector<int32_t> eperm(E), epos(E);
    {
      const MortonQ Q = morton_q(m, E);
      std::vector<std::pair<uint64_t, int32_t>> key(E);
      for (int64_t e = 0; e < E; e++) {
        double x[3] = {0, 0, 0};
        for (int a = 0; a < NL; a++) {
          const int64_t r = m->h_conn[(int64_t)a * E + e];
          for (int d = 0; d < dim; d++) x[d] += m->h_coords[(int64_t)d * m->N + r];
        }
        for (int d = 0; d < dim; d++) x[d] /= NL;
        key[e] = {Q.code(x), (int32_t)e};
      }
      std::sort(key.begin(), key.end());
      for (int64_t i = 0; i < E; i++) { eperm[i] = key[i].second; epos[key[i].second] = (int32_t)i; }
    }
    if (upload(&p->st_eperm, eperm, s) || upload(&p->st_epos, epos, s)) return fail(FEM_E_OOM, "out of device memory");
    // 2. contribution lists (device sort of the slot map)
    uint32_t *k1 = nullptr, *k2 = nullptr, *v1 = nullptr, *v2 = nullptr, *cnt = nullptr;
    int64_t* diag = nullptr;
    void* tmp = nullptr;
    size_t tmp_bytes = 0, tmp_scan = 0;
    auto cleanup = [&]() {
      cudaFree(k1); cudaFree(k2); cudaFree(v1); cudaFree(v2); cudaFree(tmp); cudaFree(diag); cudaFree(cnt);
    };
    int end_bit = 1;
    while (end_bit < 32 && ((uint64_t)1 << end_bit) <= (uint64_t)p->nnz_s) end_bit++;
    const size_t nb = sizeof(uint32_t) * (size_t)std::max<int64_t>(n, 1);
    if (cudaMalloc(&k1, nb) || cudaMalloc(&k2, nb) || cudaMalloc(&v1, nb) || cudaMalloc(&v2, nb) ||
        cudaMalloc(&p->st_off, sizeof(uint32_t) * (p->nnz_s + 1)) ||
        cudaMalloc(&diag, sizeof(int64_t) * std::max<int64_t>(n_own, 1)) ||
        cudaMalloc(&cnt, sizeof(uint32_t) * (n_own + 1)) || cudaMalloc(&p->st_roff, sizeof(uint32_t) * (n_own + 1))) {
      cleanup();
      return fail(FEM_E_OOM, "out of device memory for the contribution lists");
    }
    k_st_keys<<<grid_of(n), 256, 0, s>>>(p->slot, m->conn, p->st_eperm, E, NL, lo, hi, (uint32_t)p->nnz_s, sym, k1, v1);
    cub::DoubleBuffer<uint32_t> dk(k1, k2), dv(v1, v2);
    cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, dk, dv, (int)n, 0, end_bit, s);
    cub::DeviceScan::ExclusiveSum(nullptr, tmp_scan, cnt, p->st_roff, (int)(n_own + 1), s);
    if (cudaMalloc(&tmp, std::max<size_t>(std::max(tmp_bytes, tmp_scan), 16))) {
      cleanup();
      return fail(FEM_E_OOM, "out of device memory for the sort scratch");
    }
    cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, dk, dv, (int)n, 0, end_bit, s);
    FEM_CUDA_TRY(cudaMemsetAsync(p->st_off, 0, sizeof(uint32_t) * (p->nnz_s + 1), s));
    k_st_off<<<grid_of(n), 256, 0, s>>>(dk.Current(), n, (uint32_t)p->nnz_s, p->st_off);
    k_st_diag<<<grid_of(E * NL), 256, 0, s>>>(p->slot, m->conn, E, NL, lo, hi, diag);
    FEM_CUDA_TRY(cudaMemsetAsync(cnt, 0, sizeof(uint32_t) * (n_own + 1), s));
    k_st_rcount<<<grid_of(n_own), 256, 0, s>>>(diag, p->st_off, n_own, cnt);
    cub::DeviceScan::ExclusiveSum(tmp, tmp_scan, cnt, p->st_roff, (int)(n_own + 1), s);
    uint32_t n_ent = 0, n_rent = 0;
    cudaError_t ce = cudaMemcpyAsync(&n_ent, p->st_off + p->nnz_s, sizeof(uint32_t), cudaMemcpyDeviceToHost, s);
    if (ce == cudaSuccess) ce = cudaMemcpyAsync(&n_rent, p->st_roff + n_own, sizeof(uint32_t), cudaMemcpyDeviceToHost, s);
    if (ce == cudaSuccess) ce = cudaStreamSynchronize(s);
    if (ce != cudaSuccess) {
      cleanup();
      return fail(FEM_E_CUDA, cudaGetErrorString(ce));
    }
    if (cudaMalloc(&p->st_rent, sizeof(uint32_t) * std::max<uint32_t>(n_rent, 1))) {
      cleanup();
      return fail(FEM_E_OOM, "out of device memory for the residual lists");
    }
    k_st_rfill<<<grid_of(n_own), 256, 0, s>>>(diag, p->st_off, dv.Current(), p->st_roff, n_own, NL, sym, p->st_rent);
    ce = cudaGetLastError();
    if (ce == cudaSuccess) ce = cudaStreamSynchronize(s);
    if (ce != cudaSuccess) {
      cleanup();
      return fail(FEM_E_CUDA, cudaGetErrorString(ce));
    }
    uint32_t* keep = dv.Current();  // the sorted values are the contribution lists
    if (keep == v1) v1 = nullptr; else v2 = nullptr;
    cleanup();
    p->st_ent = keep;
    p->st_n_ent = n_ent;
    p->st_nb = NB;
    // 3. gather order of the rows: Morton order of their points (the warps in flight cover a compact patch,
    // so the two reads of a symmetric block and the list lines mostly hit L2)
    std::vector<std::pair<uint64_t, int32_t>> rk(n_own);
    {
      const MortonQ Q = morton_q(m, n_own);
      for (int64_t i = 0; i < n_own; i++) {
        double x[3] = {0, 0, 0};
        for (int d = 0; d < dim; d++) x[d] = m->h_coords[(int64_t)d * m->N + lo + i];
        rk[i] = {Q.code(x), (int32_t)i};
      }
      std::sort(rk.begin(), rk.end());
    }
    std::vector<int32_t> rows(n_own);
    for (int64_t i = 0; i < n_own; i++) rows[i] = rk[i].second;
    if (upload(&p->st_rows, rows, s)) return fail(FEM_E_OOM, "out of device memory for the row order");
    // 4. boundary facets grouped by their rank within their element (stable: set order inside a group)
    for (size_t k = 0; k < m->h_bset_elem.size(); k++) {
      const auto& be = m->h_bset_elem[k];
      const auto& bf = m->h_bset_facet[k];
      std::vector<std::pair<int32_t, int32_t>> key(be.size());  // (rank, index)
      std::vector<uint8_t> seen(E, 0);
      for (size_t j = 0; j < be.size(); j++) key[j] = {seen[be[j]]++, (int32_t)j};
      std::stable_sort(key.begin(), key.end());
      std::vector<int32_t> el(be.size());
      std::vector<int8_t> fa(be.size());
      TaskList L;
      L.n = (int64_t)be.size();
      L.col_off.push_back(0);
      for (size_t j = 0; j < key.size(); j++) {
        el[j] = be[key[j].second];
        fa[j] = bf[key[j].second];
        if (j && key[j].first != key[j - 1].first) L.col_off.push_back((int64_t)j);
      }
      L.col_off.push_back(L.n);
      if (upload(&L.elem, el, s) || upload(&L.facet, fa, s)) {
        cudaFree(L.elem);
        return fail(FEM_E_OOM, "out of device memory for the boundary groups");
      }
      p->st_bnd.push_back(L);
    }
    FEM_CUDA_TRY(cudaStreamSynchronize(s));
  }
  if (m->physics == FEM_NS && m->etype == FEM_TET && m->order == 1 && !p->st_xaos) {  // k_ns_el's node-major copies
    if (cudaMalloc(&p->st_xaos, sizeof(double) * 4 * (size_t)std::max<int64_t>(m->N, 1)) ||
        cudaMalloc(&p->st_saos, sizeof(double) * 4 * (size_t)std::max<int64_t>(m->N, 1))) {
      set_error("fem_pattern_stored_prepare: out of device memory for the node-major copies");
      return FEM_E_OOM;
    }
  }
  if (!p->st_er) {
    if (cudaMalloc(&p->st_er, sizeof(double) * (size_t)std::max<int64_t>(E * NL * KH, 1))) {
      p->st_er = nullptr;
      set_error("fem_pattern_stored_prepare: out of device memory for the element residuals");
      return FEM_E_OOM;
    }
  }
  if (with_matrix && !p->st_ek) {
    if (cudaMalloc(&p->st_ek, sizeof(double) * (size_t)std::max<int64_t>(E * NB * st_bs(KH), 1))) {
      p->st_ek = nullptr;
      set_error("fem_pattern_stored_prepare: out of device memory for the element blocks (" +
                std::to_string((double)E * NB * st_bs(KH) * 8 / 1e9) + " GB)");
      return FEM_E_OOM;
    }
  }
  return 0;
}

namespace fem {

// Boundary terms into storage: the facets of one element must not be added concurrently (they share its
// storage; facets of different elements never conflict), so a set runs as ≤ 6 launches — group g holds each
// element's g-th facet — in term order, added (the storage holds the domain part, or zeros).
static int stored_facets(const fem_mesh_s* m, const fem_pattern_s* p, const fem_problem* prob, const double* state,
                         double* ek, double* er, const int32_t* map, cudaStream_t s) {
  for (int t = 0; t < prob->n_terms; t++) {
    const fem_term& T = prob->terms[t];
    if (T.region < 0) continue;
    AsmArgs A;
    A.m = m; A.pat = p; A.F = make_form_args(prob, T); A.quad_order = prob->quad_order; A.state = state;
    A.values = nullptr; A.rhs = nullptr; A.plain = 1; A.stream = s;
    A.ek = (T.form == FEM_WF_ELAST_LOAD) ? nullptr : ek;
    A.er = er;
    A.ek_add = 1;
    A.ek_map = map;
    if (!A.ek && !A.er) continue;
    const TaskList& L = p->st_bnd[T.region];
    A.task_elem = L.elem;
    A.task_facet = L.facet;
    for (size_t c = 0; c + 1 < L.col_off.size(); c++) {
      A.task_begin = L.col_off[c];
      A.task_count = L.col_off[c + 1] - L.col_off[c];
      const int rc = launch_generic(A, true);
      if (rc) return rc;
    }
  }
  return 0;
}

int launch_stored(const fem_mesh_s* m, const fem_pattern_s* p, const fem_problem* prob, const double* state,
                  double* values, double* rhs, cudaStream_t s) {
  if (!p->st_ent || !p->st_er || (values && !p->st_ek)) {
    set_error("FEM_SCATTER_STORED: call fem_pattern_stored_prepare (with_matrix for matrix calls) first");
    return FEM_E_INVALID_ARG;
  }
  const int NL = m->n_loc, KH = m->kh;
  double* ek = values ? p->st_ek : nullptr;
  double* er = rhs ? p->st_er : nullptr;
  bool any_bnd = false;
  for (int t = 0; t < prob->n_terms; t++) any_bnd |= prob->terms[t].region >= 0;
  int rc = 0;
  // ---- element pass: domain terms store (the first) or add into the scratch at the element's position
  bool first = true;
  {
    bool handled = false;
    rc = launch_p2_el(m, prob, state, p->st_eperm, ek, er, s, &handled);
    if (!rc && !handled) rc = launch_ns_el(m, prob, state, p->st_eperm, ek, er, p->st_xaos, p->st_saos, s, &handled);
    if (!rc && !handled) rc = launch_hex_el(m, prob, state, p->st_eperm, ek, er, s, &handled);
    if (rc) return rc;
    if (handled) first = false;
  }
  for (int t = 0; t < prob->n_terms && first; t++) {  // (skipped when the P2 kernel took them all)
    if (prob->terms[t].region >= 0) continue;
    for (int t2 = t; t2 < prob->n_terms; t2++) {  // every domain term in term order: the first stores
      const fem_term& T2 = prob->terms[t2];
      if (T2.region >= 0) continue;
      AsmArgs A;
      A.m = m; A.pat = p; A.F = make_form_args(prob, T2); A.quad_order = prob->quad_order; A.state = state;
      A.values = nullptr; A.rhs = nullptr; A.plain = 1; A.stream = s;
      A.ek = ek; A.er = er; A.ek_add = t2 == t ? 0 : 1; A.ek_map = p->st_epos;
      A.task_elem = nullptr; A.task_facet = nullptr; A.task_begin = 0; A.task_count = m->dom.n;
      rc = launch_generic(A, false);
      if (rc) return rc;
    }
    first = false;
  }
  if (first) {  // no domain term: the boundary terms add into zeroed storage
    if (ek) FEM_CUDA_TRY(cudaMemsetAsync(ek, 0, sizeof(double) * m->E * p->st_nb * st_bs(KH), s));
    if (er) FEM_CUDA_TRY(cudaMemsetAsync(er, 0, sizeof(double) * m->E * NL * KH, s));
  }
  if (any_bnd) {
    rc = stored_facets(m, p, prob, state, ek, er, p->st_epos, s);
    if (rc) return rc;
  }
  // ---- gather
  if (m->n_own) {
    const int grid = grid_of(m->n_own * 32);
#define ST_GATHER(K)                                                                                             \
  (values ? k_st_gather<K, false> : k_st_gather<K, true>)<<<grid, 256, 0, s>>>(                                  \
      p->rowptr_s, m->n_own, p->nnz_s, p->st_rows, p->st_off, p->st_ent, ek, values, p->st_roff, p->st_rent, er, rhs)
    if (KH == 1) ST_GATHER(1);
    else if (KH == 2) ST_GATHER(2);
    else if (KH == 3) ST_GATHER(3);
    else ST_GATHER(4);
#undef ST_GATHER
    FEM_CUDA_TRY(cudaGetLastError());
  }
  return 0;
}

}  // namespace fem
