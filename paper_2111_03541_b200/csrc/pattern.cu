// pattern.cu — device sparsity-pattern build (fem_pattern_build), SURVEY §8(a) A2.
//
// PAPER.md Block B-1 item 4: control-point pairs (α1, α2) are collected "by variating the last input
// in each element to control point mapping, where each unique pair is only kept once";
// A-3 symbol pairs are all (κ0, κλ) (reading L6); B-4 fills I = g(κ0, α1), J = g(κλ, α2).
// Realised as: pair keys (α1-lo)·N + α2 for owned α1 -> radix sort -> unique -> scalar CSR
// (rowptr_s, colidx_s) -> κ-major block CSR (rowptr, colidx) by arithmetic -> element slot map by
// binary search.  One host sync reads the unique count.
#include <cub/cub.cuh>

#include "fem_internal.cuh"

namespace fem {

__global__ void k_pair_keys(const int32_t* __restrict__ conn, int64_t E, int NL, int64_t N, int64_t lo,
                            int64_t hi, int64_t sentinel, int64_t* __restrict__ keys) {
  const int64_t total = E * NL * NL;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = t % E;
    const int ab = (int)(t / E);
    const int a = ab / NL, b = ab % NL;
    const int64_t r = conn[(int64_t)a * E + e];
    const int64_t c = conn[(int64_t)b * E + e];
    keys[t] = (r >= lo && r < hi) ? (r - lo) * N + c : sentinel;
  }
}

__global__ void k_rowptr_s(const int64_t* __restrict__ ukeys, int64_t nnz_s, int64_t n_own, int64_t N,
                           int64_t* __restrict__ rowptr_s) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i <= n_own; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t target = i * N;  // first key of row i
    int64_t lo = 0, hi = nnz_s;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (ukeys[mid] < target) lo = mid + 1;
      else hi = mid;
    }
    rowptr_s[i] = lo;
  }
}

__global__ void k_colidx_s(const int64_t* __restrict__ ukeys, int64_t nnz_s, int64_t N, int32_t* __restrict__ colidx_s) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < nnz_s; t += (int64_t)gridDim.x * blockDim.x)
    colidx_s[t] = (int32_t)(ukeys[t] % N);
}

__global__ void k_slot(const int32_t* __restrict__ conn, int64_t E, int NL, int64_t lo, int64_t hi,
                       const int64_t* __restrict__ rowptr_s, const int32_t* __restrict__ colidx_s,
                       int32_t* __restrict__ slot) {
  const int64_t total = E * NL * NL;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = t % E;
    const int ab = (int)(t / E);
    const int a = ab / NL, b = ab % NL;
    const int64_t r = conn[(int64_t)a * E + e];
    const int32_t c = conn[(int64_t)b * E + e];
    int32_t s = -1;
    if (r >= lo && r < hi) {
      int64_t l = rowptr_s[r - lo], h = rowptr_s[r - lo + 1];
      while (l < h) {
        const int64_t mid = (l + h) >> 1;
        if (colidx_s[mid] < c) l = mid + 1;
        else h = mid;
      }
      s = (int32_t)l;
    }
    slot[t] = s;
  }
}

__global__ void k_block_rowptr(const int64_t* __restrict__ rowptr_s, int64_t n_own, int KH, int64_t nnz_s,
                               int64_t* __restrict__ rowptr) {
  const int64_t n_rows = (int64_t)KH * n_own;
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r <= n_rows; r += (int64_t)gridDim.x * blockDim.x) {
    if (r == n_rows) { rowptr[r] = (int64_t)KH * KH * nnz_s; continue; }
    const int64_t k0 = r / n_own, i = r % n_own;
    rowptr[r] = k0 * KH * nnz_s + (int64_t)KH * rowptr_s[i];
  }
}

// one thread per scalar nonzero t; writes its KH x KH block copies
__global__ void k_block_colidx(const int64_t* __restrict__ rowptr_s, const int32_t* __restrict__ colidx_s,
                               int64_t n_own, int64_t nnz_s, int KH, int64_t N, int32_t* __restrict__ colidx) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < nnz_s; t += (int64_t)gridDim.x * blockDim.x) {
    int64_t l = 0, h = n_own;  // row i: rowptr_s[i] <= t < rowptr_s[i+1]
    while (h - l > 1) {
      const int64_t mid = (l + h) >> 1;
      if (rowptr_s[mid] <= t) l = mid;
      else h = mid;
    }
    const int64_t i = l, rps = rowptr_s[i], deg = rowptr_s[i + 1] - rps, off = t - rps;
    for (int k0 = 0; k0 < KH; k0++)
      for (int kl = 0; kl < KH; kl++)
        colidx[(int64_t)k0 * KH * nnz_s + (int64_t)KH * rps + kl * deg + off] = (int32_t)(kl * N + colidx_s[t]);
  }
}

static unsigned grid_for(int64_t n) {
  int64_t b = (n + 255) / 256;
  if (b > 148 * 32) b = 148 * 32;
  if (b < 1) b = 1;
  return (unsigned)b;
}

int pattern_build(fem_mesh_s* m, cudaStream_t s, fem_pattern_s* p) {
  const int NL = m->n_loc, KH = m->kh;
  const int64_t E = m->E, N = m->N, total = E * NL * NL;
  if (total >= ((int64_t)1 << 31)) {
    set_error("pattern build: E*n_loc^2 >= 2^31 pair keys (chunked build not implemented)");
    return FEM_E_INDEX_OVERFLOW;
  }
  if ((int64_t)KH * N >= ((int64_t)1 << 31)) {
    set_error("pattern build: kappa_hat*N >= 2^31 does not fit int32 column ids");
    return FEM_E_INDEX_OVERFLOW;
  }
  const int64_t sentinel = m->n_own * N;
  int end_bit = 1;
  while (end_bit < 63 && (((int64_t)1 << end_bit) <= sentinel)) end_bit++;
  int64_t *k1 = nullptr, *k2 = nullptr;
  int* d_nsel = nullptr;
  void* tmp = nullptr;
  size_t tmp_sort = 0, tmp_uniq = 0;
  auto cleanup = [&]() {
    if (k1) cudaFree(k1);
    if (k2) cudaFree(k2);
    if (d_nsel) cudaFree(d_nsel);
    if (tmp) cudaFree(tmp);
  };
  const int n_items = (int)(total > 0 ? total : 0);
  if (cudaMalloc(&k1, sizeof(int64_t) * (total + 1)) != cudaSuccess ||
      cudaMalloc(&k2, sizeof(int64_t) * (total + 1)) != cudaSuccess || cudaMalloc(&d_nsel, sizeof(int)) != cudaSuccess) {
    cleanup();
    set_error("pattern build: out of device memory for pair keys");
    return FEM_E_OOM;
  }
  k_pair_keys<<<grid_for(total), 256, 0, s>>>(m->conn, E, NL, N, m->own_lo, m->own_hi, sentinel, k1);
  cub::DoubleBuffer<int64_t> db(k1, k2);
  cub::DeviceRadixSort::SortKeys(nullptr, tmp_sort, db, n_items, 0, end_bit, s);
  cub::DeviceSelect::Unique(nullptr, tmp_uniq, k1, k2, d_nsel, n_items, s);
  if (cudaMalloc(&tmp, tmp_sort > tmp_uniq ? tmp_sort : tmp_uniq) != cudaSuccess) {
    cleanup();
    set_error("pattern build: out of device memory for sort scratch");
    return FEM_E_OOM;
  }
  cub::DeviceRadixSort::SortKeys(tmp, tmp_sort, db, n_items, 0, end_bit, s);
  int64_t* sorted = db.Current();
  int64_t* uniq = db.Alternate();
  cub::DeviceSelect::Unique(tmp, tmp_uniq, sorted, uniq, d_nsel, n_items, s);
  int h_nsel = 0;
  cudaError_t ce = cudaMemcpyAsync(&h_nsel, d_nsel, sizeof(int), cudaMemcpyDeviceToHost, s);
  if (ce == cudaSuccess) ce = cudaStreamSynchronize(s);
  if (ce != cudaSuccess) {
    cleanup();
    set_error(std::string("pattern build: ") + cudaGetErrorString(ce));
    return FEM_E_CUDA;
  }
  int64_t nnz_s = h_nsel;
  if (nnz_s > 0) {  // drop the sentinel (non-owned rows) if present
    int64_t last = 0;
    ce = cudaMemcpyAsync(&last, uniq + nnz_s - 1, sizeof(int64_t), cudaMemcpyDeviceToHost, s);
    if (ce == cudaSuccess) ce = cudaStreamSynchronize(s);
    if (ce != cudaSuccess) { cleanup(); set_error("pattern build: copy failed"); return FEM_E_CUDA; }
    if (last == sentinel) nnz_s--;
  }
  if (nnz_s >= ((int64_t)1 << 31)) {
    cleanup();
    set_error("pattern build: scalar nnz >= 2^31 does not fit the int32 slot map");
    return FEM_E_INDEX_OVERFLOW;
  }
  p->nnz_s = nnz_s;
  p->n_rows = (int64_t)KH * m->n_own;
  p->nnz = (int64_t)KH * KH * nnz_s;
  cudaError_t a1 = cudaMalloc(&p->rowptr_s, sizeof(int64_t) * (m->n_own + 1));
  cudaError_t a2 = cudaMalloc(&p->colidx_s, sizeof(int32_t) * (nnz_s + 1));
  cudaError_t a3 = cudaMalloc(&p->slot, sizeof(int32_t) * (total + 1));
  cudaError_t a4 = cudaMalloc(&p->rowptr, sizeof(int64_t) * (p->n_rows + 1));
  cudaError_t a5 = cudaMalloc(&p->colidx, sizeof(int32_t) * (p->nnz + 1));
  if (a1 || a2 || a3 || a4 || a5) {
    cleanup();
    set_error("pattern build: out of device memory for the CSR arrays");
    return FEM_E_OOM;
  }
  k_rowptr_s<<<grid_for(m->n_own + 1), 256, 0, s>>>(uniq, nnz_s, m->n_own, N, p->rowptr_s);
  k_colidx_s<<<grid_for(nnz_s), 256, 0, s>>>(uniq, nnz_s, N, p->colidx_s);
  k_slot<<<grid_for(total), 256, 0, s>>>(m->conn, E, NL, m->own_lo, m->own_hi, p->rowptr_s, p->colidx_s, p->slot);
  k_block_rowptr<<<grid_for(p->n_rows + 1), 256, 0, s>>>(p->rowptr_s, m->n_own, KH, nnz_s, p->rowptr);
  k_block_colidx<<<grid_for(nnz_s), 256, 0, s>>>(p->rowptr_s, p->colidx_s, m->n_own, nnz_s, KH, N, p->colidx);
  ce = cudaGetLastError();
  if (ce == cudaSuccess) ce = cudaStreamSynchronize(s);
  cleanup();
  if (ce != cudaSuccess) {
    set_error(std::string("pattern build kernels: ") + cudaGetErrorString(ce));
    return FEM_E_CUDA;
  }
  return 0;
}

// ---------------------------------------------------------------- residual norms (P:439 check)
// max|·| that propagates NaN (fmax drops it): an all-NaN residual must not pass a ‖d‖∞ < atol test.
__device__ __forceinline__ double nanmax_abs(double m, double v) {
  const double a = fabs(v);
  return (a != a || m != m || a > m) ? (m != m ? m : a) : m;
}

// Σd² and max|d| over n entries with a fixed grid (norm_blocks = 4 × SMs) and a fixed summation order:
// thread t of block b reads i = b·NT + t + k·(grid·NT) in order, then a fixed xor tree, warp totals in warp
// order, and the last-arriving block sums the block partials 0..grid-1 in order — bit-reproducible run to run
// (the round-1 kernel combined blocks with a global atomicAdd, whose order varied).
constexpr int NORM_NT = 256;
__global__ void __launch_bounds__(NORM_NT) k_norms(const double* __restrict__ d, int64_t n,
                                                   double* __restrict__ partials, unsigned int* __restrict__ ticket,
                                                   double* __restrict__ out) {
  __shared__ double ss[NORM_NT / 32], sm[NORM_NT / 32];
  __shared__ bool last;
  double s = 0.0, mx = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)NORM_NT + threadIdx.x; i < n; i += (int64_t)gridDim.x * NORM_NT) {
    const double v = __ldcs(d + i);
    s = fma(v, v, s);
    mx = nanmax_abs(mx, v);
  }
  for (int o = 16; o > 0; o >>= 1) {
    s += __shfl_xor_sync(0xffffffffu, s, o);
    mx = nanmax_abs(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  }
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) { ss[w] = s; sm[w] = mx; }
  __syncthreads();
  if (threadIdx.x == 0) {
    double b = 0.0, bm = 0.0;
    for (int k = 0; k < NORM_NT / 32; k++) { b += ss[k]; bm = nanmax_abs(bm, sm[k]); }
    partials[2 * blockIdx.x] = b;
    partials[2 * blockIdx.x + 1] = bm;
    __threadfence();
    last = atomicAdd(ticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  if (threadIdx.x == 0) {
    double b = 0.0, bm = 0.0;
    for (unsigned k = 0; k < gridDim.x; k++) {
      b += __ldcg(partials + 2 * k);
      bm = nanmax_abs(bm, __ldcg(partials + 2 * k + 1));
    }
    out[0] = b;
    out[1] = bm;
    *ticket = 0u;
  }
}

int residual_norms(const fem_mesh_s* m, const double* rhs, double* norms, cudaStream_t s) {
  const int64_t n = (int64_t)m->kh * m->n_own;
  if (n <= 0) {
    FEM_CUDA_TRY(cudaMemsetAsync(norms, 0, 2 * sizeof(double), s));
    return 0;
  }
  k_norms<<<m->norm_blocks, NORM_NT, 0, s>>>(rhs, n, m->norm_partials, m->norm_ticket, norms);
  FEM_CUDA_TRY(cudaGetLastError());
  return 0;
}

}  // namespace fem
