// coo.cu — NEXT-4: the paper's COO view of the assembled system and workpiece offsets.
//
// B-4 numbers the global entries by a sparse ID over symbol pairs (κ₀, κ_λ) (A-3)
// times control-point pairs (α₁, α₂) (B-1 item 4), with I = (κ₀-1)α̂ + α₁ and
// J = (κ_λ-1)α̂ + α₂ (0-based here).  Reading L4 orders both pair sets lexicographically, so
// sparse ID = (κ₀ κ̂ + κ_λ) nnz_s + s with s the scalar-CSR slot of (α₁, α₂): the COO is a pure
// permutation of the κ-major block CSR (every κ₀ couples to all κ̂ components, reading L6), computed
// here by index arithmetic, one thread per entry.  Several workpieces form a block-diagonal system with
// the offsets n^dense (rows) and n^sp (sparse IDs): the caller passes the row offset and writes
// each workpiece's entries at its n^sp.
#include <cstdint>

#include "fem_internal.cuh"

namespace fem {

__global__ void k_coo(int64_t nnz, int64_t nnz_s, int kh, int64_t N, int64_t own_lo, const int64_t* __restrict__ rowptr_s,
                      const int32_t* __restrict__ colidx_s, int64_t n_own, int64_t row_offset, int64_t* __restrict__ I,
                      int64_t* __restrict__ J, int64_t* __restrict__ csr) {
  for (int64_t id = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; id < nnz; id += (int64_t)gridDim.x * blockDim.x) {
    const int64_t pair = id / nnz_s, s = id - pair * nnz_s;
    const int k0 = (int)(pair / kh), kl = (int)(pair - (int64_t)k0 * kh);
    int64_t lo = 0, hi = n_own;  // owned scalar row a1 with rowptr_s[a1] <= s < rowptr_s[a1 + 1]
    while (hi - lo > 1) {
      const int64_t mid = (lo + hi) >> 1;
      if (rowptr_s[mid] <= s) lo = mid;
      else hi = mid;
    }
    const int64_t a1 = lo, r0 = rowptr_s[a1], deg = rowptr_s[a1 + 1] - r0;
    if (I) I[id] = row_offset + (int64_t)k0 * N + own_lo + a1;
    if (J) J[id] = row_offset + (int64_t)kl * N + colidx_s[s];
    if (csr) csr[id] = (int64_t)k0 * kh * nnz_s + (int64_t)kh * r0 + (int64_t)kl * deg + (s - r0);
  }
}

__global__ void k_gather(int64_t n, const int64_t* __restrict__ idx, const double* __restrict__ src, double* __restrict__ dst) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = src[idx[i]];
}

}  // namespace fem

using namespace fem;

extern "C" int fem_pattern_export_coo(fem_pattern_t p, int64_t row_offset, int64_t* I, int64_t* J, int64_t* csr_index,
                                      void* stream) {
  if (!p || (!I && !J && !csr_index) || row_offset < 0) {
    set_error("fem_pattern_export_coo: invalid argument");
    return FEM_E_INVALID_ARG;
  }
  const fem_mesh_s* m = p->mesh;
  if (p->nnz == 0) return 0;
  const int64_t blocks = std::min<int64_t>((p->nnz + 255) / 256, 148 * 16);
  k_coo<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(p->nnz, p->nnz_s, m->kh, m->N, m->own_lo, p->rowptr_s, p->colidx_s,
                                                            m->n_own, row_offset, I, J, csr_index);
  FEM_CUDA_TRY(cudaGetLastError());
  return 0;
}

extern "C" int fem_gather(int64_t n, const int64_t* index, const double* src, double* dst, void* stream) {
  if (n < 0 || (n > 0 && (!index || !src || !dst))) {
    set_error("fem_gather: invalid argument");
    return FEM_E_INVALID_ARG;
  }
  if (n == 0) return 0;
  const int64_t blocks = std::min<int64_t>((n + 255) / 256, 148 * 16);
  k_gather<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(n, index, src, dst);
  FEM_CUDA_TRY(cudaGetLastError());
  return 0;
}
