// stored.cuh — device side of FEM_SCATTER_STORED (stored.cu): the per-slot gather of one owned row and its
// residual row, and the 256-bit load/store helpers shared with the element passes (tet1_ns.cu).
#pragma once
#include <cstdint>

namespace fem {

// Stored block stride (doubles): the κ̂² values of a block, contiguous.
__host__ __device__ constexpr int st_bs(int KH) { return KH * KH; }

__device__ __forceinline__ void st_st4(double* p, double a, double b, double c, double d) {
  asm volatile("st.global.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(p), "d"(a), "d"(b), "d"(c), "d"(d) : "memory");
}
__device__ __forceinline__ void st_ld4(const double* p, double& a, double& b, double& c, double& d) {
  asm volatile("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(a), "=d"(b), "=d"(c), "=d"(d) : "l"(p));
}

// One owned row li per W lanes (W = 32, or 8 for short rows: four rows per warp): lane per CSR slot of the
// row, the slot's stored blocks summed in list order (GU per trip, all loads first), κ̂² values written.
template <int KH, int W = 32>
__device__ __forceinline__ void st_gather_row(int64_t li, const int64_t* __restrict__ rowptr_s, int64_t nnz_s,
                                              const uint32_t* __restrict__ off, const uint32_t* __restrict__ ent,
                                              const double* ek, double* __restrict__ values) {
  const int lane = threadIdx.x & (W - 1);
  const int64_t rps = rowptr_s[li], deg = rowptr_s[li + 1] - rps;
  for (int64_t o = lane; o < deg; o += W) {
    const int64_t s = rps + o;
    double acc[KH * KH];
#pragma unroll
    for (int k = 0; k < KH * KH; k++) acc[k] = 0.0;
    const uint32_t j0 = __ldg(off + s), j1 = __ldg(off + s + 1);
    constexpr int GU = KH >= 3 ? 2 : 4;  // (κ̂ = 4: 32 doubles in flight)
    for (uint32_t j = j0; j < j1; j += GU) {
      uint32_t x[GU];
#pragma unroll
      for (int u = 0; u < GU; u++) x[u] = j + u < j1 ? __ldg(ent + j + u) : 0u;
      double v[GU][st_bs(KH)];
#pragma unroll
      for (int u = 0; u < GU; u++) {
        // past the list end: block 0 (a valid address; the values are not added)
        const double* src = ek + (int64_t)(j + u < j1 ? (x[u] >> 1) : 0u) * st_bs(KH);
        if constexpr (KH * KH % 4 == 0) {  // κ̂ = 2, 4: blocks are whole 32-byte sectors, 256-bit loads
#pragma unroll
          for (int q = 0; q < KH * KH / 4; q++) st_ld4(src + 4 * q, v[u][4 * q], v[u][4 * q + 1], v[u][4 * q + 2], v[u][4 * q + 3]);
        } else {
#pragma unroll
          for (int k = 0; k < KH * KH; k++) v[u][k] = __ldg(src + k);
        }
      }
#pragma unroll
      for (int u = 0; u < GU; u++) {
        if (j + u >= j1) break;
        const bool tr = x[u] & 1u;
#pragma unroll
        for (int k0 = 0; k0 < KH; k0++)
#pragma unroll
          for (int kl = 0; kl < KH; kl++) acc[k0 * KH + kl] += tr ? v[u][kl * KH + k0] : v[u][k0 * KH + kl];
      }
    }
    double* dst = values + (int64_t)KH * rps + o;
#pragma unroll
    for (int k0 = 0; k0 < KH; k0++)
#pragma unroll
      for (int kl = 0; kl < KH; kl++) __stcs(dst + (int64_t)k0 * KH * nnz_s + kl * deg, acc[k0 * KH + kl]);
  }
}

// Residual row li (W lanes per row; li < 0: no row, the lanes still take part in the shuffles): lane j
// takes entries j, j + W, ... of the row's (pos·NL + a) list; the κ̂ components are then reduced over the
// row's lanes by a fixed butterfly (deterministic) and its first lane writes them.  Called by all 32 lanes.
template <int KH, int W = 32>
__device__ __forceinline__ void st_res_row(int64_t li, int64_t n_own, const uint32_t* __restrict__ roff,
                                           const uint32_t* __restrict__ rent, const double* er, double* __restrict__ rhs) {
  const int lane = threadIdx.x & (W - 1);
  double acc[KH];
#pragma unroll
  for (int k = 0; k < KH; k++) acc[k] = 0.0;
  if (li >= 0) {
    const uint32_t j1 = __ldg(roff + li + 1);
    for (uint32_t j = __ldg(roff + li) + lane; j < j1; j += W) {
      const double* src = er + (int64_t)__ldg(rent + j) * KH;
#pragma unroll
      for (int k = 0; k < KH; k++) acc[k] += __ldg(src + k);
    }
  }
#pragma unroll
  for (int o = W / 2; o; o >>= 1)
#pragma unroll
    for (int k = 0; k < KH; k++) acc[k] += __shfl_xor_sync(0xffffffffu, acc[k], o);
  if (lane == 0 && li >= 0) {
#pragma unroll
    for (int k = 0; k < KH; k++) rhs[(int64_t)k * n_own + li] = acc[k];
  }
}

}  // namespace fem
