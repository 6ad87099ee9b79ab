// stored.cuh — device side of FEM_SCATTER_STORED (stored.cu): the per-slot gather of one owned row and the
// dataflow loop of the fused ("flow") element + gather kernels.
//
// The flow kernels run the two halves of D-2/D-3 in ONE persistent launch: a ticket counter
// hands out, in a precomputed order, element items (EI consecutive elements of the Morton element order, one warp:
// compute the local blocks, store them) and row items (RI owned rows, one warp: sum their CSR entries from the stored
// blocks).  A row item is scheduled a lag after the last element item it reads and waits on the completion
// counters of its element range, so the blocks it reads were written a few tens of MB earlier and are still
// in the 126 MB L2: the scratch is written once and read from L2, not from HBM.  Element items never wait and a row
// item only waits on items with smaller tickets, all already taken by running CTAs: no deadlock, no
// co-residency requirement.  Blocks are read with ld.global.cg (L2) because a line may be shared by two
// element items and an L1 copy of it could predate the second writer.
#pragma once
#include <climits>
#include <cstdint>

namespace fem {

struct FlowParams {
  const int32_t* sched;   // ticket -> item: >= 0 element item, < 0 row item -1 - g
  int64_t n_items;
  const int32_t* dep;     // [n_row_items][2]: first and last element item a row item reads
  uint32_t* done;         // [ceil(n_elem_items / FLOW_SB)]: finished element items per superblock (zeroed)
  int64_t n_ei;
  uint32_t* ticket;       // zeroed before every launch
  int ei, ri;             // elements per element item, rows per row item
  int64_t E, n_own, nnz_s;
  const int32_t* eperm;   // position -> element
  const int32_t* rows;    // owned rows in row-item order
  const int64_t* rowptr_s;
  const uint32_t* off;    // [nnz_s + 1] contribution list offsets
  const uint32_t* ent;    // (pos·NB + blk) << 1 | transposed
  const uint32_t* roff;   // [n_own + 1] residual list offsets
  const uint32_t* rent;   // pos·NL + a
  const int32_t* bmap;    // element -> boundary-storage index or -1 (null: no boundary terms)
  const double* fk;       // boundary-term blocks [n_bnd][NB][KH][KH]
  const double* fr;       // boundary-term residual rows [n_bnd][NL][KH]
  double* ek;
  double* er;
  double* values;
  double* rhs;
};

// Completion is counted per superblock of FLOW_SB element items (one counter read covers FLOW_SB items);
// a row item waits for whole superblocks, which is deadlock-free because the schedule places it at least
// FLOW_SB element items after the last item it reads, so every item of those superblocks has a smaller ticket.
constexpr int FLOW_SB = 64;

__device__ __forceinline__ uint32_t st_ld_acquire_gpu(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_red_release_gpu(uint32_t* p, uint32_t v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Stored block stride (doubles): κ̂² values padded to whole 32-byte sectors, so that a block is read with
// 256-bit loads (3 for κ̂ = 3 instead of 9 scalar loads: the gather is bound by L1 wavefronts, one per
// load instruction and distinct line).
__host__ __device__ constexpr int st_bs(int KH) { return KH == 1 ? 1 : (KH * KH + 3) / 4 * 4; }

template <bool LDCG>
__device__ __forceinline__ void st_ld4(const double* p, double& a, double& b, double& c, double& d) {
  if constexpr (LDCG)
    asm volatile("ld.global.cg.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(a), "=d"(b), "=d"(c), "=d"(d) : "l"(p));
  else
    asm volatile("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(a), "=d"(b), "=d"(c), "=d"(d) : "l"(p));
}
template <int KH, bool LDCG>
__device__ __forceinline__ void st_ld_block(const double* src, double (&v)[st_bs(KH)]) {
  if constexpr (KH == 1) {
    v[0] = LDCG ? __ldcg(src) : __ldg(src);
  } else {
#pragma unroll
    for (int q = 0; q < st_bs(KH) / 4; q++) st_ld4<LDCG>(src + 4 * q, v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
  }
}
__device__ __forceinline__ void st_st4(double* p, double a, double b, double c, double d) {
  asm volatile("st.global.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(p), "d"(a), "d"(b), "d"(c), "d"(d) : "memory");
}

// One owned row li (global order of the warp): lane per CSR slot of the row, the slot's stored blocks summed
// in list order (GU per trip, loads first), κ̂² values written.  LDCG: blocks through L2 (see above).
template <int KH, bool LDCG>
__device__ __forceinline__ void st_gather_row(int64_t li, const int64_t* __restrict__ rowptr_s, int64_t nnz_s,
                                              const uint32_t* __restrict__ off, const uint32_t* __restrict__ ent,
                                              const double* ek, double* __restrict__ values) {
  const int lane = threadIdx.x & 31;
  const int64_t rps = rowptr_s[li], deg = rowptr_s[li + 1] - rps;
  for (int64_t o = lane; o < deg; o += 32) {
    const int64_t s = rps + o;
    double acc[KH * KH];
#pragma unroll
    for (int k = 0; k < KH * KH; k++) acc[k] = 0.0;
    const uint32_t j0 = LDCG ? __ldcs(off + s) : __ldg(off + s), j1 = LDCG ? __ldcs(off + s + 1) : __ldg(off + s + 1);
    constexpr int GU = KH >= 3 ? 2 : 4;
    for (uint32_t j = j0; j < j1; j += GU) {
      uint32_t x[GU];
#pragma unroll
      for (int u = 0; u < GU; u++) x[u] = j + u < j1 ? (LDCG ? __ldcs(ent + j + u) : __ldg(ent + j + u)) : 0u;
      double v[GU][st_bs(KH)];
#pragma unroll
      for (int u = 0; u < GU; u++) {
        // past the list end: block 0 (a valid address; the values are not added)
        const double* src = ek + (int64_t)(j + u < j1 ? (x[u] >> 1) : 0u) * st_bs(KH);
        st_ld_block<KH, LDCG>(src, v[u]);
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

// Residual row li: lane k < KH sums component k over the row's (pos·NL + a) list.
template <int KH, bool LDCG>
__device__ __forceinline__ void st_res_row(int64_t li, int64_t n_own, const uint32_t* __restrict__ roff,
                                           const uint32_t* __restrict__ rent, const double* er, double* __restrict__ rhs) {
  const int lane = threadIdx.x & 31;
  if (lane < KH) {
    double acc = 0.0;
    const uint32_t j1 = __ldg(roff + li + 1);
    for (uint32_t j = __ldg(roff + li); j < j1; j++) {
      const double* src = er + (int64_t)__ldg(rent + j) * KH + lane;
      acc += LDCG ? __ldcg(src) : __ldg(src);
    }
    rhs[(int64_t)lane * n_own + li] = acc;
  }
}

// L2 eviction-priority hints: the stored blocks are written and read back with evict_last (they must survive
// the LAG window), the streaming traffic (lists, CSR values) goes evict_first.
__device__ __forceinline__ uint64_t st_policy_evict_last() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void st_store_keep(double* p, double v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(p), "d"(v), "l"(pol) : "memory");
}

// The dataflow loop, per warp: lane 0 takes a ticket; element items (elem_item(item) with this warp) are
// published by a release increment of their superblock counter; row items wait for their superblocks, then
// gather their rows.  No CTA barrier: the warps of a CTA run independent items.
template <int KH, class ElemItem>
__device__ __forceinline__ void flow_loop(const FlowParams& F, ElemItem&& elem_item) {
  const int lane = threadIdx.x & 31;
  for (;;) {
    int item = INT_MIN;
    if (lane == 0) {
      const uint32_t t = atomicAdd(F.ticket, 1u);
      item = (int64_t)t < F.n_items ? __ldg(F.sched + t) : INT_MIN;
    }
    item = __shfl_sync(0xffffffffu, item, 0);
    if (item == INT_MIN) break;
    if (item >= 0) {
      elem_item(item);
      __syncwarp();
      if (lane == 0) {
        __threadfence();
        st_red_release_gpu(F.done + item / FLOW_SB, 1u);
      }
    } else {
      const int g = -1 - item;
      const int lo = __ldg(F.dep + 2 * g) / FLOW_SB, hi = __ldg(F.dep + 2 * g + 1) / FLOW_SB;
      for (int j = lo + lane; j <= hi; j += 32) {
        const int64_t rest = F.n_ei - (int64_t)j * FLOW_SB;
        const uint32_t full = (uint32_t)(rest < FLOW_SB ? rest : FLOW_SB);
        while (st_ld_acquire_gpu(F.done + j) != full) __nanosleep(64);
      }
      __syncwarp();
      const int64_t r0 = (int64_t)g * F.ri;
      for (int k = 0; k < F.ri; k++) {
        const int64_t w = r0 + k;
        if (w >= F.n_own) break;
        const int64_t li = __ldg(F.rows + w);
        if (F.values) st_gather_row<KH, true>(li, F.rowptr_s, F.nnz_s, F.off, F.ent, F.ek, F.values);
        if (F.rhs) st_res_row<KH, true>(li, F.n_own, F.roff, F.rent, F.er, F.rhs);
      }
    }
  }
}

}  // namespace fem
