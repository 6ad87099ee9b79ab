// solve.cu — NEXT-1: the linear solve of the Newton sub-step on the GPU.
//
// PAPER.md D-4 solves the assembled system for the increment, K Δφ = -d (the
// linearisation of d(φ) = 0), then updates the control-point values.  For the thermal and elasticity
// forms K is symmetric and, with the paper's sign convention (reading L17), negative definite once the
// penalty terms fix the rigid modes, so s·K with s = -1 is symmetric positive definite and the solve is
// Jacobi-preconditioned conjugate gradients on (s K) x = s b.  The kernels are HBM-bound sparse/vector
// passes over the CSR of fem_pattern_build: the SpMV moves 12 B per nnz (fp64 value + int32 column) and
// the vector updates a few doubles per row.  Dot products reduce per block into a partials array whose
// last-arriving block sums it in fixed order, so every iteration is bit-identical run to run.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdlib>

#include "fem_internal.cuh"

namespace fem {

constexpr int SV_THREADS = 256;
constexpr int SV_MAX_BLOCKS = 148 * 8;  // vector kernels: persistent grid, a multiple of the SM count

// device scalars of one CG solve (in the caller's work buffer after the 5 vectors)
struct CgScal {
  double rz, rz_new, pq, rr, rr0, alpha, beta;
  unsigned int count0, count1;  // last-block tickets of the two reducing kernels
};

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Block-sum of v, then the last block to arrive sums the per-block partials in a fixed order.
// Returns true in thread 0 of that last block, with *out written.
template <int NT = SV_THREADS>
__device__ __forceinline__ bool block_reduce_last(double v, double* partials, unsigned int* ticket, double* out) {
  __shared__ double ws[NT / 32];
  __shared__ bool last;
  v = warp_sum(v);
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double b = 0.0;
    for (int i = 0; i < NT / 32; i++) b += ws[i];
    partials[blockIdx.x] = b;
    __threadfence();
    last = atomicAdd(ticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return false;
  __threadfence();
  // the whole last block sums the partials: thread j takes blocks j, j+NT, … in order, then the fixed
  // xor tree and the warp totals in warp order — a fixed order (bit-reproducible) without a 1000-long
  // serial chain of L2 loads in one thread
  double t = 0.0;
  for (unsigned i = threadIdx.x; i < gridDim.x; i += NT) t += __ldcg(partials + i);
  t = warp_sum(t);
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = t;  // thread 0 finished reading ws before the barrier
  __syncthreads();
  if (threadIdx.x == 0) {
    double b = 0.0;
    for (int i = 0; i < NT / 32; i++) b += ws[i];
    *out = b;
    *ticket = 0u;
  }
  return threadIdx.x == 0;
}

// y = alpha K x + beta y: G lanes per row (default G = 32: an 81-entry Q1 elasticity row is three
// independent loads per lane), lanes read consecutive entries of the row, (sub-)warp shuffle reduction.  The row loop is uniform per
// warp (32 / G rows per warp and step), so the shuffles never see an exited lane.
template <int G>
__device__ __forceinline__ double row_dot(int64_t r, int64_t n, int sub, const int64_t* __restrict__ rowptr,
                                          const int32_t* __restrict__ colidx, const double* __restrict__ val,
                                          const double* __restrict__ x) {
  double acc = 0.0;
  if (r < n) {
    const int64_t e = rowptr[r + 1];
    int64_t k = rowptr[r] + sub;
    if constexpr (G <= 16) {
      // predicated: a short row's loads all issue in one trip (c2 transient 14.0 -> 13.6 ms per timestep;
      // for G = 32 on 81-entry rows the peeled loop below was faster)
      for (; k < e; k += 4 * G) {
        double v[4];
        int32_t c[4];
#pragma unroll
        for (int j = 0; j < 4; j++) {
          v[j] = k + j * G < e ? __ldcs(val + k + j * G) : 0.0;
          c[j] = k + j * G < e ? __ldcs(colidx + k + j * G) : -1;
        }
#pragma unroll
        for (int j = 0; j < 4; j++)
          if (c[j] >= 0) acc = fma(v[j], __ldg(x + c[j]), acc);
      }
    } else {
      for (; k + 3 * G < e; k += 4 * G) {  // four independent loads in flight per lane
        const double v0 = __ldcs(val + k), v1 = __ldcs(val + k + G), v2 = __ldcs(val + k + 2 * G), v3 = __ldcs(val + k + 3 * G);
        const int32_t c0 = __ldcs(colidx + k), c1 = __ldcs(colidx + k + G), c2 = __ldcs(colidx + k + 2 * G),
                      c3 = __ldcs(colidx + k + 3 * G);
        acc = fma(v0, __ldg(x + c0), acc);
        acc = fma(v1, __ldg(x + c1), acc);
        acc = fma(v2, __ldg(x + c2), acc);
        acc = fma(v3, __ldg(x + c3), acc);
      }
      for (; k < e; k += G) acc = fma(__ldcs(val + k), __ldg(x + __ldcs(colidx + k)), acc);
    }
  }
#pragma unroll
  for (int o = G / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o, G);
  return acc;
}

// G = 0: a warp owns 32 consecutive rows.  Lane i loads rowptr[r0+i] (one coalesced load, no rowptr
// latency per row), then the warp walks its rows two at a time, each lane issuing up to 6 predicated
// value/column loads per trip (3 strided chunks per row: a c5 row of 81 entries is one trip) so two
// rows' loads are in flight together.  Per-lane sums and the xor tree are the G = 32 order, so
// results are bit-identical to row_dot<32>.  Lane i returns row r0+i's dot.
template <int R>
__device__ __forceinline__ double rows32_dot(int64_t r0, int64_t n, int lane, const int64_t* __restrict__ rowptr,
                                             const int32_t* __restrict__ colidx, const double* __restrict__ val,
                                             const double* __restrict__ x) {
  const int64_t b = rowptr[r0 + lane < n ? r0 + lane : n], e = rowptr[r0 + lane + 1 < n ? r0 + lane + 1 : n];
  double mine = 0.0;
  for (int i = 0; i < 32; i += R) {
    int64_t s0[R], l0[R], len = 0;
    double a[R];
#pragma unroll
    for (int q = 0; q < R; q++) {
      s0[q] = __shfl_sync(0xffffffffu, b, i + q);
      l0[q] = __shfl_sync(0xffffffffu, e, i + q) - s0[q];
      len = l0[q] > len ? l0[q] : len;
      a[q] = 0.0;
    }
    for (int64_t off = lane; off < len; off += 96) {
      double v[3 * R];
      int32_t c[3 * R];
#pragma unroll
      for (int q = 0; q < R; q++)
#pragma unroll
        for (int j = 0; j < 3; j++) {
          const int64_t o = off + 32 * j;
          v[3 * q + j] = o < l0[q] ? __ldcs(val + s0[q] + o) : 0.0;
          c[3 * q + j] = o < l0[q] ? __ldcs(colidx + s0[q] + o) : -1;
        }
#pragma unroll
      for (int j = 0; j < 3; j++)
#pragma unroll
        for (int q = 0; q < R; q++)
          if (c[3 * q + j] >= 0) a[q] = fma(v[3 * q + j], __ldg(x + c[3 * q + j]), a[q]);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
#pragma unroll
      for (int q = 0; q < R; q++) a[q] += __shfl_xor_sync(0xffffffffu, a[q], o);
#pragma unroll
    for (int q = 0; q < R; q++)
      if (lane == i + q) mine = a[q];
  }
  return mine;
}
#ifndef FEM_SPMV_R
#define FEM_SPMV_R 2
#endif
template <int G>
__device__ __forceinline__ double rows_dot(int64_t r0, int64_t r, int64_t n, int sub, int lane,
                                           const int64_t* __restrict__ rowptr, const int32_t* __restrict__ colidx,
                                           const double* __restrict__ val, const double* __restrict__ x) {
  if constexpr (G == 0) return rows32_dot<FEM_SPMV_R>(r0, n, lane, rowptr, colidx, val, x);
  else return row_dot<G>(r, n, sub, rowptr, colidx, val, x);
}
template <int G>
__global__ void __launch_bounds__(SV_THREADS) k_spmv(int64_t n, const int64_t* __restrict__ rowptr,
                                                     const int32_t* __restrict__ colidx,
                                                     const double* __restrict__ val, const double* __restrict__ x,
                                                     double* __restrict__ y, double alpha, double beta) {
  constexpr int RPW = G ? 32 / (G ? G : 1) : 32;  // rows per warp and step
  const int lane = threadIdx.x & 31, sub = G ? lane % (G ? G : 1) : 0;
  const int64_t nwarps = (int64_t)gridDim.x * (SV_THREADS / 32);
  for (int64_t w = ((int64_t)blockIdx.x * SV_THREADS + threadIdx.x) / 32; w * RPW < n; w += nwarps) {
    const int64_t r = w * RPW + (G ? lane / (G ? G : 1) : lane);
    const double acc = rows_dot<G>(w * RPW, r, n, sub, lane, rowptr, colidx, val, x);
    if (sub == 0 && r < n) y[r] = alpha * acc + (beta == 0.0 ? 0.0 : beta * y[r]);
  }
}

// q = s K p and pq = p·q
template <int G>
__global__ void __launch_bounds__(SV_THREADS) k_cg_spmv(int64_t n, const int64_t* __restrict__ rowptr,
                                                        const int32_t* __restrict__ colidx,
                                                        const double* __restrict__ val, double s,
                                                        const double* __restrict__ p, double* __restrict__ q,
                                                        double* partials, CgScal* sc) {
  constexpr int RPW = G ? 32 / (G ? G : 1) : 32;
  const int lane = threadIdx.x & 31, sub = G ? lane % (G ? G : 1) : 0;
  const int64_t nwarps = (int64_t)gridDim.x * (SV_THREADS / 32);
  double dot = 0.0;
  for (int64_t w = ((int64_t)blockIdx.x * SV_THREADS + threadIdx.x) / 32; w * RPW < n; w += nwarps) {
    const int64_t r = w * RPW + (G ? lane / (G ? G : 1) : lane);
    const double acc = rows_dot<G>(w * RPW, r, n, sub, lane, rowptr, colidx, val, p);
    if (sub == 0 && r < n) {
      const double qr = s * acc;
      q[r] = qr;
      dot = fma(p[r], qr, dot);
    }
  }
  double pq;
  if (block_reduce_last(dot, partials, &sc->count0, &pq)) {
    sc->pq = pq;
    sc->rz = sc->rz_new;  // every block of the previous k_cg_dir has used the old rz (stream order)
    // breakdown guard: p·q = 0 (p = 0 after exact convergence inside a check block, or a zero-energy
    // direction) leaves x unchanged instead of spreading 0/0 into it
    sc->alpha = pq != 0.0 ? sc->rz / pq : 0.0;
  }
}

// x += α p, r -= α q, z = D^-1 r; rz_new = r·z and rr = r·r (two reductions through one partials row each)
__global__ void __launch_bounds__(SV_THREADS) k_cg_update(int64_t n, double* __restrict__ x, double* __restrict__ r,
                                                          const double* __restrict__ p, const double* __restrict__ q,
                                                          const double* __restrict__ dinv, double* __restrict__ z,
                                                          double* partials, CgScal* sc) {
  const double alpha = sc->alpha;
  double rz = 0.0, rr = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * SV_THREADS + threadIdx.x; i < n; i += (int64_t)gridDim.x * SV_THREADS) {
    x[i] = fma(alpha, p[i], x[i]);
    const double ri = fma(-alpha, q[i], r[i]);
    r[i] = ri;
    const double zi = dinv[i] * ri;
    z[i] = zi;
    rz = fma(ri, zi, rz);
    rr = fma(ri, ri, rr);
  }
  // pack the two sums: reduce rz into partials[0..grid), rr into partials[grid..2 grid)
  double out;
  if (block_reduce_last(rz, partials, &sc->count0, &out)) {
    sc->rz_new = out;
  }
  __syncthreads();
  if (block_reduce_last(rr, partials + gridDim.x, &sc->count1, &out)) {
    sc->rr = out;
  }
}

// p = z + β p with β = rz_new / rz (rz ← rz_new happens in the next k_cg_spmv)
__global__ void __launch_bounds__(SV_THREADS) k_cg_dir(int64_t n, const double* __restrict__ z, double* __restrict__ p,
                                                       CgScal* sc, int first) {
  const double beta = (first || sc->rz == 0.0) ? 0.0 : sc->rz_new / sc->rz;
  for (int64_t i = (int64_t)blockIdx.x * SV_THREADS + threadIdx.x; i < n; i += (int64_t)gridDim.x * SV_THREADS)
    p[i] = first ? z[i] : fma(beta, p[i], z[i]);
}

// r = b - s K x (x the initial guess), z = D^-1 r, dinv from the diagonal of s K
__global__ void __launch_bounds__(SV_THREADS) k_cg_init(int64_t n, const int64_t* __restrict__ rowptr,
                                                        const int32_t* __restrict__ colidx,
                                                        const double* __restrict__ val, double s,
                                                        const double* __restrict__ b, const double* __restrict__ x,
                                                        double* __restrict__ r, double* __restrict__ z,
                                                        double* __restrict__ dinv, double* partials, CgScal* sc,
                                                        int* bad_diag) {
  double rz = 0.0, rr = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * SV_THREADS + threadIdx.x; i < n; i += (int64_t)gridDim.x * SV_THREADS) {
    double ax = 0.0, dg = 0.0;
    for (int64_t k = rowptr[i]; k < rowptr[i + 1]; k++) {
      const int32_t c = colidx[k];
      ax = fma(val[k], x[c], ax);
      if (c == i) dg = val[k];
    }
    dg *= s;
    if (!(dg > 0.0)) atomicExch(bad_diag, 1);
    const double di = 1.0 / dg;
    dinv[i] = di;
    const double ri = s * b[i] - s * ax;
    r[i] = ri;
    z[i] = di * ri;
    rz = fma(ri, di * ri, rz);
    rr = fma(ri, ri, rr);
  }
  double out;
  if (block_reduce_last(rz, partials, &sc->count0, &out)) {
    sc->rz_new = out;
  }
  __syncthreads();
  if (block_reduce_last(rr, partials + gridDim.x, &sc->count1, &out)) {
    sc->rr = out;
    sc->rr0 = out;
  }
}

// ---- Jacobi-preconditioned BiCGStab (van der Vorst) for the non-symmetric systems: the thermal FIX term
// k N_a n·∇T and the NS forms make K non-symmetric, so CG does not apply.
// Vectors in the work buffer: r, rh (shadow residual), p, v, y, s, z, t, dinv; scalars in BiScal.
struct BiScal {
  double rho, rho_new, alpha, omega, rv, ts, tt, rr, rr0;
  unsigned int count0, count1;
};

// p = r + β (p - ω v), β = (ρ_new / ρ)(α / ω); y = D^-1 p   (first: p = r)
__global__ void __launch_bounds__(SV_THREADS) k_bi_dir(int64_t n, const double* __restrict__ r, double* __restrict__ p,
                                                       const double* __restrict__ v, const double* __restrict__ dinv,
                                                       double* __restrict__ y, const BiScal* sc, int first) {
  // breakdown guards (ρ = 0 or ω = 0): restart the direction from r instead of propagating NaN
  const bool restart = first || sc->rho == 0.0 || sc->omega == 0.0;
  const double beta = restart ? 0.0 : (sc->rho_new / sc->rho) * (sc->alpha / sc->omega), om = sc->omega;
  for (int64_t i = (int64_t)blockIdx.x * SV_THREADS + threadIdx.x; i < n; i += (int64_t)gridDim.x * SV_THREADS) {
    const double pi = restart ? r[i] : fma(beta, p[i] - om * v[i], r[i]);
    p[i] = pi;
    y[i] = dinv[i] * pi;
  }
}

// out = A in (A = K), and (a · out) [, (out · out)] reduced; the last block forms α or ω
template <int G, int MODE>  // MODE 0: v = A y, α = ρ_new / (rh·v);  MODE 1: t = A z, ω = (t·s)/(t·t)
__global__ void __launch_bounds__(SV_THREADS) k_bi_spmv(int64_t n, const int64_t* __restrict__ rowptr,
                                                        const int32_t* __restrict__ colidx,
                                                        const double* __restrict__ val, const double* __restrict__ in,
                                                        double* __restrict__ out, const double* __restrict__ a,
                                                        double* partials, BiScal* sc) {
  constexpr int RPW = G ? 32 / (G ? G : 1) : 32;
  const int lane = threadIdx.x & 31, sub = G ? lane % (G ? G : 1) : 0;
  const int64_t nwarps = (int64_t)gridDim.x * (SV_THREADS / 32);
  double d0 = 0.0, d1 = 0.0;
  for (int64_t w = ((int64_t)blockIdx.x * SV_THREADS + threadIdx.x) / 32; w * RPW < n; w += nwarps) {
    const int64_t r = w * RPW + (G ? lane / (G ? G : 1) : lane);
    const double acc = rows_dot<G>(w * RPW, r, n, sub, lane, rowptr, colidx, val, in);
    if (sub == 0 && r < n) {
      out[r] = acc;
      d0 = fma(a[r], acc, d0);
      if (MODE == 1) d1 = fma(acc, acc, d1);
    }
  }
  double o;
  if (block_reduce_last(d0, partials, &sc->count0, &o)) {
    if (MODE == 0) {
      sc->rv = o;
      sc->rho = sc->rho_new;  // k_bi_dir of this iteration has used the old ρ (stream order)
      sc->alpha = o != 0.0 ? sc->rho / o : 0.0;
    } else {
      sc->ts = o;
    }
  }
  if (MODE == 1) {
    __syncthreads();
    if (block_reduce_last(d1, partials + gridDim.x, &sc->count1, &o)) {
      sc->tt = o;
      sc->omega = o != 0.0 ? sc->ts / o : 0.0;
    }
  }
}

// x += α y; s = r - α v; z = D^-1 s
__global__ void __launch_bounds__(SV_THREADS) k_bi_half(int64_t n, double* __restrict__ x, const double* __restrict__ y,
                                                        const double* __restrict__ r, const double* __restrict__ v,
                                                        const double* __restrict__ dinv, double* __restrict__ sv,
                                                        double* __restrict__ z, const BiScal* sc) {
  const double al = sc->alpha;
  for (int64_t i = (int64_t)blockIdx.x * SV_THREADS + threadIdx.x; i < n; i += (int64_t)gridDim.x * SV_THREADS) {
    x[i] = fma(al, y[i], x[i]);
    const double si = fma(-al, v[i], r[i]);
    sv[i] = si;
    z[i] = dinv[i] * si;
  }
}

// x += ω z; r = s - ω t; ρ_new = rh·r, rr = r·r
__global__ void __launch_bounds__(SV_THREADS) k_bi_fin(int64_t n, double* __restrict__ x, const double* __restrict__ z,
                                                       const double* __restrict__ sv, const double* __restrict__ t,
                                                       const double* __restrict__ rh, double* __restrict__ r,
                                                       double* partials, BiScal* sc) {
  const double om = sc->omega;
  double d0 = 0.0, d1 = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * SV_THREADS + threadIdx.x; i < n; i += (int64_t)gridDim.x * SV_THREADS) {
    x[i] = fma(om, z[i], x[i]);
    const double ri = fma(-om, t[i], sv[i]);
    r[i] = ri;
    d0 = fma(rh[i], ri, d0);
    d1 = fma(ri, ri, d1);
  }
  double o;
  if (block_reduce_last(d0, partials, &sc->count0, &o)) sc->rho_new = o;
  __syncthreads();
  if (block_reduce_last(d1, partials + gridDim.x, &sc->count1, &o)) sc->rr = o;
}

// r = b - A x, rh = r, dinv = 1 / diag(A) (non-zero diagonal required), ρ_new = r·r = rr0
__global__ void __launch_bounds__(SV_THREADS) k_bi_init(int64_t n, const int64_t* __restrict__ rowptr,
                                                        const int32_t* __restrict__ colidx,
                                                        const double* __restrict__ val, const double* __restrict__ b,
                                                        const double* __restrict__ x, double* __restrict__ r,
                                                        double* __restrict__ rh, double* __restrict__ dinv,
                                                        double* partials, BiScal* sc, int* bad_diag) {
  double d0 = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * SV_THREADS + threadIdx.x; i < n; i += (int64_t)gridDim.x * SV_THREADS) {
    double ax = 0.0, dg = 0.0;
    for (int64_t k = rowptr[i]; k < rowptr[i + 1]; k++) {
      const int32_t c = colidx[k];
      ax = fma(val[k], x[c], ax);
      if (c == i) dg = val[k];
    }
    if (dg == 0.0) atomicExch(bad_diag, 1);
    dinv[i] = 1.0 / dg;
    const double ri = b[i] - ax;
    r[i] = ri;
    rh[i] = ri;
    d0 = fma(ri, ri, d0);
  }
  double o;
  if (block_reduce_last(d0, partials, &sc->count0, &o)) {
    sc->rho_new = o;
    sc->rr = o;
    sc->rr0 = o;
    sc->rho = 1.0;
    sc->alpha = 1.0;
    sc->omega = 1.0;
  }
}

// Row mapping of the SpMV kernels from the average row length (one 8-byte read + sync, next to the init
// sync the solvers already do): long rows (Q1 elasticity, 81 entries) take the warp-owned 32-row blocks
// (c5: 11.4 ms vs 12.8 for 32 lanes per row, 14.6 for 8), short rows (scalar Q1, 27) 8 lanes per row
// (c2 transient: 7% faster than the row blocks).
static int solver_lanes(const int64_t* rowptr, int64_t n, cudaStream_t s, int* g) {
  int64_t nnz = 0;
  FEM_CUDA_TRY(cudaMemcpyAsync(&nnz, rowptr + n, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  FEM_CUDA_TRY(cudaStreamSynchronize(s));
  *g = (n > 0 && nnz >= 48 * n) ? 0 : 8;
  return 0;
}

static int grid_for(int64_t n, int per_thread_rows) {
  const int64_t need = (n * per_thread_rows + SV_THREADS - 1) / SV_THREADS;
  return (int)std::max<int64_t>(1, std::min<int64_t>(need, SV_MAX_BLOCKS));
}

}  // namespace fem

using namespace fem;

extern "C" int fem_spmv(int64_t n_rows, const int64_t* rowptr, const int32_t* colidx, const double* values,
                        const double* x, double* y, double alpha, double beta, void* stream) {
  if (n_rows < 0 || (n_rows > 0 && (!rowptr || !colidx || !values || !x || !y))) {
    set_error("fem_spmv: invalid argument");
    return FEM_E_INVALID_ARG;
  }
  if (n_rows == 0) return 0;
  // no host sync here (the solvers pick the row mapping from the average row length): warp-owned 32-row blocks
  k_spmv<0><<<grid_for(n_rows, 1), SV_THREADS, 0, (cudaStream_t)stream>>>(n_rows, rowptr, colidx, values, x, y, alpha, beta);
  FEM_CUDA_TRY(cudaGetLastError());
  return 0;
}

// y = alpha x + beta y, each product and the sum correctly rounded (no FMA contraction): the Newton update
// φ ← φ - Δ of D-4 and the sign flips around the solves, done in the library not the binding.
__global__ void __launch_bounds__(SV_THREADS) k_axpby(int64_t n, double alpha, const double* __restrict__ x, double beta,
                                                      double* __restrict__ y) {
  for (int64_t i = (int64_t)blockIdx.x * SV_THREADS + threadIdx.x; i < n; i += (int64_t)gridDim.x * SV_THREADS)
    y[i] = __dadd_rn(__dmul_rn(alpha, x[i]), __dmul_rn(beta, y[i]));
}

extern "C" int fem_vec_axpby(int64_t n, double alpha, const double* x, double beta, double* y, void* stream) {
  if (n < 0 || (n > 0 && (!x || !y))) {
    set_error("fem_vec_axpby: invalid argument");
    return FEM_E_INVALID_ARG;
  }
  if (n == 0) return 0;
  k_axpby<<<grid_for(n, 1), SV_THREADS, 0, (cudaStream_t)stream>>>(n, alpha, x, beta, y);
  FEM_CUDA_TRY(cudaGetLastError());
  return 0;
}

extern "C" int64_t fem_cg_work_doubles(int64_t n_rows) {
  return 5 * n_rows + 2 * SV_MAX_BLOCKS + (int64_t)(sizeof(CgScal) + 7) / 8 + 8;
}

extern "C" int fem_cg_solve(int64_t n_rows, const int64_t* rowptr, const int32_t* colidx, const double* values,
                            const double* b, double* x, double spd_sign, int max_iter, double rtol, int check_every,
                            double* work, int* iters_out, double* relres_out, void* stream) {
  if (n_rows <= 0 || !rowptr || !colidx || !values || !b || !x || !work || max_iter < 0 || !(rtol >= 0.0) ||
      (spd_sign != 1.0 && spd_sign != -1.0)) {
    set_error("fem_cg_solve: invalid argument (n_rows > 0, non-NULL pointers, spd_sign = ±1, rtol >= 0)");
    return FEM_E_INVALID_ARG;
  }
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t n = n_rows;
  double* r = work;
  double* z = r + n;
  double* p = z + n;
  double* q = p + n;
  double* dinv = q + n;
  double* partials = dinv + n;
  CgScal* sc = reinterpret_cast<CgScal*>(partials + 2 * SV_MAX_BLOCKS);
  int* bad = reinterpret_cast<int*>(reinterpret_cast<char*>(sc) + sizeof(CgScal));
  FEM_CUDA_TRY(cudaMemsetAsync(sc, 0, sizeof(CgScal) + 8, s));
  int g = 0;
  if (int rc = solver_lanes(rowptr, n, s, &g)) return rc;
  const int gv = grid_for(n, 1), gm = grid_for(n, g ? g : 1);
  k_cg_init<<<gv, SV_THREADS, 0, s>>>(n, rowptr, colidx, values, spd_sign, b, x, r, z, dinv, partials, sc, bad);
  k_cg_dir<<<gv, SV_THREADS, 0, s>>>(n, z, p, sc, 1);
  FEM_CUDA_TRY(cudaGetLastError());
  CgScal h{};
  int hbad = 0;
  FEM_CUDA_TRY(cudaMemcpyAsync(&h, sc, sizeof(CgScal), cudaMemcpyDeviceToHost, s));
  FEM_CUDA_TRY(cudaMemcpyAsync(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost, s));
  FEM_CUDA_TRY(cudaStreamSynchronize(s));
  if (hbad) {
    set_error("fem_cg_solve: a diagonal entry of spd_sign*K is not positive (matrix not SPD with this sign)");
    return FEM_E_INVALID_ARG;
  }
  const double rr0 = h.rr0;
  int it = 0;
  double rel = rr0 > 0.0 ? 1.0 : 0.0;
  const int chk = check_every > 0 ? check_every : 16;
  while (rr0 > 0.0 && it < max_iter && rel > rtol) {
    const int todo = std::min(chk, max_iter - it);
    for (int k = 0; k < todo; k++) {
      if (g == 0) k_cg_spmv<0><<<gm, SV_THREADS, 0, s>>>(n, rowptr, colidx, values, spd_sign, p, q, partials, sc);
      else k_cg_spmv<8><<<gm, SV_THREADS, 0, s>>>(n, rowptr, colidx, values, spd_sign, p, q, partials, sc);
      k_cg_update<<<gv, SV_THREADS, 0, s>>>(n, x, r, p, q, dinv, z, partials, sc);
      k_cg_dir<<<gv, SV_THREADS, 0, s>>>(n, z, p, sc, 0);
    }
    FEM_CUDA_TRY(cudaGetLastError());
    it += todo;
    FEM_CUDA_TRY(cudaMemcpyAsync(&h, sc, sizeof(CgScal), cudaMemcpyDeviceToHost, s));
    FEM_CUDA_TRY(cudaStreamSynchronize(s));
    rel = sqrt(h.rr / rr0);
    if (!(rel == rel)) {
      set_error("fem_cg_solve: breakdown (NaN in the recurrence)");
      if (iters_out) *iters_out = it;
      if (relres_out) *relres_out = rel;
      return FEM_E_NAN;
    }
  }
  if (iters_out) *iters_out = it;
  if (relres_out) *relres_out = rel;
  return 0;
}

extern "C" int64_t fem_bicgstab_work_doubles(int64_t n_rows) {
  return 9 * n_rows + 2 * SV_MAX_BLOCKS + (int64_t)(sizeof(BiScal) + 7) / 8 + 8;
}

extern "C" int fem_bicgstab_solve(int64_t n_rows, const int64_t* rowptr, const int32_t* colidx, const double* values,
                                  const double* b, double* x, int max_iter, double rtol, int check_every, double* work,
                                  int* iters_out, double* relres_out, void* stream) {
  if (n_rows <= 0 || !rowptr || !colidx || !values || !b || !x || !work || max_iter < 0 || !(rtol >= 0.0)) {
    set_error("fem_bicgstab_solve: invalid argument (n_rows > 0, non-NULL pointers, rtol >= 0)");
    return FEM_E_INVALID_ARG;
  }
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t n = n_rows;
  double* r = work;
  double* rh = r + n;
  double* p = rh + n;
  double* v = p + n;
  double* y = v + n;
  double* sv = y + n;
  double* z = sv + n;
  double* t = z + n;
  double* dinv = t + n;
  double* partials = dinv + n;
  BiScal* sc = reinterpret_cast<BiScal*>(partials + 2 * SV_MAX_BLOCKS);
  int* bad = reinterpret_cast<int*>(reinterpret_cast<char*>(sc) + sizeof(BiScal));
  FEM_CUDA_TRY(cudaMemsetAsync(sc, 0, sizeof(BiScal) + 8, st));
  int g = 0;
  if (int rc = solver_lanes(rowptr, n, st, &g)) return rc;
  const int gv = grid_for(n, 1), gm = grid_for(n, g ? g : 1);
  k_bi_init<<<gv, SV_THREADS, 0, st>>>(n, rowptr, colidx, values, b, x, r, rh, dinv, partials, sc, bad);
  FEM_CUDA_TRY(cudaGetLastError());
  BiScal h{};
  int hbad = 0;
  FEM_CUDA_TRY(cudaMemcpyAsync(&h, sc, sizeof(BiScal), cudaMemcpyDeviceToHost, st));
  FEM_CUDA_TRY(cudaMemcpyAsync(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost, st));
  FEM_CUDA_TRY(cudaStreamSynchronize(st));
  if (hbad) {
    set_error("fem_bicgstab_solve: zero diagonal entry (Jacobi preconditioner undefined)");
    return FEM_E_INVALID_ARG;
  }
  const double rr0 = h.rr0;
  int it = 0;
  double rel = rr0 > 0.0 ? 1.0 : 0.0;
  const int chk = check_every > 0 ? check_every : 16;
  while (rr0 > 0.0 && it < max_iter && rel > rtol) {
    const int todo = std::min(chk, max_iter - it);
    for (int k = 0; k < todo; k++) {
      k_bi_dir<<<gv, SV_THREADS, 0, st>>>(n, r, p, v, dinv, y, sc, it + k == 0);
#define BI_SPMV(MODE, IN, OUT, A)                                                                                 \
  if (g == 0) k_bi_spmv<0, MODE><<<gm, SV_THREADS, 0, st>>>(n, rowptr, colidx, values, IN, OUT, A, partials, sc); \
  else k_bi_spmv<8, MODE><<<gm, SV_THREADS, 0, st>>>(n, rowptr, colidx, values, IN, OUT, A, partials, sc);
      BI_SPMV(0, y, v, rh)
      k_bi_half<<<gv, SV_THREADS, 0, st>>>(n, x, y, r, v, dinv, sv, z, sc);
      BI_SPMV(1, z, t, sv)
#undef BI_SPMV
      k_bi_fin<<<gv, SV_THREADS, 0, st>>>(n, x, z, sv, t, rh, r, partials, sc);
    }
    FEM_CUDA_TRY(cudaGetLastError());
    it += todo;
    FEM_CUDA_TRY(cudaMemcpyAsync(&h, sc, sizeof(BiScal), cudaMemcpyDeviceToHost, st));
    FEM_CUDA_TRY(cudaStreamSynchronize(st));
    rel = sqrt(h.rr / rr0);
    if (!(rel == rel)) {
      set_error("fem_bicgstab_solve: breakdown (NaN in the recurrence)");
      if (iters_out) *iters_out = it;
      if (relres_out) *relres_out = rel;
      return FEM_E_NAN;
    }
  }
  if (iters_out) *iters_out = it;
  if (relres_out) *relres_out = rel;
  return 0;
}
