// timestep.cu — NEXT-3: the generalized-α vector updates around the assembly.
//
// PAPER.md Block C (C-1..C-3) refreshes the increments at the start of a timestep and Block D
// updates the effective values (D-1) and the increments after each sub-step's solve (D-4,
// P:459-465).  All three are elementwise over the (ν̂+1) × n arrays [ν][n] (n = κ̂N rows of the system,
// κ-major numbering of fem_pattern_build), so each is one HBM pass: a persistent grid (a multiple of the
// 148 SMs) strides over n, every thread handling all ν̂+1 levels of its entries so no level is re-read.
// C and D-4 optionally write the next D-1 effective values in the same pass (one read of φ⁰/Δφ saved).
//
// Readings: L13 — D-4 divides by Π_{β'≤ν}(b_β' Δt) (Eq. gen_alpha, Eq.
// time_constraints P:227-228; P:463 prints a product); L14 — C-3 seeds Δ∂^ν φ = Δt(∂^{ν+1}φ +
// b_{ν+1}Δ∂^{ν+1}φ) from Eq. time_constraints (P:416 as printed contradicts it).
// Arithmetic is explicitly rounded (__dmul_rn/__dadd_rn/__ddiv_rn, no FMA contraction) so each value is
// the correctly rounded result of the paper's expression evaluated left to right.
#include <algorithm>
#include <cstdint>

#include "fem_internal.cuh"

namespace fem {

constexpr int TS_THREADS = 256;
constexpr int TS_MAX_BLOCKS = 148 * 8;

struct TsCoef {
  double dt, b[2], c[3];
  int nu_hat;
};

__device__ __forceinline__ double prod_b_dt(const TsCoef& k, int nu) {  // Π_{β'=1}^{ν}(b_β' Δt), empty = 1
  double p = 1.0;
  for (int j = 0; j < nu; j++) p = __dmul_rn(p, __dmul_rn(k.b[j], k.dt));
  return p;
}

// Block C (+ optional D-1): C-1 φ⁰ += Δφ; C-2 Δ∂^ν̂ φ = 0; C-3 ν = ν̂-1..0 (reading L14)
template <int NU>
__global__ void __launch_bounds__(TS_THREADS) k_time_init(TsCoef k, int64_t n, double* __restrict__ phi0,
                                                          double* __restrict__ incr, double* __restrict__ eff) {
  for (int64_t i = blockIdx.x * (int64_t)TS_THREADS + threadIdx.x; i < n; i += (int64_t)gridDim.x * TS_THREADS) {
    double p[NU + 1], d[NU + 1];
#pragma unroll
    for (int v = 0; v <= NU; v++) p[v] = __dadd_rn(phi0[v * n + i], incr[v * n + i]);  // C-1
    d[NU] = 0.0;                                                                         // C-2
#pragma unroll
    for (int v = NU - 1; v >= 0; v--) d[v] = __dmul_rn(k.dt, __dadd_rn(p[v + 1], __dmul_rn(k.b[v], d[v + 1])));
#pragma unroll
    for (int v = 0; v <= NU; v++) {
      phi0[v * n + i] = p[v];
      incr[v * n + i] = d[v];
      if (eff) eff[v * n + i] = __dadd_rn(__dmul_rn(k.c[v], d[v]), p[v]);  // D-1
    }
  }
}

// D-1: ∂^ν φ̃ = c_{ν+1} Δ∂^ν φ + ∂^ν φ
template <int NU>
__global__ void __launch_bounds__(TS_THREADS) k_time_effective(TsCoef k, int64_t n, const double* __restrict__ phi0,
                                                               const double* __restrict__ incr, double* __restrict__ eff) {
  for (int64_t i = blockIdx.x * (int64_t)TS_THREADS + threadIdx.x; i < n; i += (int64_t)gridDim.x * TS_THREADS) {
#pragma unroll
    for (int v = 0; v <= NU; v++) eff[v * n + i] = __dadd_rn(__dmul_rn(k.c[v], incr[v * n + i]), phi0[v * n + i]);
  }
}

// D-4 (reading L13): Δ∂^ν φ += Δ_sub φ / Π_{β'≤ν}(b_β' Δt)  (+ optional D-1 of the next sub-step)
template <int NU>
__global__ void __launch_bounds__(TS_THREADS) k_time_increment(TsCoef k, int64_t n, const double* __restrict__ dsub,
                                                               double* __restrict__ incr, const double* __restrict__ phi0,
                                                               double* __restrict__ eff) {
  double P[NU + 1];
#pragma unroll
  for (int v = 0; v <= NU; v++) P[v] = prod_b_dt(k, v);
  for (int64_t i = blockIdx.x * (int64_t)TS_THREADS + threadIdx.x; i < n; i += (int64_t)gridDim.x * TS_THREADS) {
    const double s = dsub[i];
#pragma unroll
    for (int v = 0; v <= NU; v++) {
      const double d = __dadd_rn(incr[v * n + i], __ddiv_rn(s, P[v]));
      incr[v * n + i] = d;
      if (eff) eff[v * n + i] = __dadd_rn(__dmul_rn(k.c[v], d), phi0[v * n + i]);
    }
  }
}

static int ts_coef(const fem_time_scheme* ts, int64_t n, const char* who, TsCoef* k) {
  if (!ts || n < 0 || ts->kind != FEM_TIME_GENALPHA || ts->nu_hat < 0 || ts->nu_hat > 2 || !(ts->dt > 0.0) ||
      (ts->nu_hat >= 1 && ts->b1 == 0.0) || (ts->nu_hat >= 2 && ts->b2 == 0.0)) {
    set_error(std::string(who) + ": invalid argument (kind = FEM_TIME_GENALPHA, 0 <= nu_hat <= 2, dt > 0, "
              "b_nu != 0 for nu <= nu_hat, n >= 0)");
    return FEM_E_INVALID_ARG;
  }
  *k = TsCoef{ts->dt, {ts->b1, ts->b2}, {ts->c1, ts->c2, ts->c3}, ts->nu_hat};
  return 0;
}

static unsigned ts_grid(int64_t n) {
  return (unsigned)std::max<int64_t>(1, std::min<int64_t>((n + TS_THREADS - 1) / TS_THREADS, TS_MAX_BLOCKS));
}

}  // namespace fem

using namespace fem;

#define TS_DISPATCH(KERNEL, ...)                                                               \
  switch (k.nu_hat) {                                                                          \
    case 0: KERNEL<0><<<ts_grid(n), TS_THREADS, 0, (cudaStream_t)stream>>>(__VA_ARGS__); break; \
    case 1: KERNEL<1><<<ts_grid(n), TS_THREADS, 0, (cudaStream_t)stream>>>(__VA_ARGS__); break; \
    default: KERNEL<2><<<ts_grid(n), TS_THREADS, 0, (cudaStream_t)stream>>>(__VA_ARGS__); break; \
  }

extern "C" int fem_time_init(const fem_time_scheme* ts, int64_t n, double* phi0, double* incr, double* eff,
                             void* stream) {
  TsCoef k;
  if (int rc = ts_coef(ts, n, "fem_time_init", &k)) return rc;
  if (n == 0) return 0;
  if (!phi0 || !incr) {
    set_error("fem_time_init: NULL array");
    return FEM_E_INVALID_ARG;
  }
  TS_DISPATCH(k_time_init, k, n, phi0, incr, eff);
  FEM_CUDA_TRY(cudaGetLastError());
  return 0;
}

extern "C" int fem_time_effective(const fem_time_scheme* ts, int64_t n, const double* phi0, const double* incr,
                                  double* eff, void* stream) {
  TsCoef k;
  if (int rc = ts_coef(ts, n, "fem_time_effective", &k)) return rc;
  if (n == 0) return 0;
  if (!phi0 || !incr || !eff) {
    set_error("fem_time_effective: NULL array");
    return FEM_E_INVALID_ARG;
  }
  TS_DISPATCH(k_time_effective, k, n, phi0, incr, eff);
  FEM_CUDA_TRY(cudaGetLastError());
  return 0;
}

extern "C" int fem_time_increment(const fem_time_scheme* ts, int64_t n, const double* delta_sub, double* incr,
                                  const double* phi0, double* eff, void* stream) {
  TsCoef k;
  if (int rc = ts_coef(ts, n, "fem_time_increment", &k)) return rc;
  if (n == 0) return 0;
  if (!delta_sub || !incr || (eff && !phi0)) {
    set_error("fem_time_increment: NULL array (phi0 is required when eff is given)");
    return FEM_E_INVALID_ARG;
  }
  TS_DISPATCH(k_time_increment, k, n, delta_sub, incr, phi0, eff);
  FEM_CUDA_TRY(cudaGetLastError());
  return 0;
}
