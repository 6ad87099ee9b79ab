// gmres.cu — NEXT-1 remainder: the linear solve of the Newton sub-step (D-4) for the stabilised
// Navier-Stokes system, whose SUPG/PSPG saddle point defeats Jacobi-BiCGStab.
//
// Restarted GMRES(m) with right preconditioning by POINT-BLOCK Jacobi: in the paper's κ-major numbering
// (B-3) the unknowns of control point α are rows κ·N + α, κ = 0..κ̂-1 (u_1..u_3, p for NS); their
// κ̂ x κ̂ diagonal block couples the velocity and the pressure of one point (the PSPG pp entry keeps it
// regular), and its inverse is the preconditioner block.  Arnoldi by classical Gram-Schmidt with one
// re-orthogonalisation (CGS2): the j+1 inner products of a step are one fixed-order multi-reduction, the
// update one pass.  Every reduction sums per block and then over the blocks in block order, so a solve is
// bit-identical run to run.  The (m+1) x m Hessenberg least-squares problem (Givens rotations) is solved
// on the host; one host sync per Arnoldi step reads its column.
//
// Gauge (reading L29): the paper's NS forms put NS_boundary_BASE on every boundary group, so for
// a constant pressure the domain term -(u_i,i, p) and the boundary term (u_i, p n_i) cancel in every momentum
// row (divergence theorem, exact under the rules) and no row depends on the pressure level: K has the
// constant-pressure null vector and d a component outside K's range.  pin_row >= 0 solves the system with
// that row and column replaced by the identity and the pinned increment 0 (the pressure of one point fixed).
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <vector>

#include "fem_internal.cuh"

namespace fem {

constexpr int GM_THREADS = 256;
constexpr int GM_BLOCKS = 148 * 4;  // fixed grid: the reduction order does not depend on the launch
constexpr int GM_MAX_RESTART = 1024;
constexpr int GM_MAX_KH = 4;

// Block inverse per control point: gather the kh x kh diagonal block of point a from the CSR rows
// κ·N + a (column κλ·N + a), invert by Gauss-Jordan with partial pivoting.  bad = 1 on a singular block.
__global__ void k_pbj_build(int64_t N, int kh, const int64_t* __restrict__ rowptr, const int32_t* __restrict__ colidx,
                            const double* __restrict__ val, double* __restrict__ binv, int* bad, int64_t pin) {
  for (int64_t a = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; a < N; a += (int64_t)gridDim.x * blockDim.x) {
    double A[GM_MAX_KH][2 * GM_MAX_KH];
    for (int i = 0; i < kh; i++) {
      for (int j = 0; j < 2 * kh; j++) A[i][j] = (j - kh == i) ? 1.0 : 0.0;
      const int64_t r = (int64_t)i * N + a, b = rowptr[r], e = rowptr[r + 1];
      for (int j = 0; j < kh; j++) {
        const int32_t col = (int32_t)((int64_t)j * N + a);
        int64_t lo = b, hi = e - 1;  // columns ascending within the row (reading L4)
        while (lo <= hi) {
          const int64_t mid = (lo + hi) >> 1;
          if (colidx[mid] < col) lo = mid + 1; else hi = mid - 1;
        }
        A[i][j] = (lo < e && colidx[lo] == col) ? val[lo] : 0.0;
      }
    }
    if (pin >= 0 && pin % N == a) {  // the pinned unknown: identity row and column
      const int kp = (int)(pin / N);
      for (int j = 0; j < kh; j++) { A[kp][j] = 0.0; A[j][kp] = 0.0; }
      A[kp][kp] = 1.0;
    }
    bool sing = false;
    for (int c = 0; c < kh; c++) {
      int piv = c;
      for (int i = c + 1; i < kh; i++)
        if (fabs(A[i][c]) > fabs(A[piv][c])) piv = i;
      if (!(fabs(A[piv][c]) > 0.0)) { sing = true; break; }
      if (piv != c)
        for (int j = 0; j < 2 * kh; j++) { const double t = A[c][j]; A[c][j] = A[piv][j]; A[piv][j] = t; }
      const double inv = 1.0 / A[c][c];
      for (int j = 0; j < 2 * kh; j++) A[c][j] *= inv;
      for (int i = 0; i < kh; i++)
        if (i != c) {
          const double f = A[i][c];
          for (int j = 0; j < 2 * kh; j++) A[i][j] = fma(-f, A[c][j], A[i][j]);
        }
    }
    if (sing) atomicExch(bad, 1);
    for (int i = 0; i < kh; i++)
      for (int j = 0; j < kh; j++) binv[(a * kh + i) * kh + j] = sing ? 0.0 : A[i][kh + j];
  }
}

// z = M^{-1} v: per point, z_(κ,a) = Σ_λ Binv[a][κ][λ] v_(λ,a)
__global__ void k_pbj_apply(int64_t N, int kh, const double* __restrict__ binv, const double* __restrict__ v,
                            double* __restrict__ z) {
  for (int64_t a = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; a < N; a += (int64_t)gridDim.x * blockDim.x) {
    double vv[GM_MAX_KH];
    for (int l = 0; l < kh; l++) vv[l] = v[(int64_t)l * N + a];
    for (int k = 0; k < kh; k++) {
      double s = 0.0;
      for (int l = 0; l < kh; l++) s = fma(binv[(a * kh + k) * kh + l], vv[l], s);
      z[(int64_t)k * N + a] = s;
    }
  }
}

// y = A x (rows of the CSR, a warp per row block as fem_spmv; here a plain warp-per-row kernel keeps the
// per-row sum order fixed: lanes stride the row, xor tree)
// pin >= 0: the operator with row and column `pin` replaced by the identity (the gauge of a singular K)
__global__ void k_gm_spmv(int64_t n, const int64_t* __restrict__ rowptr, const int32_t* __restrict__ colidx,
                          const double* __restrict__ val, const double* __restrict__ x, double* __restrict__ y,
                          const double* __restrict__ b, double alpha, int64_t pin) {
  const int lane = threadIdx.x & 31;
  for (int64_t r = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; r < n;
       r += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    double s = 0.0;
    if (r == pin) {
      s = x[pin];
    } else {
      for (int64_t k = rowptr[r] + lane; k < rowptr[r + 1]; k += 32) {
        const int32_t c = __ldcs(colidx + k);
        if (c != pin) s = fma(__ldcs(val + k), __ldg(x + c), s);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    }
    if (lane == 0) y[r] = b ? (r == pin ? 0.0 : b[r]) + alpha * s : alpha * s;
  }
}

// partial[i][block] = Σ_{rows of the block's grid stride} V_i[r] w[r], i < nv (V_i = V + i n); fixed order
__global__ void __launch_bounds__(GM_THREADS) k_gm_dots(int64_t n, int nv, const double* __restrict__ V,
                                                        const double* __restrict__ w, double* __restrict__ partial) {
  __shared__ double red[GM_THREADS / 32];
  for (int i = 0; i < nv; i++) {
    const double* vi = V + (int64_t)i * n;
    double s = 0.0;
    for (int64_t r = blockIdx.x * (int64_t)GM_THREADS + threadIdx.x; r < n; r += (int64_t)gridDim.x * GM_THREADS)
      s = fma(vi[r], w[r], s);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = 0.0;
      for (int k = 0; k < GM_THREADS / 32; k++) t += red[k];
      partial[(int64_t)i * gridDim.x + blockIdx.x] = t;
    }
    __syncthreads();
  }
}
// out[i] = Σ_block partial[i][block] in block order (one warp per i)
__global__ void k_gm_dots_final(int nv, int nblocks, const double* __restrict__ partial, double* __restrict__ out) {
  const int i = blockIdx.x;
  if (i >= nv || threadIdx.x != 0) return;
  double t = 0.0;
  for (int k = 0; k < nblocks; k++) t += partial[(int64_t)i * nblocks + k];
  out[i] = t;
}
// w -= Σ_i h_i V_i
__global__ void k_gm_update(int64_t n, int nv, const double* __restrict__ V, const double* __restrict__ h,
                            double* __restrict__ w) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x) {
    double s = w[r];
    for (int i = 0; i < nv; i++) s = fma(-h[i], V[(int64_t)i * n + r], s);
    w[r] = s;
  }
}
// y = alpha x (+ y if acc)
__global__ void k_gm_scale(int64_t n, double alpha, const double* __restrict__ x, double* __restrict__ y, int acc) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x)
    y[r] = acc ? fma(alpha, x[r], y[r]) : alpha * x[r];
}

}  // namespace fem

using namespace fem;

extern "C" int64_t fem_gmres_work_doubles(int64_t n_rows, int64_t n_points, int kappa_hat, int restart) {
  const int m = std::min(std::max(restart, 1), GM_MAX_RESTART);
  return (int64_t)(m + 1) * n_rows + 2 * n_rows + n_points * kappa_hat * kappa_hat +
         (int64_t)(m + 2) * GM_BLOCKS + 2 * (m + 2) + 8;
}

extern "C" int fem_gmres_solve(int64_t n_rows, const int64_t* rowptr, const int32_t* colidx, const double* values,
                               int64_t n_points, int kappa_hat, const double* b, double* x, int restart, int max_iter,
                               double rtol, int64_t pin_row, double* work, int* iters_out, double* relres_out,
                               void* stream) {
  const int m = std::min(std::max(restart, 1), GM_MAX_RESTART);
  if (n_rows <= 0 || !rowptr || !colidx || !values || !b || !x || !work || max_iter < 0 || !(rtol >= 0.0) ||
      kappa_hat < 1 || kappa_hat > GM_MAX_KH || n_points * kappa_hat != n_rows || pin_row >= n_rows) {
    set_error("fem_gmres_solve: invalid argument (n_rows = n_points * kappa_hat, kappa_hat 1..4, non-NULL pointers)");
    return FEM_E_INVALID_ARG;
  }
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t n = n_rows, N = n_points;
  double* V = work;                                // (m+1) Krylov vectors
  double* w = V + (int64_t)(m + 1) * n;            // work vector
  double* z = w + n;                               // preconditioned vector
  double* binv = z + n;                            // point blocks
  double* partial = binv + N * kappa_hat * kappa_hat;
  double* hd = partial + (int64_t)(m + 2) * GM_BLOCKS;  // device copy of dot results / coefficients
  int* bad = reinterpret_cast<int*>(hd + 2 * (m + 2));
  const int gv = (int)std::min<int64_t>((n + GM_THREADS - 1) / GM_THREADS, GM_BLOCKS);
  const int gp = (int)std::min<int64_t>((N + GM_THREADS - 1) / GM_THREADS, GM_BLOCKS);
  const int gs = (int)std::min<int64_t>((n * 32 + GM_THREADS - 1) / GM_THREADS, 148 * 16);
  FEM_CUDA_TRY(cudaMemsetAsync(bad, 0, sizeof(int), s));
  const int64_t pin = pin_row < 0 ? -1 : pin_row;
  k_pbj_build<<<gp, GM_THREADS, 0, s>>>(N, kappa_hat, rowptr, colidx, values, binv, bad, pin);
  int hbad = 0;
  FEM_CUDA_TRY(cudaMemcpyAsync(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost, s));
  FEM_CUDA_TRY(cudaStreamSynchronize(s));
  if (hbad) {
    set_error("fem_gmres_solve: a point block of the diagonal is singular (point-block Jacobi undefined)");
    return FEM_E_INVALID_ARG;
  }
  // host helpers around the fixed-order device reductions
  auto dots = [&](int nv, const double* Vb, const double* vec, double* out) -> int {
    k_gm_dots<<<GM_BLOCKS, GM_THREADS, 0, s>>>(n, nv, Vb, vec, partial);
    k_gm_dots_final<<<nv, 32, 0, s>>>(nv, GM_BLOCKS, partial, hd);
    FEM_CUDA_TRY(cudaGetLastError());
    FEM_CUDA_TRY(cudaMemcpyAsync(out, hd, sizeof(double) * nv, cudaMemcpyDeviceToHost, s));
    FEM_CUDA_TRY(cudaStreamSynchronize(s));
    return 0;
  };
  // the pinned right-hand side (b with b_pin = 0: the pinned unknown keeps its initial value; x_pin should be 0)
  k_gm_scale<<<gv, GM_THREADS, 0, s>>>(n, 1.0, b, z, 0);
  if (pin >= 0) FEM_CUDA_TRY(cudaMemsetAsync(z + pin, 0, sizeof(double), s));
  double bb = 0.0;
  if (int rc = dots(1, z, z, &bb)) return rc;
  const double bnorm = std::sqrt(bb);
  int it = 0;
  double rel = bnorm > 0.0 ? 1.0 : 0.0;
  std::vector<double> H((m + 1) * m), cs(m), sn(m), g(m + 1), y(m), hcol(m + 2);
  while (bnorm > 0.0 && it < max_iter) {
    // r0 = b - A x  -> V_0
    k_gm_spmv<<<gs, GM_THREADS, 0, s>>>(n, rowptr, colidx, values, x, V, b, -1.0, pin);
    double rr = 0.0;
    if (int rc = dots(1, V, V, &rr)) return rc;
    const double beta = std::sqrt(rr);
    rel = beta / bnorm;
    if (!(rel == rel)) { set_error("fem_gmres_solve: NaN residual"); return FEM_E_NAN; }
    if (rel <= rtol) break;
    k_gm_scale<<<gv, GM_THREADS, 0, s>>>(n, 1.0 / beta, V, V, 0);
    std::fill(g.begin(), g.end(), 0.0);
    g[0] = beta;
    int j = 0;
    for (; j < m && it < max_iter; j++, it++) {
      double* vj = V + (int64_t)j * n;
      k_pbj_apply<<<gp, GM_THREADS, 0, s>>>(N, kappa_hat, binv, vj, z);
      k_gm_spmv<<<gs, GM_THREADS, 0, s>>>(n, rowptr, colidx, values, z, w, nullptr, 1.0, pin);
      // CGS2: two passes of h = V^T w, w -= V h
      for (int i = 0; i <= j; i++) H[i * m + j] = 0.0;
      for (int pass = 0; pass < 2; pass++) {
        if (int rc = dots(j + 1, V, w, hcol.data())) return rc;
        FEM_CUDA_TRY(cudaMemcpyAsync(hd, hcol.data(), sizeof(double) * (j + 1), cudaMemcpyHostToDevice, s));
        k_gm_update<<<gv, GM_THREADS, 0, s>>>(n, j + 1, V, hd, w);
        for (int i = 0; i <= j; i++) H[i * m + j] += hcol[i];
      }
      double ww = 0.0;
      if (int rc = dots(1, w, w, &ww)) return rc;
      const double hn = std::sqrt(ww);
      H[(j + 1) * m + j] = hn;
      if (hn > 0.0) k_gm_scale<<<gv, GM_THREADS, 0, s>>>(n, 1.0 / hn, w, V + (int64_t)(j + 1) * n, 0);
      // Givens rotations on column j
      for (int i = 0; i < j; i++) {
        const double a = H[i * m + j], c2 = H[(i + 1) * m + j];
        H[i * m + j] = cs[i] * a + sn[i] * c2;
        H[(i + 1) * m + j] = -sn[i] * a + cs[i] * c2;
      }
      const double a = H[j * m + j], c2 = H[(j + 1) * m + j], rho = std::hypot(a, c2);
      cs[j] = rho > 0.0 ? a / rho : 1.0;
      sn[j] = rho > 0.0 ? c2 / rho : 0.0;
      H[j * m + j] = rho;
      H[(j + 1) * m + j] = 0.0;
      g[j + 1] = -sn[j] * g[j];
      g[j] = cs[j] * g[j];
      rel = std::fabs(g[j + 1]) / bnorm;
      if (!(rel == rel)) { set_error("fem_gmres_solve: breakdown (NaN)"); return FEM_E_NAN; }
      if (rel <= rtol || hn == 0.0) { j++; it++; break; }
    }
    // y = H^{-1} g (upper triangular j x j), x += M^{-1} (V y)
    for (int i = j - 1; i >= 0; i--) {
      double t = g[i];
      for (int k = i + 1; k < j; k++) t -= H[i * m + k] * y[k];
      y[i] = H[i * m + i] != 0.0 ? t / H[i * m + i] : 0.0;
    }
    FEM_CUDA_TRY(cudaMemsetAsync(w, 0, sizeof(double) * n, s));
    for (int i = 0; i < j; i++) {
      FEM_CUDA_TRY(cudaMemcpyAsync(hd, &y[i], sizeof(double), cudaMemcpyHostToDevice, s));
      FEM_CUDA_TRY(cudaStreamSynchronize(s));
      k_gm_scale<<<gv, GM_THREADS, 0, s>>>(n, y[i], V + (int64_t)i * n, w, 1);
    }
    k_pbj_apply<<<gp, GM_THREADS, 0, s>>>(N, kappa_hat, binv, w, z);
    k_gm_scale<<<gv, GM_THREADS, 0, s>>>(n, 1.0, z, x, 1);
    FEM_CUDA_TRY(cudaGetLastError());
    if (rel <= rtol) {  // true residual of the final iterate
      k_gm_spmv<<<gs, GM_THREADS, 0, s>>>(n, rowptr, colidx, values, x, w, b, -1.0, pin);
      double tr = 0.0;
      if (int rc = dots(1, w, w, &tr)) return rc;
      rel = std::sqrt(tr) / bnorm;
      if (rel <= rtol * 10.0) break;  // (the recurrence's estimate drifts a little from the true residual)
    }
  }
  if (iters_out) *iters_out = it;
  if (relres_out) *relres_out = rel;
  return 0;
}
