// Top-k eigenvectors of the mode-1 Gram -> the sketch S (Algorithm 2 line 2).
//
// S* = (U^(1))_k^T: the first k left singular vectors of A_(1), i.e. the top-k eigenvectors
// of G = A_(1) A_(1)^T (symmetric PSD, m x m).  The paper gives no algorithm for this step
// (reading c4); we use:
//   * m <= dense_max_m : one dense one-sided Jacobi eigensolve of G (fp64),
//   * otherwise block subspace iteration with Rayleigh-Ritz (reading c15):
//       Z = G Q            3xTF32 tensor-core product (gemm_tc.cu), fp64 result
//       H = Q^T Z          fp64, symmetrised
//       H = W diag(theta) W^T   one-sided Jacobi (jacobi.cu)
//       X = Q W            Ritz vectors;  Y = Z W diag(1/theta)  (= G X / theta)
//       residual_c = theta_c ||Y_c - X_c|| = ||G x_c - theta_c x_c||
//       Q <- CholQR2(Y)    fp64 Cholesky QR, twice (Y is column-scaled: well conditioned)
//     with block size p = k + oversample, stopped when every top-k Ritz pair has backward
//     error ||G x_c - theta_c x_c|| <= tol * theta_1 (tol * ||G||_2), default 5e-7: about the
//     3xTF32 G Q floor (~2-4e-7), and tight enough that the Ky Fan deficit of S stays ~1e-7 on
//     the flat C3/C4 spectra (at 1e-6 it measured 1.5e-6).
// Output rows of S are the top-k Ritz vectors in decreasing theta order, each normalised
// and sign-fixed so its largest-|entry| is positive (reading c5).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "dense64.cuh"
#include "eig_kernels.cuh"
#include "ptx.cuh"
#include "tsk_internal.h"

namespace tsk {

__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

// deterministic start block: uniform(-1, 1) entries from a counter-based hash
__global__ void hash_fill_kernel(double* Y, int m, int p, uint64_t salt, double scale, int add) {
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (long long)m * p) return;
  const uint64_t h = splitmix64((uint64_t)idx * 0x2545F4914F6CDD1Dull + salt);
  const double u = ((double)(h >> 11) * (1.0 / 9007199254740992.0)) * 2.0 - 1.0;
  Y[idx] = add ? Y[idx] + scale * u : scale * u;
}

// G64 [m][m] -> G32 [m][ms] (zero pad to a 16-byte row pitch)
__global__ void g_to_f32_kernel(const double* __restrict__ G, int m, int ms, float* __restrict__ G32) {
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (long long)m * ms) return;
  const int i = (int)(idx / ms), j = (int)(idx % ms);
  G32[idx] = j < m ? (float)G[(size_t)i * m + j] : 0.f;
}

// Q [m][p] fp64 -> Qt32 [p][ms] fp32 (transposed, K-major for the tensor core), and Q <- fp64(fp32(Q))
__global__ void q_to_f32t_kernel(double* __restrict__ Q, int m, int p, int ms, float* __restrict__ Qt) {
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (long long)p * ms) return;
  const int c = (int)(idx / ms), i = (int)(idx % ms);
  if (i < m) {
    const float v = (float)Q[(size_t)i * p + c];
    Qt[idx] = v;
    Q[(size_t)i * p + c] = (double)v;
  } else {
    Qt[idx] = 0.f;
  }
}

__global__ void inv_theta_kernel(const double* __restrict__ theta, int p, double* __restrict__ inv) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= p) return;
  const double t = theta[c];
  const double t0 = theta[0];
  inv[c] = (fabs(t) > 1e-300 && fabs(t) > 1e-14 * fabs(t0)) ? 1.0 / t : (t0 != 0.0 ? 1.0 / t0 : 1.0);
}

// res[c] = theta_c * ||Y_c - X_c||  for c < k   (one block per column)
__global__ void ritz_residual_kernel(const double* __restrict__ Y, const double* __restrict__ X, const double* theta,
                                     int m, int p, double* __restrict__ res) {
  const int c = blockIdx.x;
  double s = 0.0;
  for (int i = threadIdx.x; i < m; i += blockDim.x) {
    const double d = Y[(size_t)i * p + c] - X[(size_t)i * p + c];
    s += d * d;
  }
  __shared__ double red[256];
  red[threadIdx.x] = s;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) res[c] = fabs(theta[c]) * sqrt(red[0]);
}

// S[c][i] = sgn_c * V[i][c] / ||V_c||  for c < k  (V: [m][ldv]); sign makes the largest-|entry| positive
__global__ void write_sketch_kernel(const double* __restrict__ V, int m, int ldv, float* __restrict__ S) {
  const int c = blockIdx.x;
  __shared__ double best_v[256];
  __shared__ int best_i[256];
  __shared__ double nrm[256];
  double bv = -1.0, ss = 0.0;
  int bi = 0x7fffffff;
  for (int i = threadIdx.x; i < m; i += blockDim.x) {
    const double v = V[(size_t)i * ldv + c];
    ss += v * v;
    const double a = fabs(v);
    if (a > bv || (a == bv && i < bi)) { bv = a; bi = i; }
  }
  best_v[threadIdx.x] = bv;
  best_i[threadIdx.x] = bi;
  nrm[threadIdx.x] = ss;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) {
      const double v2 = best_v[threadIdx.x + o];
      const int i2 = best_i[threadIdx.x + o];
      if (v2 > best_v[threadIdx.x] || (v2 == best_v[threadIdx.x] && i2 < best_i[threadIdx.x])) {
        best_v[threadIdx.x] = v2;
        best_i[threadIdx.x] = i2;
      }
      nrm[threadIdx.x] += nrm[threadIdx.x + o];
    }
    __syncthreads();
  }
  const double sgn = V[(size_t)best_i[0] * ldv + c] < 0 ? -1.0 : 1.0;
  const double inv = nrm[0] > 0 ? sgn / sqrt(nrm[0]) : 0.0;
  for (int i = threadIdx.x; i < m; i += blockDim.x) S[(size_t)c * m + i] = (float)(V[(size_t)i * ldv + c] * inv);
}

static inline unsigned nblk(long long n, int t) { return (unsigned)((n + t - 1) / t); }

// ||G||_F^2 in a fixed order: gridDim.x CTAs sum contiguous slices (thread-strided partial sums,
// tree reduction) into part[], then one CTA reduces part[] the same way (sum_kernel).  The
// one-CTA version took 170 us at m = 1080.
__global__ void fro2_part_kernel(const double* __restrict__ G, long long n, double* __restrict__ part) {
  __shared__ double red[256];
  const long long per = (n + gridDim.x - 1) / gridDim.x;
  const long long e0 = (long long)blockIdx.x * per, e1 = min(n, e0 + per);
  double sacc = 0.0;
  for (long long e = e0 + threadIdx.x; e < e1; e += blockDim.x) sacc += G[e] * G[e];
  red[threadIdx.x] = sacc;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if ((int)threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = red[0];
}
__global__ void sum_kernel(const double* __restrict__ x, long long n, double* __restrict__ out) {
  __shared__ double red[1024];
  double sacc = 0.0;
  for (long long e = threadIdx.x; e < n; e += blockDim.x) sacc += x[e];
  red[threadIdx.x] = sacc;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if ((int)threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = red[0];
}

// Y[i][c] = S0[c][i] for c < k (Y: [m][p] fp64, S0: [k][m] fp32)
__global__ void init_cols_kernel(double* __restrict__ Y, int m, int p, const float* __restrict__ S0, int k) {
  const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (long long)m * k) return;
  const int c = (int)(e / m), i = (int)(e % m);
  Y[(size_t)i * p + c] = (double)S0[(size_t)c * m + i];
}

// Y = Z diag(scale)   (m x p, row-major)
__global__ void colscale_kernel(const double* __restrict__ Z, const double* __restrict__ scale, int m, int p,
                                double* __restrict__ Y) {
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (long long)m * p) return;
  Y[idx] = Z[idx] * scale[idx % p];
}

// Q <- orthonormal basis of range(Y) by CholQR2 (fp64): C = Y^T Y = L L^T, Q1 = Y L^-T, twice.
// Y arrives column-scaled (each column ~ G x_c / theta_c), so C is well conditioned and one
// pass is already orthonormal to ~cond(Y)^2 eps; the second pass removes that residue.
// flags[0..1] (device) receive the first failed pivot + 1 of each pass (0 = success): a failure
// means rank(Y) < p, repaired by the caller.

// G64[i][j] -= sum_t theta_t x_t[i] x_t[j]  (deflation of locked Ritz pairs; X: [m][ldx] columns t0..t1)
__global__ void deflate_kernel(double* __restrict__ G, int m, const double* __restrict__ X, int ldx, int t0, int t1,
                               const double* __restrict__ theta) {
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (long long)m * m) return;
  const int i = (int)(idx / m), j = (int)(idx % m);
  double s = 0.0;
  for (int t = t0; t < t1; ++t) s += theta[t] * X[(size_t)i * ldx + t] * X[(size_t)j * ldx + t];
  G[idx] -= s;
}

// Chebyshev three-term step:  Ynew = alpha (Z - c Y) - beta Yprev   (m x p, row-major)
__global__ void cheb_step_kernel(const double* __restrict__ Z, const double* __restrict__ Yc,
                                 const double* __restrict__ Yp, long long n, double c, double alpha, double beta,
                                 double* __restrict__ Yn) {
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= n) return;
  const double v = alpha * (Z[idx] - c * Yc[idx]);
  Yn[idx] = beta != 0.0 ? v - beta * Yp[idx] : v;
}

// column norms of Y (m x p) -> inverse norms (0 for a zero column); one block per column
__global__ void inv_colnorm_kernel(const double* __restrict__ Y, int m, int p, double* __restrict__ inv) {
  const int c = blockIdx.x;
  double s = 0.0;
  for (int i = threadIdx.x; i < m; i += blockDim.x) {
    const double v = Y[(size_t)i * p + c];
    s += v * v;
  }
  __shared__ double red[256];
  red[threadIdx.x] = s;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) inv[c] = red[0] > 0.0 ? 1.0 / sqrt(red[0]) : 0.0;
}

// copy columns [c0, c0+nc) of src [m][lds] to columns [d0, d0+nc) of dst [m][ldd]
__global__ void copy_cols_kernel(const double* __restrict__ src, int lds, int c0, double* __restrict__ dst, int ldd,
                                 int d0, int m, int nc) {
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (long long)m * nc) return;
  const int i = (int)(idx / nc), c = (int)(idx % nc);
  dst[(size_t)i * ldd + d0 + c] = src[(size_t)i * lds + c0 + c];
}

// one CholQR pass Q = Y R^{-1}: C = Y^T Y (fp64), R^{-1} from one-CTA Cholesky + inverse, Q = Y R^{-1}
// (parallel fp64 GEMM); for large blocks (p > 116) the row-parallel TRSM path is used instead.
static tsk_status cholqr_pass(Ctx* ctx, const double* Y, double* Q, int m, int p, double* C, double* R, int* flag) {
  tsk_status st;
  if ((st = gemm_tn_f64(ctx, Y, p, 0, Y, p, 0, m, p, p, 1, C, p, 0, 1, WS_EIG_SMALL)) != TSK_OK) return st;
  if ((size_t)2 * p * (p | 1) * 8 <= 220 * 1024 && p <= 128) {
    if ((st = chol_inv2(ctx, C, p, 1, 1e-13, R, flag)) != TSK_OK) return st;
    return gemm_nn_f64(ctx, Y, p, 0, R, p, 0, m, p, p, 1, nullptr, Q, p, 0);
  }
  if ((st = chol(ctx, C, p, 1, 1e-13, R, flag, WS_JACOBI)) != TSK_OK) return st;
  return trsm_rlt(ctx, Y, R, m, p, Q);
}

static tsk_status cholqr1(Ctx* ctx, const double* Y, double* Q, int m, int p, double* C, double* R, int* flags) {
  return cholqr_pass(ctx, Y, Q, m, p, C, R, flags);
}

tsk_status cholqr2(Ctx* ctx, const double* Y, double* Q1, double* Q, int m, int p, double* C, double* R,
                          int* flags) {
  tsk_status st;
  if ((st = cholqr_pass(ctx, Y, Q1, m, p, C, R, flags)) != TSK_OK) return st;
  return cholqr_pass(ctx, Q1, Q, m, p, C, R, flags + 1);
}

tsk_status topk_eigen(Ctx* ctx, const double* G64, int m, int k, float* S, double* lambda,
                      const tsk_train_opts* o, tsk_train_info* info) {
  return topk_eigen_ex(ctx, G64, m, k, S, lambda, o, info, 0, nullptr);
}

// f64_products: G Q in fp64 (SIMT GEMM on the fp64 master copy) instead of 3xTF32 -- for small
// dense matrices (the matrix-free sketch's Rayleigh-Ritz matrix, m <= 256) where fp64 is cheap and
// the one-CTA Jacobi would have to leave shared memory (m > 116); tolerances scale accordingly.
// X64 (optional, device [m][k] fp64): the output eigenvectors as columns, before the fp32 rounding
// of S (same order; sign rule applied to S only).
tsk_status topk_eigen_ex(Ctx* ctx, const double* G64, int m, int k, float* S, double* lambda,
                         const tsk_train_opts* o, tsk_train_info* info, int f64_products, double* X64) {
  if (m < 1 || k < 1 || k > m) return TSK_EINVAL;
  tsk_train_opts opt{};
  if (o) opt = *o;
  const bool f64 = f64_products != 0;
  const int dense_max = opt.dense_max_m > 0 ? opt.dense_max_m : (f64 ? 116 : 256);
  const int max_iters = opt.max_iters > 0 ? opt.max_iters : 300;
  const double tol = opt.tol > 0 ? opt.tol : (f64 ? 1e-11 : 5e-7);

  // block size p = k + 16 by default: measured on C3/C4 spectra (flat near k), larger blocks cut
  // iterations less than they raise the cost of each p x p Rayleigh-Ritz solve
  int p = opt.oversample > 0 ? k + opt.oversample : k + 16;
  p = std::min(p, m);
  cudaStream_t s = ctx->stream;
  tsk_status st;

  if (m <= dense_max || p >= m || (!f64 && m <= 256)) {
    if (m > 256) return TSK_EINVAL;
    double* W = reinterpret_cast<double*>(ctx->workspace(WS_EIG_A, (size_t)m * m * 8));
    double* lam = reinterpret_cast<double*>(ctx->workspace(WS_EIG_SMALL, (size_t)m * 8 + 64));
    if (!W || !lam) return TSK_ENOMEM;
    if ((st = jacobi_eig_batched(ctx, G64, m, 1, W, lam)) != TSK_OK) return st;
    write_sketch_kernel<<<k, 256, 0, s>>>(W, m, m, S);
    ctx->count_launch();
    if (X64) {
      copy_cols_kernel<<<nblk((long long)m * k, 256), 256, 0, s>>>(W, m, 0, X64, k, 0, m, k);
      ctx->count_launch();
    }
    if (lambda) cudaMemcpyAsync(lambda, lam, (size_t)k * 8, cudaMemcpyDeviceToDevice, s);
    if (info) {
      info->iters = 0;
      std::vector<double> h(k);
      cudaMemcpyAsync(h.data(), lam, (size_t)k * 8, cudaMemcpyDeviceToHost, s);
      cudaStreamSynchronize(s);
      double kf = 0;
      for (double v : h) kf += v;
      info->kyfan = kf;
      info->max_resid = 0.0;
      double lk1 = 0.0;
      if (k < m) cudaMemcpy(&lk1, lam + k, 8, cudaMemcpyDeviceToHost);
      info->gap_est = lk1 > 0.0 ? h[k - 1] / lk1 : INFINITY;
    }
    return cudaPeekAtLastError() == cudaSuccess ? TSK_OK : TSK_ECUDA;
  }

  const int ms = (m + 3) & ~3;
  const size_t mp = (size_t)m * p;
  // workspace carve-up
  double* big = reinterpret_cast<double*>(ctx->workspace(WS_EIG_A, mp * 8 * 8));
  double* small = reinterpret_cast<double*>(ctx->workspace(WS_EIG_B, ((size_t)p * p * 4 + p * 12) * 8 + 256));
  float* G32 = reinterpret_cast<float*>(ctx->workspace(WS_EIG_G32, (size_t)m * ms * 4));
  float* Qt = reinterpret_cast<float*>(ctx->workspace(WS_EIG_Q32, (size_t)p * ms * 4));
  double* Gd = reinterpret_cast<double*>(ctx->workspace(WS_EIG_C, (size_t)m * m * 8));
  double* hostbuf = reinterpret_cast<double*>(ctx->pinned((size_t)(4 * p + 16) * 8));
  if (!big || !small || !G32 || !Qt || !Gd || !hostbuf) return TSK_ENOMEM;
  double *Q = big, *Z = big + mp, *X = big + 2 * mp, *Y = big + 3 * mp, *Q1 = big + 4 * mp;
  double *Y0 = big + 5 * mp, *Y1 = big + 6 * mp, *Xl = big + 7 * mp;  // Xl: locked Ritz vectors [m][p]
  double *H = small, *W = small + (size_t)p * p, *C = small + 2 * (size_t)p * p, *Rinv = small + 3 * (size_t)p * p;
  double *theta = small + 4 * (size_t)p * p, *invt = theta + p, *res = theta + 2 * p, *thl = theta + 3 * p;
  double* ncol = theta + 4 * p;
  int* flags = reinterpret_cast<int*>(theta + 6 * p);

  // The iteration works on the deflated Gram G' = G - sum_locked theta_t x_t x_t^T (fp64 master
  // copy Gd, fp32 copy G32 for the tensor-core products).
  cudaMemcpyAsync(Gd, G64, (size_t)m * m * 8, cudaMemcpyDeviceToDevice, s);
  g_to_f32_kernel<<<nblk((long long)m * ms, 256), 256, 0, s>>>(Gd, m, ms, G32);
  hash_fill_kernel<<<nblk((long long)mp, 256), 256, 0, s>>>(Y, m, p, 0x5EEDull, 1.0, 0);
  ctx->count_launch(2);
  if (opt.init_S) {  // warm start: the first k columns of the starting block are the given rows
    init_cols_kernel<<<nblk((long long)m * k, 256), 256, 0, s>>>(Y, m, p, opt.init_S, k);
    ctx->count_launch();
  }
  cudaMemsetAsync(flags, 0, 2 * sizeof(int), s);
  if ((st = cholqr2(ctx, Y, Q1, Q, m, p, C, Rinv, flags)) != TSK_OK) return st;
  // Working-precision floor of the Ritz residual: the 3xTF32 G Q products carry an error of
  // ~1e-8 ||G||_F (measured at C5, where ||G||_F / theta_1 = 61 and the residual stalls at 6e-7);
  // the requested tol is raised to 4x that floor, and a Ky Fan energy that no longer changes
  // (< 1e-12 relative over two outer iterations) also ends the iteration.
  fro2_part_kernel<<<128, 256, 0, s>>>(G64, (long long)m * m, X);  // X: scratch until the loop
  sum_kernel<<<1, 128, 0, s>>>(X, 128, ncol);
  ctx->count_launch(2);
  double gfro2 = 0.0;
  cudaMemcpyAsync(&gfro2, ncol, 8, cudaMemcpyDeviceToHost, s);
  if (cudaStreamSynchronize(s) != cudaSuccess) return TSK_ECUDA;
  const double gfro = std::sqrt(std::max(gfro2, 0.0));
  double kyfan_prev = -1.0, kf_change_prev = -1.0;
  int kyfan_still = 0;
  constexpr double kKyFanTol = 5e-7;  // estimated remaining Ky Fan deficit at the stop (half the 1e-6 check)

  GemmProblem gp;
  gp.X = G32;
  gp.Y = Qt;
  gp.M = m;
  gp.n = m;
  gp.D = 1;
  gp.x_row_stride = ms;
  gp.x_slice_stride = (long long)m * ms;
  gp.y_row_stride = ms;
  gp.min_chunks_per_unit = 2;
  gp.chain = 1;  // short TMEM chains: the eigensolver needs G Q to ~3e-7, not ~1e-6

  // Z = G' B for an m x pa fp64 block B (fp32 copy for the tensor cores; B <- fp64(fp32(B)))
  auto gq = [&](double* B, int pa) -> tsk_status {
    if (f64) return gemm_nn_f64(ctx, Gd, m, 0, B, pa, 0, m, m, pa, 1, nullptr, Z, pa, 0);
    q_to_f32t_kernel<<<nblk((long long)pa * ms, 256), 256, 0, s>>>(B, m, pa, ms, Qt);
    ctx->count_launch();
    gp.N = pa;
    gp.y_slice_stride = (long long)pa * ms;
    gp.out64 = Z;
    gp.ldo64 = pa;
    return gemm_tf32x3(ctx, gp);
  };

  // Outer iteration: Rayleigh-Ritz on span(Q) -> convergence test -> lock + deflate the leading
  // converged Ritz pairs that sit well above the wanted edge -> Chebyshev filter of degree d on
  // [0, b] (b = smallest Ritz value of the block) applied to the remaining Ritz vectors, with d
  // the largest degree keeping the filter's dynamic range T_d(x_max) <= 1e6 (so CholQR2 stays
  // accurate) -> CholQR2.  Deflating the dominant pairs (C3/C4: the frame mean is 1e4 x the rest)
  // is what makes the filter usable; on its own each filter degree replaces d power steps.
  int nl = 0;           // locked pairs
  int pa = p;           // active block size
  int outer = 0, products = 0;
  bool converged = false;
  double max_res = 0.0, kyfan = 0.0, theta_top = 0.0;
  int repairs = 0;
  if (!opt.init_S) {
    // One plain power step from the random start before the first Rayleigh-Ritz: the Ritz pairs of
    // a random block are not worth a p x p eigensolve (C4: 7 Jacobi sweeps).  G Q's columns are all
    // pulled toward x_1 (cond ~ lambda_1 / lambda_p, 2.5e4 at C4), well within CholQR2's fp64 reach;
    // if it breaks down anyway (extreme spectra) the random block is kept.
    cudaMemcpyAsync(Y0, Q, (size_t)m * pa * 8, cudaMemcpyDeviceToDevice, s);
    if ((st = gq(Q, pa)) != TSK_OK) return st;
    ++products;
    cudaMemsetAsync(flags, 0, 2 * sizeof(int), s);
    if ((st = cholqr2(ctx, Z, Q1, Q, m, pa, C, Rinv, flags)) != TSK_OK) return st;
    int hf[2] = {0, 0};
    if (cudaMemcpyAsync(hf, flags, sizeof(hf), cudaMemcpyDeviceToHost, s) != cudaSuccess ||
        cudaStreamSynchronize(s) != cudaSuccess)
      return TSK_ECUDA;
    if (hf[0] | hf[1]) {
      cudaMemcpyAsync(Q, Y0, (size_t)m * pa * 8, cudaMemcpyDeviceToDevice, s);
      cudaMemsetAsync(flags, 0, 2 * sizeof(int), s);
    }
  }
  for (outer = 1; outer <= max_iters; ++outer) {
    const int kr = k - nl;  // wanted pairs still active
    if ((st = gq(Q, pa)) != TSK_OK) return st;
    ++products;
    if ((st = gemm_tn_f64(ctx, Q, pa, 0, Z, pa, 0, m, pa, pa, 1, H, pa, 0, 1, WS_EIG_SMALL)) != TSK_OK) return st;
    // Rayleigh-Ritz accuracy follows the iteration: a Jacobi threshold tau leaves the Ritz vectors
    // mixed by ~tau, which inflates their residuals by ~tau theta and leaves span(Q) unchanged, so
    // tau = 0.1 x the previous max residual (1e-3 on the first, random, block) costs nothing in
    // convergence, and the residual test below measures the vectors actually produced.
    const double tol_rr = outer == 1 ? 1e-3 : std::max(f64 ? 1e-12 : 1e-9, std::min(1e-3, 0.1 * max_res));
    if ((st = jacobi_eig_batched(ctx, H, pa, 1, W, theta, flags + 2, tol_rr)) != TSK_OK) return st;
    inv_theta_kernel<<<nblk(pa, 128), 128, 0, s>>>(theta, pa, invt);
    ctx->count_launch();
    if ((st = gemm_nn_f64(ctx, Z, pa, 0, W, pa, 0, m, pa, pa, 1, invt, Y, pa, 0)) != TSK_OK) return st;  // G'X/theta
    if ((st = gemm_nn_f64(ctx, Q, pa, 0, W, pa, 0, m, pa, pa, 1, nullptr, X, pa, 0)) != TSK_OK) return st;  // X = QW
    ritz_residual_kernel<<<kr, 256, 0, s>>>(Y, X, theta, m, pa, res);
    ctx->count_launch();
    cudaMemcpyAsync(hostbuf, theta, (size_t)pa * 8, cudaMemcpyDeviceToHost, s);
    cudaMemcpyAsync(hostbuf + p, res, (size_t)kr * 8, cudaMemcpyDeviceToHost, s);
    cudaMemcpyAsync(hostbuf + 2 * p, flags, 3 * sizeof(int), cudaMemcpyDeviceToHost, s);
    cudaMemsetAsync(flags, 0, 2 * sizeof(int), s);
    if (cudaStreamSynchronize(s) != cudaSuccess) return TSK_ECUDA;
    const double* hth = hostbuf;
    const double* hres = hostbuf + p;
    const int* hflags = reinterpret_cast<const int*>(hostbuf + 2 * p);
    if (nl == 0) theta_top = hth[0];
    double kf_now = 0.0;    // Ky Fan energy of the current k wanted values (locked + active)
    double locked2 = 0.0;   // sum of the squared locked Ritz values
    {
      std::vector<double> hl(nl);
      if (nl > 0) {
        cudaMemcpyAsync(hl.data(), thl, (size_t)nl * 8, cudaMemcpyDeviceToHost, s);
        cudaStreamSynchronize(s);
      }
      for (double v : hl) {
        kf_now += v;
        locked2 += v * v;
      }
      for (int c = 0; c < kr; ++c) kf_now += hth[c];
    }
    // residual scale: theta_1 (reading c15), or with tol_active the top of the active (deflated)
    // block, whose Gram norm ||G'||_F ~ sqrt(||G||_F^2 - sum locked theta^2) also sets the floor
    const bool act = opt.tol_active && nl > 0 && hth[0] > 0.0;
    const double ref = act ? hth[0] : theta_top;
    const double gref = act ? std::sqrt(std::max(gfro2 - locked2, 0.0)) : gfro;
    max_res = 0.0;
    for (int c = 0; c < kr; ++c) max_res = std::max(max_res, hres[c]);
    max_res /= ref > 0 ? ref : 1.0;
    const double floor_rel = f64 ? 1e-14 : 4e-8;  // working-precision floor of the G Q products
    const double tol_eff = std::max(tol, ref > 0 ? floor_rel * gref / ref : tol);
    // Ky Fan convergence: the residual test alone (relative to theta_1) stops too early when a dominant
    // eigenvalue sits far above a flat rest (measured: deficits up to 1.2e-5 after 16 products,
    // scripts/random_sweep5.py); the remaining deficit is extrapolated from the last two changes of
    // the Ky Fan energy (geometric convergence, ratio rho) and must also be small
    const double kf_change = kyfan_prev > 0 ? std::fabs(kf_now - kyfan_prev) : -1.0;
    double kf_remaining;  // estimated remaining Ky Fan deficit, relative
    if (kf_change < 0.0) {
      kf_remaining = max_res <= 0.1 * tol_eff ? 0.0 : INFINITY;  // first outer: only a block already converged
    } else {
      const double rho = kf_change_prev > 0.0 ? std::min(kf_change / kf_change_prev, 0.99) : 0.5;
      kf_remaining = kf_change * rho / (1.0 - rho) / std::max(kf_now, 1e-300);
    }
    kf_change_prev = kf_change;
    if (kf_change >= 0.0 && kf_change <= 1e-12 * kf_now) ++kyfan_still;
    else kyfan_still = 0;
    kyfan_prev = kf_now;
    if (getenv("TSK_EIG_TRACE"))
      fprintf(stderr, "[eig] outer=%d products=%d locked=%d max_res=%.3e (tol %.2e) theta0=%.4e theta_k=%.4e theta_p=%.4e "
              "kyfan=%.12e rr_sweeps=%d res0=%.3e cholqr_flags=%d,%d\n", outer, products, nl, max_res, tol_eff, hth[0],
              hth[kr - 1], hth[pa - 1], kf_now, hflags[2], hres[0] / theta_top, hflags[0], hflags[1]);
    if (hflags[0] + hflags[1] > 0) {
      // rank-deficient block (rank(G) < p): perturb with fresh directions and re-orthonormalise
      if (++repairs > 8) return TSK_ECUDA;
      cudaMemcpyAsync(Y, Q, (size_t)m * pa * 8, cudaMemcpyDeviceToDevice, s);
      hash_fill_kernel<<<nblk((long long)m * pa, 256), 256, 0, s>>>(Y, m, pa, 0xBADC0DEull + repairs, 1e-3, 1);
      ctx->count_launch();
      if ((st = cholqr2(ctx, Y, Q1, Q, m, pa, C, Rinv, flags)) != TSK_OK) return st;
      continue;
    }
    if ((max_res <= tol_eff && kf_remaining <= kKyFanTol) || (kyfan_still >= 2 && max_res <= 1e-4)) {
      converged = true;
      break;
    }
    if (outer == max_iters) break;
    // ---- lock the leading converged pairs well above the wanted edge (theta >= 2 theta_{k-1})
    int nnew = 0;
    while (nnew < kr - 1 && hres[nnew] <= tol * ref && hth[nnew] >= 2.0 * hth[kr - 1]) ++nnew;
    const double* tha = theta;  // device Ritz values of the active block
    int off = 0;                // first active column of X / theta after locking
    if (nnew > 0) {
      copy_cols_kernel<<<nblk((long long)m * nnew, 256), 256, 0, s>>>(X, pa, 0, Xl, p, nl, m, nnew);
      cudaMemcpyAsync(thl + nl, theta, (size_t)nnew * 8, cudaMemcpyDeviceToDevice, s);
      deflate_kernel<<<nblk((long long)m * m, 256), 256, 0, s>>>(Gd, m, X, pa, 0, nnew, theta);
      g_to_f32_kernel<<<nblk((long long)m * ms, 256), 256, 0, s>>>(Gd, m, ms, G32);
      ctx->count_launch(3);
      nl += nnew;
      off = nnew;
    }
    const int pn = pa - off;
    // ---- Chebyshev filter on [0, b] applied to the remaining Ritz vectors X[:, off:pa]
    const double b = hth[pa - 1];
    // the filter's dynamic range is set by the top of the spectrum: after the first Rayleigh-Ritz
    // step (random start) theta_0 can underestimate lambda_max by orders of magnitude (C4: 7.7e6 vs
    // 1.04e9), and a filter designed on it overflows the block into one direction (CholQR breaks
    // down); there the upper bound ||G||_F >= lambda_max is used instead
    const double top = outer == 1 ? std::max(hth[off], gfro) : hth[off];
    const double xmax = 2.0 * top / b - 1.0;
    int d = 1;
    if (b > 0.0 && xmax > 1.0 + 1e-12) {
      const double ach = acosh(xmax);
      d = (int)std::floor(std::log(2e6) / ach);  // T_d(x) ~ exp(d acosh x) / 2 <= 1e6
      d = std::max(1, std::min(d, opt.cheb_degree > 0 ? std::min(12, opt.cheb_degree) : 12));
    }
    if (getenv("TSK_EIG_TRACE")) fprintf(stderr, "[eig]   lock %d, filter degree %d on [0, %.4e], x_max %.3e\n", nnew, d, b, xmax);
    copy_cols_kernel<<<nblk((long long)m * pn, 256), 256, 0, s>>>(X, pa, off, Y0, pn, 0, m, pn);
    ctx->count_launch();
    if (d == 1) {
      // plain step Y = G' X / theta (the scaled power step of the previous version)
      copy_cols_kernel<<<nblk((long long)m * pn, 256), 256, 0, s>>>(Y, pa, off, Y1, pn, 0, m, pn);
      ctx->count_launch();
    } else {
      const double cc = 0.5 * b, ee = 0.5 * b;
      double* Yprev = nullptr;
      double* Ycur = Y0;
      double* Ynext = Y1;
      double* spare = Q1;  // free until the CholQR below
      for (int j = 1; j <= d; ++j) {
        if ((st = gq(Ycur, pn)) != TSK_OK) return st;
        ++products;
        const double alpha = (j == 1) ? 1.0 / ee : 2.0 / ee;
        cheb_step_kernel<<<nblk((long long)m * pn, 256), 256, 0, s>>>(Z, Ycur, Yprev, (long long)m * pn, cc, alpha,
                                                                       j == 1 ? 0.0 : 1.0, Ynext);
        ctx->count_launch();
        double* t = Yprev ? Yprev : spare;
        Yprev = Ycur;
        Ycur = Ynext;
        Ynext = t;
      }
      // normalise the filtered columns (their norms spread up to T_d(x_max)) into Y1
      inv_colnorm_kernel<<<pn, 256, 0, s>>>(Ycur, m, pn, ncol);
      colscale_kernel<<<nblk((long long)m * pn, 256), 256, 0, s>>>(Ycur, ncol, m, pn, Y1);
      ctx->count_launch(2);
    }
    pa = pn;
    if (nl > 0) {
      // keep the active block orthogonal to the locked vectors: Y1 -= Xl (Xl^T Y1)
      if ((st = gemm_tn_f64(ctx, Xl, p, 0, Y1, pa, 0, m, nl, pa, 1, C, pa, 0, 0, WS_EIG_SMALL)) != TSK_OK) return st;
      if ((st = gemm_nn_f64(ctx, Xl, p, 0, C, pa, 0, m, nl, pa, 1, nullptr, Q1, pa, 0)) != TSK_OK) return st;
      cheb_step_kernel<<<nblk((long long)m * pa, 256), 256, 0, s>>>(Y1, Y1, Q1, (long long)m * pa, 0.0, 1.0, 1.0, Y1);
      ctx->count_launch();
    }
    if ((st = cholqr2(ctx, Y1, Q1, Q, m, pa, C, Rinv, flags)) != TSK_OK) return st;
    (void)tha;
  }
  // output: locked pairs first (largest), then the leading active Ritz pairs; a final CholQR2 of
  // the combined k columns (Gram-Schmidt order: locked columns are kept, active ones are made
  // orthogonal to them) removes the residual locked/active coupling of the deflated iteration
  const int kr = k - nl;
  double* Xo = Y0;
  if (nl > 0) copy_cols_kernel<<<nblk((long long)m * nl, 256), 256, 0, s>>>(Xl, p, 0, Xo, k, 0, m, nl);
  copy_cols_kernel<<<nblk((long long)m * kr, 256), 256, 0, s>>>(X, pa, 0, Xo, k, nl, m, kr);
  ctx->count_launch(2);
  if (nl > 0) {
    if ((st = cholqr2(ctx, Xo, Q1, Y1, m, k, C, Rinv, flags)) != TSK_OK) return st;
    Xo = Y1;
  }
  write_sketch_kernel<<<k, 256, 0, s>>>(Xo, m, k, S);
  ctx->count_launch();
  if (X64) cudaMemcpyAsync(X64, Xo, (size_t)m * k * 8, cudaMemcpyDeviceToDevice, s);
  if (lambda) {
    if (nl > 0) cudaMemcpyAsync(lambda, thl, (size_t)nl * 8, cudaMemcpyDeviceToDevice, s);
    cudaMemcpyAsync(lambda + nl, theta, (size_t)kr * 8, cudaMemcpyDeviceToDevice, s);
  }
  if (info) {
    info->iters = products;
    std::vector<double> hl(k);
    cudaMemcpyAsync(hl.data(), thl, (size_t)nl * 8, cudaMemcpyDeviceToHost, s);
    cudaMemcpyAsync(hl.data() + nl, theta, (size_t)kr * 8, cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    kyfan = 0.0;
    for (double v : hl) kyfan += v;
    info->kyfan = kyfan;
    info->max_resid = max_res;
    // hostbuf holds the Ritz values of the last Rayleigh-Ritz step (active block, decreasing)
    info->gap_est = (kr >= 1 && kr < pa && hostbuf[kr] > 0.0) ? hostbuf[kr - 1] / hostbuf[kr] : INFINITY;
  }
  if (cudaPeekAtLastError() != cudaSuccess) return TSK_ECUDA;
  return converged ? TSK_OK : TSK_WARN_NOT_CONVERGED;
}

}  // namespace tsk
