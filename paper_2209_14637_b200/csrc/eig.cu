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
static tsk_status cholqr1(Ctx* ctx, const double* Y, double* Q, int m, int p, double* C, double* L, int* flags) {
  tsk_status st;
  if ((st = gemm_tn_f64(ctx, Y, p, 0, Y, p, 0, m, p, p, 1, C, p, 0, 1, WS_EIG_SMALL)) != TSK_OK) return st;
  if ((st = chol(ctx, C, p, 1, 1e-13, L, flags, WS_JACOBI)) != TSK_OK) return st;
  return trsm_rlt(ctx, Y, L, m, p, Q);
}

static tsk_status cholqr2(Ctx* ctx, const double* Y, double* Q1, double* Q, int m, int p, double* C, double* L,
                          int* flags) {
  tsk_status st;
  if ((st = gemm_tn_f64(ctx, Y, p, 0, Y, p, 0, m, p, p, 1, C, p, 0, 1, WS_EIG_SMALL)) != TSK_OK) return st;
  if ((st = chol(ctx, C, p, 1, 1e-13, L, flags, WS_JACOBI)) != TSK_OK) return st;
  if ((st = trsm_rlt(ctx, Y, L, m, p, Q1)) != TSK_OK) return st;
  if ((st = gemm_tn_f64(ctx, Q1, p, 0, Q1, p, 0, m, p, p, 1, C, p, 0, 1, WS_EIG_SMALL)) != TSK_OK) return st;
  if ((st = chol(ctx, C, p, 1, 1e-13, L, flags + 1, WS_JACOBI)) != TSK_OK) return st;
  return trsm_rlt(ctx, Q1, L, m, p, Q);
}

tsk_status topk_eigen(Ctx* ctx, const double* G64, int m, int k, float* S, double* lambda,
                      const tsk_train_opts* o, tsk_train_info* info) {
  if (m < 1 || k < 1 || k > m) return TSK_EINVAL;
  tsk_train_opts opt{};
  if (o) opt = *o;
  const int dense_max = opt.dense_max_m > 0 ? opt.dense_max_m : 256;
  const int max_iters = opt.max_iters > 0 ? opt.max_iters : 300;
  const double tol = opt.tol > 0 ? opt.tol : 5e-7;

  // block size p = k + 16 by default: measured on C3/C4 spectra (flat near k), larger blocks cut
  // iterations less than they raise the cost of each p x p Rayleigh-Ritz solve
  int p = opt.oversample > 0 ? k + opt.oversample : k + 16;
  p = std::min(p, m);
  cudaStream_t s = ctx->stream;
  tsk_status st;

  if (m <= dense_max || p >= m || m <= 256) {
    if (m > 256) return TSK_EINVAL;
    double* W = reinterpret_cast<double*>(ctx->workspace(WS_EIG_A, (size_t)m * m * 8));
    double* lam = reinterpret_cast<double*>(ctx->workspace(WS_EIG_SMALL, (size_t)m * 8 + 64));
    if (!W || !lam) return TSK_ENOMEM;
    if ((st = jacobi_eig_batched(ctx, G64, m, 1, W, lam)) != TSK_OK) return st;
    write_sketch_kernel<<<k, 256, 0, s>>>(W, m, m, S);
    ctx->count_launch();
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
    }
    return cudaPeekAtLastError() == cudaSuccess ? TSK_OK : TSK_ECUDA;
  }

  const int ms = (m + 3) & ~3;
  const size_t mp = (size_t)m * p;
  // workspace carve-up
  double* big = reinterpret_cast<double*>(ctx->workspace(WS_EIG_A, mp * 8 * 5));
  double* small = reinterpret_cast<double*>(ctx->workspace(WS_EIG_B, ((size_t)p * p * 4 + p * 8) * 8 + 256));
  float* G32 = reinterpret_cast<float*>(ctx->workspace(WS_EIG_G32, (size_t)m * ms * 4));
  float* Qt = reinterpret_cast<float*>(ctx->workspace(WS_EIG_Q32, (size_t)p * ms * 4));
  double* hostbuf = reinterpret_cast<double*>(ctx->pinned((size_t)(4 * p + 16) * 8));
  if (!big || !small || !G32 || !Qt || !hostbuf) return TSK_ENOMEM;
  double *Q = big, *Z = big + mp, *X = big + 2 * mp, *Y = big + 3 * mp, *Q1 = big + 4 * mp;
  double *H = small, *W = small + (size_t)p * p, *C = small + 2 * (size_t)p * p, *Rinv = small + 3 * (size_t)p * p;
  double *theta = small + 4 * (size_t)p * p, *invt = theta + p, *res = theta + 2 * p;
  int* flags = reinterpret_cast<int*>(theta + 5 * p);

  g_to_f32_kernel<<<nblk((long long)m * ms, 256), 256, 0, s>>>(G64, m, ms, G32);
  hash_fill_kernel<<<nblk((long long)mp, 256), 256, 0, s>>>(Y, m, p, 0x5EEDull, 1.0, 0);
  ctx->count_launch(2);
  if ((st = cholqr2(ctx, Y, Q1, Q, m, p, C, Rinv, flags)) != TSK_OK) return st;

  GemmProblem gp;
  gp.X = G32;
  gp.Y = Qt;
  gp.M = m;
  gp.N = p;
  gp.n = m;
  gp.D = 1;
  gp.x_row_stride = ms;
  gp.x_slice_stride = (long long)m * ms;
  gp.y_row_stride = ms;
  gp.y_slice_stride = (long long)p * ms;
  gp.sym = 0;
  gp.out64 = Z;
  gp.ldo64 = p;
  gp.min_chunks_per_unit = 2;
  gp.chain = 1;  // short TMEM chains: the eigensolver needs G Q to ~3e-7, not ~1e-6

  // Rayleigh-Ritz (and the convergence test) every `rr_every` iterations; span(Q) -- and so
  // the convergence of the subspace -- does not depend on the basis, so the iterations in
  // between only orthonormalise Y = G Q diag(1/theta) (columns stay aligned with the last
  // Ritz vectors, which keeps Y well conditioned).
  const int rr_every = 4;
  int it = 0;
  bool converged = false;
  double max_res = 0.0, kyfan = 0.0;
  int repairs = 0;
  cudaMemsetAsync(flags, 0, 2 * sizeof(int), s);
  for (it = 1; it <= max_iters; ++it) {
    q_to_f32t_kernel<<<nblk((long long)p * ms, 256), 256, 0, s>>>(Q, m, p, ms, Qt);
    ctx->count_launch();
    if ((st = gemm_tf32x3(ctx, gp)) != TSK_OK) return st;  // Z = G Q
    const bool do_rr = (it % rr_every) == 1 || rr_every == 1 || it == max_iters;
    if (!do_rr) {
      colscale_kernel<<<nblk((long long)mp, 256), 256, 0, s>>>(Z, invt, m, p, Y);
      ctx->count_launch();
      // one CholQR pass between checks (Y is column-scaled, so orthonormal to ~cond(Y)^2 eps),
      // two passes before the Rayleigh-Ritz check
      const bool next_rr = ((it + 1) % rr_every) == 1 || it + 1 == max_iters;
      if ((st = next_rr ? cholqr2(ctx, Y, Q1, Q, m, p, C, Rinv, flags) : cholqr1(ctx, Y, Q, m, p, C, Rinv, flags)) !=
          TSK_OK)
        return st;
      continue;
    }
    if ((st = gemm_tn_f64(ctx, Q, p, 0, Z, p, 0, m, p, p, 1, H, p, 0, 1, WS_EIG_SMALL)) != TSK_OK) return st;  // H
    // loose rotation threshold: the Rayleigh-Ritz basis only needs ~1e-9 accuracy (span(Q) carries the
    // convergence; S is returned in fp32), and it saves most of the Jacobi sweeps
    if ((st = jacobi_eig_batched(ctx, H, p, 1, W, theta, nullptr, 1e-9)) != TSK_OK) return st;
    inv_theta_kernel<<<nblk(p, 128), 128, 0, s>>>(theta, p, invt);
    ctx->count_launch();
    if ((st = gemm_nn_f64(ctx, Z, p, 0, W, p, 0, m, p, p, 1, invt, Y, p, 0)) != TSK_OK) return st;     // Y = GX/theta
    if ((st = gemm_nn_f64(ctx, Q, p, 0, W, p, 0, m, p, p, 1, nullptr, X, p, 0)) != TSK_OK) return st;  // X = QW
    ritz_residual_kernel<<<k, 256, 0, s>>>(Y, X, theta, m, p, res);
    ctx->count_launch();
    // host check: theta[0..k), res[0..k), pivot flags of the orthonormalisations since the last check
    cudaMemcpyAsync(hostbuf, theta, (size_t)k * 8, cudaMemcpyDeviceToHost, s);
    cudaMemcpyAsync(hostbuf + p, res, (size_t)k * 8, cudaMemcpyDeviceToHost, s);
    cudaMemcpyAsync(hostbuf + 2 * p, flags, 2 * sizeof(int), cudaMemcpyDeviceToHost, s);
    cudaMemsetAsync(flags, 0, 2 * sizeof(int), s);
    if (cudaStreamSynchronize(s) != cudaSuccess) return TSK_ECUDA;
    const int* hflags = reinterpret_cast<const int*>(hostbuf + 2 * p);
    const int ndeg = hflags[0] + hflags[1];
    kyfan = 0.0;
    max_res = 0.0;
    for (int c = 0; c < k; ++c) {
      kyfan += hostbuf[c];
      max_res = std::max(max_res, hostbuf[p + c]);
    }
    max_res = hostbuf[0] > 0 ? max_res / hostbuf[0] : max_res;
    if (getenv("TSK_EIG_TRACE")) {
      int am = 0;
      for (int c = 0; c < k; ++c)
        if (hostbuf[p + c] > hostbuf[p + am]) am = c;
      fprintf(stderr, "[eig] it=%d max_res=%.3e at c=%d theta_c=%.6e theta_0=%.6e theta_k-1=%.6e flags=%d\n", it,
              max_res, am, hostbuf[am], hostbuf[0], hostbuf[k - 1], ndeg);
    }
    if (ndeg > 0) {
      // rank-deficient block (rank(G) < p): perturb with fresh directions and re-orthonormalise
      if (++repairs > 8) return TSK_ECUDA;
      hash_fill_kernel<<<nblk((long long)mp, 256), 256, 0, s>>>(Y, m, p, 0xBADC0DEull + repairs, 1e-3, 1);
      ctx->count_launch();
      if ((st = cholqr2(ctx, Y, Q1, Q, m, p, C, Rinv, flags)) != TSK_OK) return st;
      continue;
    }
    if (max_res <= tol) {
      converged = true;
      break;
    }
    if (it == max_iters) break;
    if ((st = cholqr2(ctx, Y, Q1, Q, m, p, C, Rinv, flags)) != TSK_OK) return st;
  }
  write_sketch_kernel<<<k, 256, 0, s>>>(X, m, p, S);
  ctx->count_launch();
  if (lambda) cudaMemcpyAsync(lambda, theta, (size_t)k * 8, cudaMemcpyDeviceToDevice, s);
  if (info) {
    info->iters = std::min(it, max_iters);
    info->kyfan = kyfan;
    info->max_resid = max_res;
  }
  if (cudaPeekAtLastError() != cudaSuccess) return TSK_ECUDA;
  return converged ? TSK_OK : TSK_WARN_NOT_CONVERGED;
}

}  // namespace tsk
