// Batched SCW (Algorithm 1) and per-matrix errors on the test stream.
//
// For each test matrix A_b (m x n) and sketch S (k x m):
//   1. B   = S A_b                        (k x n)   -- Alg. 1 line 1 operand
//   2. V^T = orthonormal basis of rowspace(B) (k x n): eigen-orthonormalisation
//            B B^T = W diag(mu) W^T,  V^T = diag(mu^{-1/2}) W^T B  (directions with
//            mu <= 1e-13 mu_max dropped; reading c2).  "The full SVD in line 1 is used for
//            orthogonalization ... can be replaced" -- any orthonormal basis of the
//            row space gives the same A_hat.
//   3. Z^T = (A_b V)^T                     (k x m)
//   4. Z^T Z = W2 diag(sigma^2) W2^T       (the SVD of AV, line 2, through its k x k Gram)
//   5. L = Z W2_r = U2_r diag(sigma_r) (m x r),  R = V W2_r (n x r)  =>  A_hat = [AV]_r V^T = L R^T
//   6. e_b = ||A_b - L R^T||_F             dense residual, fp64 reduction (not the identity
//            ||A||^2 - sum sigma^2, which cancels catastrophically)
// Products 1, 3, 6 accumulate fp32 products on CUDA cores; small Gram / rotation steps are
// fp64.  Everything is batched over b (grid.y / grid.z) with deterministic reductions.
#include <algorithm>
#include <cmath>

#include "ptx.cuh"
#include "tsk_internal.h"

namespace tsk {

// ---------------------------------------------------------------- 1. B = S A
template <int KMAX>
__global__ void __launch_bounds__(128) scw_sa_kernel(const float* __restrict__ A, const float* __restrict__ S, int m,
                                                     int n, int k, float* __restrict__ Bm) {
  __shared__ float Ss[KMAX][33];
  const int b = blockIdx.y;
  const int j = blockIdx.x * 128 + threadIdx.x;
  const float* Ab = A + (size_t)b * m * n;
  float acc[KMAX];
#pragma unroll
  for (int c = 0; c < KMAX; ++c) acc[c] = 0.f;
  for (int i0 = 0; i0 < m; i0 += 32) {
    for (int e = threadIdx.x; e < KMAX * 32; e += 128) {
      const int c = e >> 5, ii = e & 31;
      Ss[c][ii] = (c < k && i0 + ii < m) ? S[(size_t)c * m + i0 + ii] : 0.f;
    }
    __syncthreads();
    if (j < n) {
      const int lim = min(32, m - i0);
      for (int ii = 0; ii < lim; ++ii) {
        const float a = Ab[(size_t)(i0 + ii) * n + j];
#pragma unroll
        for (int c = 0; c < KMAX; ++c) acc[c] = fmaf(Ss[c][ii], a, acc[c]);
      }
    }
    __syncthreads();
  }
  if (j < n) {
    float* Bb = Bm + (size_t)b * k * n;
#pragma unroll
    for (int c = 0; c < KMAX; ++c)
      if (c < k) Bb[(size_t)c * n + j] = acc[c];
  }
}

// ---------------------------------------------------------------- C = X X^T (rows of an fp32 k x len matrix), fp64
// grid (ceil(npairs / (256*kPer)), batch); each thread owns kPer lower-triangle pairs (a >= c).
constexpr int kGramPer = 8;
__global__ void __launch_bounds__(256) gram_rows_kernel(const float* __restrict__ X, int k, int len,
                                                        double* __restrict__ C) {
  extern __shared__ float xs[];  // [k][65]
  const int b = blockIdx.y;
  const float* Xb = X + (size_t)b * k * len;
  const int npairs = k * (k + 1) / 2;
  double acc[kGramPer];
  int pa[kGramPer], pc[kGramPer];
#pragma unroll
  for (int u = 0; u < kGramPer; ++u) {
    acc[u] = 0.0;
    const int e = blockIdx.x * 256 * kGramPer + u * 256 + threadIdx.x;
    if (e < npairs) {
      int a = (int)((sqrtf(8.0f * e + 1.0f) - 1.0f) * 0.5f);
      while ((a + 1) * (a + 2) / 2 <= e) ++a;
      while (a * (a + 1) / 2 > e) --a;
      pa[u] = a;
      pc[u] = e - a * (a + 1) / 2;
    } else {
      pa[u] = -1;
      pc[u] = 0;
    }
  }
  for (int j0 = 0; j0 < len; j0 += 64) {
    for (int e = threadIdx.x; e < k * 64; e += 256) {
      const int a = e >> 6, jj = e & 63;
      xs[a * 65 + jj] = (j0 + jj < len) ? Xb[(size_t)a * len + j0 + jj] : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int u = 0; u < kGramPer; ++u) {
      if (pa[u] >= 0) {
        const float* ra = xs + pa[u] * 65;
        const float* rc = xs + pc[u] * 65;
        double s = 0.0;
#pragma unroll 8
        for (int jj = 0; jj < 64; ++jj) s += (double)ra[jj] * (double)rc[jj];
        acc[u] += s;
      }
    }
    __syncthreads();
  }
  double* Cb = C + (size_t)b * k * k;
#pragma unroll
  for (int u = 0; u < kGramPer; ++u)
    if (pa[u] >= 0) {
      Cb[(size_t)pa[u] * k + pc[u]] = acc[u];
      Cb[(size_t)pc[u] * k + pa[u]] = acc[u];
    }
}

static void launch_gram_rows(const float* X, int k, int len, int batch, double* C, cudaStream_t s) {
  const int npairs = k * (k + 1) / 2;
  dim3 g((npairs + 256 * kGramPer - 1) / (256 * kGramPer), batch);
  gram_rows_kernel<<<g, 256, (size_t)k * 65 * 4, s>>>(X, k, len, C);
}

// ---------------------------------------------------------------- 2. V^T = diag(mu^-1/2) W^T B
__global__ void __launch_bounds__(256) scw_vt_kernel(const float* __restrict__ Bm, const double* __restrict__ Wc,
                                                     const double* __restrict__ mu, int k, int n,
                                                     float* __restrict__ Vt) {
  extern __shared__ double ws[];  // [k][k] W, then [k] scale
  const int b = blockIdx.y;
  const double* Wb = Wc + (size_t)b * k * k;
  for (int e = threadIdx.x; e < k * k; e += blockDim.x) ws[e] = Wb[e];
  double* sc = ws + k * k;
  if (threadIdx.x < k) {
    const double m0 = mu[(size_t)b * k];
    const double mc = mu[(size_t)b * k + threadIdx.x];
    sc[threadIdx.x] = (mc > 0.0 && mc > 1e-13 * m0) ? 1.0 / sqrt(mc) : 0.0;
  }
  __syncthreads();
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  const float* Bb = Bm + (size_t)b * k * n;
  float* Vb = Vt + (size_t)b * k * n;
  for (int c = 0; c < k; ++c) {
    double s = 0.0;
    for (int a = 0; a < k; ++a) s += ws[a * k + c] * (double)Bb[(size_t)a * n + j];
    Vb[(size_t)c * n + j] = (float)(s * sc[c]);
  }
}

// ---------------------------------------------------------------- 3. Z^T = V^T A^T  (k x m)
template <int KMAX>
__global__ void __launch_bounds__(256) scw_av_kernel(const float* __restrict__ A, const float* __restrict__ Vt, int m,
                                                     int n, int k, float* __restrict__ Zt) {
  __shared__ float As[64][33];
  __shared__ float Vs[KMAX][33];
  const int b = blockIdx.y;
  const int i0 = blockIdx.x * 64;
  const int r = threadIdx.x & 63, g = threadIdx.x >> 6;
  const float* Ab = A + (size_t)b * m * n;
  const float* Vb = Vt + (size_t)b * k * n;
  constexpr int kOut = KMAX / 4;
  float acc[kOut];
#pragma unroll
  for (int u = 0; u < kOut; ++u) acc[u] = 0.f;
  for (int j0 = 0; j0 < n; j0 += 32) {
    for (int e = threadIdx.x; e < 64 * 32; e += 256) {
      const int ii = e >> 5, jj = e & 31;
      As[ii][jj] = (i0 + ii < m && j0 + jj < n) ? Ab[(size_t)(i0 + ii) * n + j0 + jj] : 0.f;
    }
    for (int e = threadIdx.x; e < KMAX * 32; e += 256) {
      const int c = e >> 5, jj = e & 31;
      Vs[c][jj] = (c < k && j0 + jj < n) ? Vb[(size_t)c * n + j0 + jj] : 0.f;
    }
    __syncthreads();
#pragma unroll 4
    for (int jj = 0; jj < 32; ++jj) {
      const float a = As[r][jj];
#pragma unroll
      for (int u = 0; u < kOut; ++u) acc[u] = fmaf(Vs[g + 4 * u][jj], a, acc[u]);
    }
    __syncthreads();
  }
  if (i0 + r < m) {
    float* Zb = Zt + (size_t)b * k * m;
#pragma unroll
    for (int u = 0; u < kOut; ++u) {
      const int c = g + 4 * u;
      if (c < k) Zb[(size_t)c * m + i0 + r] = acc[u];
    }
  }
}

// ---------------------------------------------------------------- 5. out[i][c] = sum_a In[a][i] W[a][c], c < r
__global__ void __launch_bounds__(256) scw_combine_kernel(const float* __restrict__ In, const double* __restrict__ W,
                                                          int k, int len, int r, float* __restrict__ Out) {
  extern __shared__ double wsm[];  // [k][r]
  const int b = blockIdx.y;
  const double* Wb = W + (size_t)b * k * k;
  for (int e = threadIdx.x; e < k * r; e += blockDim.x) wsm[e] = Wb[(size_t)(e / r) * k + (e % r)];
  __syncthreads();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= len) return;
  const float* Ib = In + (size_t)b * k * len;
  float* Ob = Out + (size_t)b * len * r;
  for (int c = 0; c < r; ++c) {
    double s = 0.0;
    for (int a = 0; a < k; ++a) s += (double)Ib[(size_t)a * len + i] * wsm[a * r + c];
    Ob[(size_t)i * r + c] = (float)s;
  }
}

__global__ void scw_sigma_kernel(const double* __restrict__ sig2, int k, int r, long long B, float* __restrict__ sigma) {
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= B * r) return;
  const long long b = idx / r;
  const int c = (int)(idx % r);
  sigma[idx] = (float)sqrt(fmax(sig2[b * k + c], 0.0));
}

// ---------------------------------------------------------------- 6. e^2 partials: sum (A - L R^T)^2
template <int RMAX>
__global__ void __launch_bounds__(256) scw_residual_kernel(const float* __restrict__ A, const float* __restrict__ L,
                                                           const float* __restrict__ R, int m, int n, int r,
                                                           int rows_per_block, double* __restrict__ part) {
  __shared__ float Ls[16][RMAX];
  __shared__ double red[256];
  const int b = blockIdx.y;
  const int tile = blockIdx.x;
  const float* Ab = A + (size_t)b * m * n;
  const float* Lb = L + (size_t)b * m * r;
  const float* Rb = R + (size_t)b * n * r;
  const int i_begin = tile * rows_per_block;
  const int i_end = min(m, i_begin + rows_per_block);
  double acc = 0.0;
  for (int jb = 0; jb < n; jb += 256) {
    const int j = jb + threadIdx.x;
    float rr[RMAX];
#pragma unroll
    for (int c = 0; c < RMAX; ++c) rr[c] = (j < n && c < r) ? Rb[(size_t)j * r + c] : 0.f;
    for (int i0 = i_begin; i0 < i_end; i0 += 16) {
      __syncthreads();
      for (int e = threadIdx.x; e < 16 * RMAX; e += 256) {
        const int ii = e / RMAX, c = e % RMAX;
        Ls[ii][c] = (i0 + ii < i_end && c < r) ? Lb[(size_t)(i0 + ii) * r + c] : 0.f;
      }
      __syncthreads();
      if (j < n) {
        const int lim = min(16, i_end - i0);
        for (int ii = 0; ii < lim; ++ii) {
          float pred = 0.f;
#pragma unroll
          for (int c = 0; c < RMAX; ++c) pred = fmaf(Ls[ii][c], rr[c], pred);
          const double d = (double)Ab[(size_t)(i0 + ii) * n + j] - (double)pred;
          acc += d * d;
        }
      }
    }
  }
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[(size_t)b * gridDim.x + tile] = red[0];
}

__global__ void scw_err_reduce_kernel(const double* __restrict__ part, int tiles, long long B, double* __restrict__ err) {
  const long long b = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  double s = 0.0;
  for (int t = 0; t < tiles; ++t) s += part[b * tiles + t];
  err[b] = sqrt(s);
}

static inline unsigned nb(long long n, int t) { return (unsigned)((n + t - 1) / t); }

tsk_status scw_run(Ctx* ctx, const float* A, long long B, int m, int n, const float* S, int k, int r, float* L,
                   float* R, float* sigma, double* err) {
  if (B == 0) return TSK_OK;
  if (k > 128 || r > 64) return TSK_EINVAL;
  cudaStream_t s = ctx->stream;
  const long long chunk = std::min<long long>(B, 512);
  const size_t kn = (size_t)k * n, km = (size_t)k * m, kk = (size_t)k * k;
  float* Bm = reinterpret_cast<float*>(ctx->workspace(WS_SCW_0, chunk * kn * 4));
  float* Vt = reinterpret_cast<float*>(ctx->workspace(WS_SCW_1, chunk * kn * 4));
  float* Zt = reinterpret_cast<float*>(ctx->workspace(WS_SCW_2, chunk * km * 4));
  double* small = reinterpret_cast<double*>(ctx->workspace(WS_SCW_3, chunk * (4 * kk + 2 * k) * 8));
  const int rows_per_block = 64;
  const int tiles = (m + rows_per_block - 1) / rows_per_block;
  float* Lw = reinterpret_cast<float*>(ctx->workspace(WS_SCW_4, chunk * ((size_t)m + n) * r * 4));
  double* part = reinterpret_cast<double*>(ctx->workspace(WS_SCW_5, chunk * (size_t)tiles * 8 + 64));
  if (!Bm || !Vt || !Zt || !small || !Lw || !part) return TSK_ENOMEM;
  double* Cb = small;
  double* Wc = small + chunk * kk;
  double* H = small + 2 * chunk * kk;
  double* W2 = small + 3 * chunk * kk;
  double* mu = small + 4 * chunk * kk;
  double* sig2 = mu + chunk * k;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(scw_vt_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
    cudaFuncSetAttribute(scw_combine_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
    attr = true;
  }
  tsk_status st;
  for (long long b0 = 0; b0 < B; b0 += chunk) {
    const int bc = (int)std::min(chunk, B - b0);
    const float* Ac = A + (size_t)b0 * m * n;
    // 1. B = S A
    dim3 gsa(nb(n, 128), bc);
    if (k <= 32) scw_sa_kernel<32><<<gsa, 128, 0, s>>>(Ac, S, m, n, k, Bm);
    else if (k <= 64) scw_sa_kernel<64><<<gsa, 128, 0, s>>>(Ac, S, m, n, k, Bm);
    else scw_sa_kernel<128><<<gsa, 128, 0, s>>>(Ac, S, m, n, k, Bm);
    // 2. orthonormal row basis of B
    launch_gram_rows(Bm, k, n, bc, Cb, s);
    ctx->count_launch(2);
    if ((st = jacobi_eig_batched(ctx, Cb, k, bc, Wc, mu)) != TSK_OK) return st;
    scw_vt_kernel<<<dim3(nb(n, 256), bc), 256, (kk + k) * 8, s>>>(Bm, Wc, mu, k, n, Vt);
    // 3. Z^T = V^T A^T
    dim3 gav(nb(m, 64), bc);
    if (k <= 32) scw_av_kernel<32><<<gav, 256, 0, s>>>(Ac, Vt, m, n, k, Zt);
    else if (k <= 64) scw_av_kernel<64><<<gav, 256, 0, s>>>(Ac, Vt, m, n, k, Zt);
    else scw_av_kernel<128><<<gav, 256, 0, s>>>(Ac, Vt, m, n, k, Zt);
    // 4. SVD of AV through its Gram
    launch_gram_rows(Zt, k, m, bc, H, s);
    ctx->count_launch(3);
    if ((st = jacobi_eig_batched(ctx, H, k, bc, W2, sig2)) != TSK_OK) return st;
    // 5. factors
    float* Lc = L ? L + (size_t)b0 * m * r : Lw;
    float* Rc = R ? R + (size_t)b0 * n * r : Lw + (size_t)chunk * m * r;
    scw_combine_kernel<<<dim3(nb(m, 256), bc), 256, (size_t)k * r * 8, s>>>(Zt, W2, k, m, r, Lc);
    scw_combine_kernel<<<dim3(nb(n, 256), bc), 256, (size_t)k * r * 8, s>>>(Vt, W2, k, n, r, Rc);
    ctx->count_launch(2);
    if (sigma) {
      scw_sigma_kernel<<<nb((long long)bc * r, 256), 256, 0, s>>>(sig2, k, r, bc, sigma + (size_t)b0 * r);
      ctx->count_launch();
    }
    // 6. dense residual
    if (err) {
      dim3 gres(tiles, bc);
      if (r <= 32) scw_residual_kernel<32><<<gres, 256, 0, s>>>(Ac, Lc, Rc, m, n, r, rows_per_block, part);
      else scw_residual_kernel<64><<<gres, 256, 0, s>>>(Ac, Lc, Rc, m, n, r, rows_per_block, part);
      scw_err_reduce_kernel<<<nb(bc, 128), 128, 0, s>>>(part, tiles, bc, err + b0);
      ctx->count_launch(2);
    }
    if (cudaPeekAtLastError() != cudaSuccess) return TSK_ECUDA;
  }
  return TSK_OK;
}

}  // namespace tsk
