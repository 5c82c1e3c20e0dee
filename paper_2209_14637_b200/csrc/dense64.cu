// Small fp64 dense kernels for the eigensolver and SCW (CUDA cores; these are the
// p x p / m x p pieces around the tensor-core products, latency- rather than
// throughput-bound).  Deterministic: split reductions are summed in fixed order.
#include <algorithm>
#include <cmath>

#include "dense64.cuh"
#include "ptx.cuh"

namespace tsk {

// global -> shared copy of n doubles by nthreads threads, 8 loads in flight per thread
__device__ __forceinline__ void copy_to_shared(double* dst, const double* __restrict__ src, int n, int tid,
                                               int nthreads) {
  int e = tid;
  for (; e + 7 * nthreads < n; e += 8 * nthreads) {
    double v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = src[e + u * nthreads];
#pragma unroll
    for (int u = 0; u < 8; ++u) dst[e + u * nthreads] = v[u];
  }
  for (; e < n; e += nthreads) dst[e] = src[e];
}

// ---------------------------------------------------------------- C = X^T Y (contraction over rows)
// X: [batch][m][p] (ldx), Y: [batch][m][q] (ldy), partial: [batch][splits][p][q]
__global__ void gemm_tn_f64_kernel(const double* __restrict__ X, long long ldx, long long sx,
                                   const double* __restrict__ Y, long long ldy, long long sy, int m, int p, int q,
                                   int splits, double* __restrict__ part) {
  __shared__ double Xs[32][33];
  __shared__ double Ys[32][33];
  const int b = blockIdx.z / splits;
  const int sp = blockIdx.z % splits;
  const int a0 = blockIdx.y * 32, c0 = blockIdx.x * 32;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;  // 256 threads
  const int r0 = (int)((long long)sp * m / splits), r1 = (int)((long long)(sp + 1) * m / splits);
  const double* Xb = X + (size_t)b * sx;
  const double* Yb = Y + (size_t)b * sy;
  double acc[2][2] = {{0, 0}, {0, 0}};
  for (int i0 = r0; i0 < r1; i0 += 32) {
    for (int e = threadIdx.x; e < 32 * 32; e += 256) {
      const int ii = e >> 5, cc = e & 31;
      const int i = i0 + ii;
      Xs[ii][cc] = (i < r1 && a0 + cc < p) ? Xb[(size_t)i * ldx + a0 + cc] : 0.0;
      Ys[ii][cc] = (i < r1 && c0 + cc < q) ? Yb[(size_t)i * ldy + c0 + cc] : 0.0;
    }
    __syncthreads();
#pragma unroll 8
    for (int ii = 0; ii < 32; ++ii) {
      const double x0 = Xs[ii][ty * 2], x1 = Xs[ii][ty * 2 + 1];
      const double y0 = Ys[ii][tx * 2], y1 = Ys[ii][tx * 2 + 1];
      acc[0][0] += x0 * y0;
      acc[0][1] += x0 * y1;
      acc[1][0] += x1 * y0;
      acc[1][1] += x1 * y1;
    }
    __syncthreads();
  }
  double* P = part + ((size_t)b * splits + sp) * p * q;
#pragma unroll
  for (int u = 0; u < 2; ++u)
#pragma unroll
    for (int v = 0; v < 2; ++v) {
      const int a = a0 + ty * 2 + u, c = c0 + tx * 2 + v;
      if (a < p && c < q) P[(size_t)a * q + c] = acc[u][v];
    }
}

__global__ void reduce_splits_kernel(const double* __restrict__ part, int splits, int p, int q, int batch, int sym,
                                     double* __restrict__ C, long long ldc, long long sc) {
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long tot = (long long)batch * p * q;
  if (idx >= tot) return;
  const int b = (int)(idx / ((long long)p * q));
  const int rem = (int)(idx % ((long long)p * q));
  const int a = rem / q, c = rem % q;
  const double* P = part + (size_t)b * splits * p * q;
  double s = 0.0;
  for (int k = 0; k < splits; ++k) s += P[(size_t)k * p * q + rem];
  if (sym) {
    double t = 0.0;
    for (int k = 0; k < splits; ++k) t += P[(size_t)k * p * q + (size_t)c * q + a];
    s = 0.5 * (s + t);
  }
  C[(size_t)b * sc + (size_t)a * ldc + c] = s;
}

tsk_status gemm_tn_f64(Ctx* ctx, const double* X, long long ldx, long long sx, const double* Y, long long ldy,
                       long long sy, int m, int p, int q, int batch, double* C, long long ldc, long long sc, int sym,
                       int ws_id) {
  const int tiles = ((p + 31) / 32) * ((q + 31) / 32) * batch;
  int splits = std::max(1, std::min((ctx->num_sms * 2 + tiles - 1) / tiles, std::max(1, m / 64)));
  double* part = reinterpret_cast<double*>(ctx->workspace(ws_id, (size_t)batch * splits * p * q * sizeof(double)));
  if (!part) return TSK_ENOMEM;
  dim3 grid((q + 31) / 32, (p + 31) / 32, batch * splits);
  gemm_tn_f64_kernel<<<grid, 256, 0, ctx->stream>>>(X, ldx, sx, Y, ldy, sy, m, p, q, splits, part);
  const long long tot = (long long)batch * p * q;
  reduce_splits_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, ctx->stream>>>(part, splits, p, q, batch, sym, C, ldc,
                                                                                 sc);
  ctx->count_launch(2);
  return cudaPeekAtLastError() == cudaSuccess ? TSK_OK : TSK_ECUDA;
}

// ---------------------------------------------------------------- Y = alpha * Z W, optional column scale
// Z: [batch][m][p] (ldz), W: [batch][p][q] (ldw, stride sw; sw = 0 broadcasts one W), Y: [batch][m][q]
__global__ void gemm_nn_f64_kernel(const double* __restrict__ Z, long long ldz, long long sz,
                                   const double* __restrict__ W, long long ldw, long long sw, int m, int p, int q,
                                   const double* __restrict__ colscale, double* __restrict__ Y, long long ldy,
                                   long long sy) {
  __shared__ double Zs[64][33];
  __shared__ double Ws[32][33];
  const int b = blockIdx.z;
  const int i0 = blockIdx.y * 64, c0 = blockIdx.x * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 256 threads: ty 0..7 -> 8 rows each
  const double* Zb = Z + (size_t)b * sz;
  const double* Wb = W + (size_t)b * sw;
  double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  for (int a0 = 0; a0 < p; a0 += 32) {
    for (int e = threadIdx.x; e < 64 * 32; e += 256) {
      const int ii = e >> 5, aa = e & 31;
      Zs[ii][aa] = (i0 + ii < m && a0 + aa < p) ? Zb[(size_t)(i0 + ii) * ldz + a0 + aa] : 0.0;
    }
    for (int e = threadIdx.x; e < 32 * 32; e += 256) {
      const int aa = e >> 5, cc = e & 31;
      Ws[aa][cc] = (a0 + aa < p && c0 + cc < q) ? Wb[(size_t)(a0 + aa) * ldw + c0 + cc] : 0.0;
    }
    __syncthreads();
#pragma unroll 4
    for (int aa = 0; aa < 32; ++aa) {
      const double w = Ws[aa][tx];
#pragma unroll
      for (int u = 0; u < 8; ++u) acc[u] += Zs[ty * 8 + u][aa] * w;
    }
    __syncthreads();
  }
  const int c = c0 + tx;
  if (c < q) {
    const double s = colscale ? colscale[(size_t)b * q + c] : 1.0;
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int i = i0 + ty * 8 + u;
      if (i < m) Y[(size_t)b * sy + (size_t)i * ldy + c] = acc[u] * s;
    }
  }
}

tsk_status gemm_nn_f64(Ctx* ctx, const double* Z, long long ldz, long long sz, const double* W, long long ldw,
                       long long sw, int m, int p, int q, int batch, const double* colscale, double* Y, long long ldy,
                       long long sy) {
  dim3 grid((q + 31) / 32, (m + 63) / 64, batch);
  gemm_nn_f64_kernel<<<grid, 256, 0, ctx->stream>>>(Z, ldz, sz, W, ldw, sw, m, p, q, colscale, Y, ldy, sy);
  ctx->count_launch();
  return cudaPeekAtLastError() == cudaSuccess ? TSK_OK : TSK_ECUDA;
}

// ---------------------------------------------------------------- Cholesky C = L L^T
// One CTA of 256 threads per matrix, factor in shared memory (global scratch if too large).
// Right-looking: p dependent steps; the trailing update of step j is spread over all threads
// as a flat list of lower-triangle entries.  L: [batch][p][p] lower (row-major, upper = 0).
// On failure flag[b] = index+1 of the first pivot <= rel_tol * max diag (untouched on success:
// the caller clears it); the factorisation continues with a benign pivot, the caller repairs.
constexpr int kCholThreads = 256;
__global__ void __launch_bounds__(kCholThreads) chol_kernel(const double* __restrict__ C, int p, double rel_tol,
                                                            double* __restrict__ L, int* __restrict__ flag,
                                                            double* __restrict__ gscratch, int use_smem) {
  extern __shared__ double csm[];
  __shared__ double dmax;
  __shared__ int fail;
  const int b = blockIdx.x;
  const int tid = threadIdx.x;
  double* Lm = use_smem ? csm : gscratch + (size_t)b * p * p;
  const double* Cb = C + (size_t)b * p * p;
  copy_to_shared(Lm, Cb, p * p, tid, kCholThreads);
  if (tid == 0) {
    double d = 0;
    for (int i = 0; i < p; ++i) d = fmax(d, Cb[(size_t)i * p + i]);
    dmax = d;
    fail = 0;
  }
  __syncthreads();
  for (int j = 0; j < p; ++j) {
    double d = Lm[(size_t)j * p + j];
    if (!(d > rel_tol * dmax)) {
      if (tid == 0 && fail == 0) fail = j + 1;
      d = fmax(dmax, 1e-300);
    }
    const double inv = rsqrt(d);
    for (int i = j + 1 + tid; i < p; i += kCholThreads) Lm[(size_t)i * p + j] *= inv;
    __syncthreads();
    if (tid == 0) Lm[(size_t)j * p + j] = d * inv;
    // trailing lower triangle (i >= l > j): 16 x 16 thread grid, rows strided by 16, cols by 16
    {
      const int ty = tid >> 4, tx = tid & 15;
      for (int i = j + 1 + ty; i < p; i += 16) {
        const double lij = Lm[(size_t)i * p + j];
        double* row = Lm + (size_t)i * p;
        for (int l = j + 1 + tx; l <= i; l += 16) row[l] -= lij * Lm[(size_t)l * p + j];
      }
    }
    __syncthreads();
  }
  double* Lb = L + (size_t)b * p * p;
  for (int e = tid; e < p * p; e += kCholThreads) {
    const int i = e / p, l = e % p;
    Lb[e] = (l <= i) ? Lm[e] : 0.0;
  }
  if (tid == 0 && fail) flag[b] = fail;
}

// ---------------------------------------------------------------- Q = Y L^{-T}  (row-parallel)
// Each thread solves q L^T = y for one row of Y (forward substitution over columns), with L in
// shared memory (all threads read the same L entry at the same time: broadcast) and its own
// q row in a padded shared-memory slot.
__global__ void trsm_rlt_kernel(const double* __restrict__ Y, const double* __restrict__ L, int m, int p,
                                int rows_per_block, double* __restrict__ Q) {
  extern __shared__ double tsm[];
  double* Ls = tsm;                         // [p][p]
  const int ld = p | 1;                     // odd stride in doubles for the per-thread rows
  double* qs = tsm + (size_t)p * p;         // [rows_per_block][ld]
  copy_to_shared(Ls, L, p * p, threadIdx.x, blockDim.x);
  __syncthreads();
  const int row = blockIdx.x * rows_per_block + threadIdx.x;
  if (threadIdx.x >= rows_per_block || row >= m) return;
  double* q = qs + (size_t)threadIdx.x * ld;
  const double* y = Y + (size_t)row * p;
  for (int c = 0; c < p; ++c) {
    const double* Lc = Ls + (size_t)c * p;
    double s0 = y[c], s1 = 0.0, s2 = 0.0, s3 = 0.0;
    int a = 0;
    for (; a + 3 < c; a += 4) {
      s0 -= q[a] * Lc[a];
      s1 -= q[a + 1] * Lc[a + 1];
      s2 -= q[a + 2] * Lc[a + 2];
      s3 -= q[a + 3] * Lc[a + 3];
    }
    for (; a < c; ++a) s0 -= q[a] * Lc[a];
    q[c] = ((s0 + s1) + (s2 + s3)) / Lc[c];
  }
  double* out = Q + (size_t)row * p;
  for (int c = 0; c < p; ++c) out[c] = q[c];
}

// ---------------------------------------------------------------- Cholesky + inverse: Rinv = L^{-T}
// One CTA (256 threads, 16 x 16 grid) per matrix; C and the factor live in shared memory.
// Factorisation: right-looking with the column scaling deferred (step j updates the trailing
// triangle with L_ij L_lj / d_j from the unscaled column j).  Inverse: forward elimination of
// [L | I] row by row.  The column (row) consumed by each step is first copied into a separate
// static shared array, so the compiler can prove the update's stores do not alias its operands.
// Output Rinv[a][c] = Linv[c][a] (upper triangular): Q = Y Rinv has orthonormal columns when
// C = Y^T Y.  flag as in chol_kernel.
__global__ void __launch_bounds__(256) chol_inv2_kernel(const double* __restrict__ C, int p, double rel_tol,
                                                        double* __restrict__ Rinv, int* __restrict__ flag) {
  extern __shared__ double sm2[];
  const int ld = p | 1;
  double* Lm = sm2;                      // [p][ld]
  double* X = sm2 + (size_t)p * ld;      // [p][ld]  L^{-1}
  __shared__ double dmax;
  __shared__ int fail;
  __shared__ double colj[128];
  const int b = blockIdx.x, tid = threadIdx.x, ty = tid >> 4, tx = tid & 15;
  const double* Cb = C + (size_t)b * p * p;
  for (int e = tid; e < p * p; e += 256) {
    const int i = e / p, l = e - (e / p) * p;
    Lm[i * ld + l] = Cb[e];
    X[i * ld + l] = (i == l) ? 1.0 : 0.0;
  }
  if (tid == 0) {
    double d = 0;
    for (int i = 0; i < p; ++i) d = fmax(d, Cb[(size_t)i * p + i]);
    dmax = d;
    fail = 0;
  }
  __syncthreads();
  const double floor_piv = rel_tol * dmax;
  for (int j = 0; j < p; ++j) {
    double d = Lm[j * ld + j];
    if (!(d > floor_piv)) {
      if (tid == 0 && fail == 0) fail = j + 1;
      d = fmax(dmax, 1e-300);
      if (tid == 0) Lm[j * ld + j] = d;
    }
    const double inv_d = 1.0 / d;
    for (int i = j + 1 + tid; i < p; i += 256) colj[i] = Lm[i * ld + j];
    __syncthreads();
    for (int i = j + 1 + ty; i < p; i += 16) {
      const double f = colj[i] * inv_d;
      double* row = Lm + i * ld;
      for (int l = j + 1 + tx; l <= i; l += 16) row[l] -= f * colj[l];
    }
    __syncthreads();
  }
  // deferred scaling: L_ij = C'_ij / sqrt(d_j) for i > j, L_jj = sqrt(d_j)
  for (int e = tid; e < p * p; e += 256) {
    const int i = e / p, j = e - (e / p) * p;
    if (j < i) Lm[i * ld + j] *= rsqrt(Lm[j * ld + j]);
  }
  __syncthreads();
  for (int j = tid; j < p; j += 256) Lm[j * ld + j] = sqrt(Lm[j * ld + j]);
  __syncthreads();
  // forward elimination: row j of X scaled by 1/L_jj, then X[i,:] -= L_ij X[j,:] for i > j
  for (int j = 0; j < p; ++j) {
    const double ljj = Lm[j * ld + j];
    for (int c = tid; c <= j; c += 256) {
      const double v = X[j * ld + c] / ljj;
      X[j * ld + c] = v;
      colj[c] = v;
    }
    __syncthreads();
    for (int i = j + 1 + ty; i < p; i += 16) {
      const double lij = Lm[i * ld + j];
      double* row = X + i * ld;
      for (int c = tx; c <= j; c += 16) row[c] -= lij * colj[c];
    }
    __syncthreads();
  }
  double* Rb = Rinv + (size_t)b * p * p;
  for (int e = tid; e < p * p; e += 256) {
    const int a = e / p, c = e - (e / p) * p;
    Rb[e] = X[c * ld + a];
  }
  if (tid == 0 && fail) flag[b] = fail;
}

tsk_status chol_inv2(Ctx* ctx, const double* C, int p, int batch, double rel_tol, double* Rinv, int* flag) {
  const size_t smem = (size_t)2 * p * (p | 1) * sizeof(double);
  if (smem > 220 * 1024 || p > 128) return TSK_EINVAL;
  static uint64_t attr = 0;
  if (!(attr & device_bit())) {
    if (cudaFuncSetAttribute(chol_inv2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024) != cudaSuccess)
      return TSK_ECUDA;
    attr |= device_bit();
  }
  chol_inv2_kernel<<<batch, 256, smem, ctx->stream>>>(C, p, rel_tol, Rinv, flag);
  ctx->count_launch();
  return cudaPeekAtLastError() == cudaSuccess ? TSK_OK : TSK_ECUDA;
}

tsk_status chol(Ctx* ctx, const double* C, int p, int batch, double rel_tol, double* L, int* flag, int ws_id) {
  const size_t need = (size_t)p * p * sizeof(double);
  const int use_smem = need <= 200 * 1024;
  double* scratch = nullptr;
  if (!use_smem) {
    scratch = reinterpret_cast<double*>(ctx->workspace(ws_id, need * batch));
    if (!scratch) return TSK_ENOMEM;
  }
  static uint64_t attr = 0;
  if (!(attr & device_bit())) {
    if (cudaFuncSetAttribute(chol_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024) != cudaSuccess ||
        cudaFuncSetAttribute(trsm_rlt_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024) != cudaSuccess)
      return TSK_ECUDA;
    attr |= device_bit();
  }
  chol_kernel<<<batch, kCholThreads, use_smem ? need : 0, ctx->stream>>>(C, p, rel_tol, L, flag, scratch, use_smem);
  ctx->count_launch();
  return cudaPeekAtLastError() == cudaSuccess ? TSK_OK : TSK_ECUDA;
}

tsk_status trsm_rlt(Ctx* ctx, const double* Y, const double* L, int m, int p, double* Q) {
  const size_t lbytes = (size_t)p * p * 8;
  const int ld = p | 1;
  if (lbytes + (size_t)32 * ld * 8 > 220 * 1024) return TSK_EINVAL;  // p <= ~150
  // one warp per block: the kernel is shared-memory-bandwidth bound per SM, so spread rows
  const int rows = 32;
  const size_t smem = lbytes + (size_t)rows * ld * 8;
  // 256 threads copy L into shared memory; the first `rows` of them then solve one row each
  trsm_rlt_kernel<<<(m + rows - 1) / rows, 256, smem, ctx->stream>>>(Y, L, m, p, rows, Q);
  ctx->count_launch();
  return cudaPeekAtLastError() == cudaSuccess ? TSK_OK : TSK_ECUDA;
}

}  // namespace tsk
