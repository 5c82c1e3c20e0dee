// Batched SCW (Algorithm 1) and per-matrix errors on the test stream.
//
// For each test matrix A_b (m x n) and sketch S (k x m):
//   1. B   = S A_b                        (k x n)   -- Alg. 1 line 1 operand, P:61, P:276;
//            tcgen05 3xTF32, A_b read transposed (gemm_tc.cu, xt)
//   2. V^T = orthonormal basis of rowspace(B) (k x n): fp64 Gram C = B B^T, pivoted Cholesky
//            P C P^T = L L^T, V^T = L^{-1} P B (pivots <= 1e-13 max diag dropped; reading c2).
//            "The full SVD in line 1 is used for orthogonalization ... it can be replaced with
//            QR" -- any orthonormal basis of the row space gives the same A_hat.
//   3. Z^T = (A_b V)^T                     (k x m)   -- tcgen05 3xTF32
//   4. Z^T Z = W2 diag(sigma^2) W2^T       (the SVD of AV, line 2, through its k x k Gram; Jacobi)
//   5. L = Z W2_r = U2_r diag(sigma_r) (m x r),  R = V W2_r (n x r)  =>  A_hat = [AV]_r V^T = L R^T
//   6. e_b = ||A_b - L R^T||_F             dense residual, fp64 reduction (not the identity
//            ||A||^2 - sum sigma^2, which cancels catastrophically)
// Small Grams, factorizations and rotations are fp64.  Everything is batched over b with
// deterministic (fixed-order) reductions.
#include <algorithm>
#include <cmath>

#include "ptx.cuh"
#include "tsk_internal.h"

namespace tsk {

// ---------------------------------------------------------------- fp64-coefficient combinations
// Out_b[c][j] (kVt) or Out_b[j][c] = sc_c sum_{a<k} W_b[a][c] In_b[a][j],  c < nout, j < len
// (kVt: V^T = L^{-1} P B with sc from mu; else the factors L = Z W_r, R = V W_r with sc = 1).
// Thread per two columns j: the 2 x 16 fp64 accumulators of a 16-wide block of outputs take the
// coefficients from shared memory as broadcast double2 reads (row pitch ldn = nout rounded up to
// even, 16 doubles of slack after the last row for the over-read of a partial block).
template <int KMAX, bool kVt>
__global__ void __launch_bounds__(128) scw_combine_kernel(const float* __restrict__ In, const double* __restrict__ W,
                                                          const double* __restrict__ mu, int k, int len, int nout,
                                                          int ldw, long long wst, float* __restrict__ Out, int ldo) {
  extern __shared__ double wsm[];  // [k][ldn] coefficients, 16 slack, then [nout] scales
  const int b = blockIdx.y;
  const int ldn = (nout + 1) & ~1;
  const double* Wb = W + (size_t)b * wst;
  for (int e = threadIdx.x; e < k * nout; e += blockDim.x)
    wsm[(size_t)(e / nout) * ldn + (e % nout)] = Wb[(size_t)(e / nout) * ldw + (e % nout)];
  double* sc = wsm + (size_t)k * ldn + 16;
  for (int c = threadIdx.x; c < nout; c += blockDim.x) {
    if (kVt) {
      const double m0 = mu[(size_t)b * k];
      const double mc = mu[(size_t)b * k + c];
      sc[c] = (mc > 0.0 && mc > 1e-13 * m0) ? 1.0 / sqrt(mc) : 0.0;
    } else {
      sc[c] = 1.0;
    }
  }
  __syncthreads();
  // two columns per thread (j0, j0 + blockDim.x): every coefficient pair read from shared memory
  // (one double2, a broadcast) feeds 4 DFMA -- one coefficient per DFMA made the kernel
  // shared-memory-issue bound at half the fp64 rate
  const int j0 = blockIdx.x * 2 * blockDim.x + threadIdx.x, j1 = j0 + blockDim.x;
  if (j0 >= len) return;
  const bool has1 = j1 < len;
  const float* Ib = In + (size_t)b * k * len;
  float* Ob = Out + (size_t)b * (kVt ? (size_t)nout * len : (size_t)len * ldo);
  for (int c0 = 0; c0 < nout; c0 += 16) {
    double s0[16], s1[16];
#pragma unroll
    for (int q = 0; q < 16; ++q) s0[q] = s1[q] = 0.0;
#pragma unroll 4
    for (int a = 0; a < KMAX; ++a) {
      if (a < k) {
        const double x0 = (double)Ib[(size_t)a * len + j0];
        const double x1 = has1 ? (double)Ib[(size_t)a * len + j1] : 0.0;
        const double2* wr = reinterpret_cast<const double2*>(wsm + (size_t)a * ldn + c0);
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const double2 w = wr[q];
          s0[2 * q] = fma(w.x, x0, s0[2 * q]);
          s0[2 * q + 1] = fma(w.y, x0, s0[2 * q + 1]);
          s1[2 * q] = fma(w.x, x1, s1[2 * q]);
          s1[2 * q + 1] = fma(w.y, x1, s1[2 * q + 1]);
        }
      }
    }
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      const int c = c0 + q;
      if (c < nout) {
        const float v0 = (float)(s0[q] * sc[c]);
        const float v1 = (float)(s1[q] * sc[c]);
        if (kVt) {
          Ob[(size_t)c * len + j0] = v0;
          if (has1) Ob[(size_t)c * len + j1] = v1;
        } else {
          Ob[(size_t)j0 * ldo + c] = v0;
          if (has1) Ob[(size_t)j1 * ldo + c] = v1;
        }
      }
    }
  }
}

// Tiled version (round 2): the CTA computes CT outputs c x 64 columns j of one matrix with the inputs
// staged through shared memory 16 rows a at a time (fp32 -> fp64 on the way in); thread (cg, jg) owns
// c = c0 + cg + (CT/4) u and j = j0 + jg + 16 v (u, v < 4): conflict-free / broadcast shared reads,
// coalesced global loads and (kVt) stores.  The one-column-pair-per-thread kernel above re-read its
// inputs from global memory once per 16 outputs (latency-bound, ~25 % of the fp64 rate).
template <int CT, bool kVt>
__global__ void __launch_bounds__(CT * 4) scw_combine2_kernel(const float* __restrict__ In,
                                                              const double* __restrict__ W,
                                                              const double* __restrict__ mu, int k, int len,
                                                              int nout, int ldw, long long wst,
                                                              float* __restrict__ Out, int ldo,
                                                              const int* __restrict__ only) {
  constexpr int JT = 64, KC = 16, CG = CT / 4;
  if (only && only[blockIdx.z] == 0) return;  // error-only path: factors of the dense-marked matrices only
  __shared__ double Ws[KC][CT + 1];
  __shared__ double Is[KC][JT + 1];
  __shared__ double sc[CT];
  const int b = blockIdx.z, j0 = blockIdx.x * JT, c0 = blockIdx.y * CT;
  const int tid = threadIdx.x, nt = blockDim.x;
  const int cg = tid >> 4, jg = tid & 15;
  const double* Wb = W + (size_t)b * wst;
  const float* Ib = In + (size_t)b * k * len;
  for (int c = tid; c < CT; c += nt) {
    double v = 1.0;
    if (kVt && c0 + c < nout) {
      const double m0 = mu[(size_t)b * k];
      const double mc = mu[(size_t)b * k + c0 + c];
      v = (mc > 0.0 && mc > 1e-13 * m0) ? 1.0 / sqrt(mc) : 0.0;
    }
    sc[c] = v;
  }
  double acc[4][4];
#pragma unroll
  for (int u = 0; u < 4; ++u)
#pragma unroll
    for (int v = 0; v < 4; ++v) acc[u][v] = 0.0;
  for (int a0 = 0; a0 < k; a0 += KC) {
    for (int e = tid; e < KC * CT; e += nt) {
      const int kk = e / CT, cc = e % CT;
      Ws[kk][cc] = (a0 + kk < k && c0 + cc < nout) ? Wb[(size_t)(a0 + kk) * ldw + c0 + cc] : 0.0;
    }
    for (int e = tid; e < KC * JT; e += nt) {
      const int kk = e / JT, jj = e % JT;
      Is[kk][jj] = (a0 + kk < k && j0 + jj < len) ? (double)Ib[(size_t)(a0 + kk) * len + j0 + jj] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < KC; ++kk) {
      double w[4], x[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) w[u] = Ws[kk][cg + CG * u];
#pragma unroll
      for (int v = 0; v < 4; ++v) x[v] = Is[kk][jg + 16 * v];
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) acc[u][v] = fma(w[u], x[v], acc[u][v]);
    }
    __syncthreads();
  }
  float* Ob = Out + (size_t)b * (kVt ? (size_t)nout * len : (size_t)len * ldo);
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int c = c0 + cg + CG * u;
    if (c >= nout) continue;
    const double scl = sc[cg + CG * u];
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      const int j = j0 + jg + 16 * v;
      if (j >= len) continue;
      if (kVt) Ob[(size_t)c * len + j] = (float)(acc[u][v] * scl);
      else Ob[(size_t)j * ldo + c] = (float)(acc[u][v] * scl);
    }
  }
}

// Out = combination of the k rows of In by W (see scw_combine_kernel), tiled over (64 columns, CT outputs);
// only (optional, [batch]): matrices with only[b] == 0 are skipped
template <bool kVt>
static void launch_combine2(const float* In, const double* W, const double* mu, int k, int len, int nout, int ldw,
                            long long wst, float* Out, int ldo, int batch, cudaStream_t s,
                            const int* only = nullptr) {
  if (nout <= 32)
    scw_combine2_kernel<32, kVt><<<dim3((len + 63) / 64, 1, batch), 128, 0, s>>>(In, W, mu, k, len, nout, ldw, wst,
                                                                                 Out, ldo, only);
  else
    scw_combine2_kernel<64, kVt><<<dim3((len + 63) / 64, (nout + 63) / 64, batch), 256, 0, s>>>(
        In, W, mu, k, len, nout, ldw, wst, Out, ldo, only);
}

// V^T = sc (W^T B) for k <= 64 on the fp64 tensor cores (round 2): V^T[c][j] = sc_c sum_a W[a][c] B[a][j], one CTA
// per (matrix, 128 columns j), 4 warps; W^T is staged once per CTA (rows c, pitch 68: conflict-free A
// fragments), B streamed 32 columns at a time as fp64 (pitch 44: conflict-free B fragments); warp w owns
// the output rows 16 w .. 16 w + 15 (two m8 tiles) x the 4 n8 tiles of a 32-column block, 2 x 4 DMMA
// (mma.sync m8n8k4 f64) per k4 step.  The DFMA tile kernel above reached ~33 % of the fp64 rate here
// (287 us per 250 C4 matrices).
constexpr int kVtCols = 128, kVtBlk = 32, kVtWP = 68, kVtBP = 44;
constexpr size_t kVtSmem = (size_t)64 * (kVtWP + kVtBP) * sizeof(double);
__global__ void __launch_bounds__(128) scw_vt_dmma_kernel(const float* __restrict__ In, const double* __restrict__ W,
                                                          const double* __restrict__ mu, int k, int len, long long wst,
                                                          float* __restrict__ Out) {
  extern __shared__ __align__(16) double vt_sm[];
  double (*Wt)[kVtWP] = reinterpret_cast<double (*)[kVtWP]>(vt_sm);             // [64][kVtWP]
  double (*Bs)[kVtBP] = reinterpret_cast<double (*)[kVtBP]>(vt_sm + 64 * kVtWP);  // [64][kVtBP]
  __shared__ double sc[64];
  const int b = blockIdx.y, jbase = blockIdx.x * kVtCols;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const double* Wb = W + (size_t)b * wst;
  const float* Ib = In + (size_t)b * k * len;
  float* Ob = Out + (size_t)b * k * len;
  const int kp = (k + 3) & ~3;  // K padded to the k4 step (zero rows / columns)
  for (int e = tid; e < 64 * 64; e += 128) {
    const int c = e >> 6, a = e & 63;  // Wt[c][a] = W[a][c]
    Wt[c][a] = (c < k && a < k) ? Wb[(size_t)a * k + c] : 0.0;
  }
  for (int c = tid; c < 64; c += 128) {
    double v = 0.0;
    if (c < k) {
      const double m0 = mu[(size_t)b * k], mc = mu[(size_t)b * k + c];
      v = (mc > 0.0 && mc > 1e-13 * m0) ? 1.0 / sqrt(mc) : 0.0;
    }
    sc[c] = v;
  }
  const int fr = lane >> 2, fk = lane & 3;
  // the next 32-column block of B is loaded into registers while the current one is multiplied
  constexpr int kPre = 64 * kVtBlk / 128;  // 16 floats per thread
  float pre[kPre];
  auto fetch = [&](int j0) {
#pragma unroll
    for (int t = 0; t < kPre; ++t) {
      const int e = tid + t * 128, a = e >> 5, jj = e & 31;
      pre[t] = (a < k && j0 + jj < len) ? __ldg(Ib + (size_t)a * len + j0 + jj) : 0.0f;
    }
  };
  const int jend = min(jbase + kVtCols, len);
  fetch(jbase);
  for (int j0 = jbase; j0 < jend; j0 += kVtBlk) {
    __syncthreads();  // Wt / sc staged; the previous block's Bs consumed
#pragma unroll
    for (int t = 0; t < kPre; ++t) {
      const int e = tid + t * 128;
      Bs[e >> 5][e & 31] = (double)pre[t];
    }
    __syncthreads();
    if (j0 + kVtBlk < jend) fetch(j0 + kVtBlk);
    double acc[2][4][2];
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) acc[mt][nt][0] = acc[mt][nt][1] = 0.0;
    const int r0 = 16 * w;
#pragma unroll 4
    for (int a0 = 0; a0 < kp; a0 += 4) {
      const double x0 = Wt[r0 + fr][a0 + fk], x1 = Wt[r0 + 8 + fr][a0 + fk];
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) {
        const double y = Bs[a0 + fk][8 * nt + fr];
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(acc[0][nt][0]), "+d"(acc[0][nt][1]) : "d"(x0), "d"(y));
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(acc[1][nt][0]), "+d"(acc[1][nt][1]) : "d"(x1), "d"(y));
      }
    }
#pragma unroll
    for (int mt = 0; mt < 2; ++mt) {
      const int c = r0 + 8 * mt + fr;
      if (c >= k) continue;
      const double scl = sc[c];
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) {
        const int j = j0 + 8 * nt + 2 * fk;
        if (j + 1 < len) {
          *reinterpret_cast<float2*>(Ob + (size_t)c * len + j) =
              make_float2((float)(acc[mt][nt][0] * scl), (float)(acc[mt][nt][1] * scl));
        } else if (j < len) {
          Ob[(size_t)c * len + j] = (float)(acc[mt][nt][0] * scl);
        }
      }
    }
  }
}

static inline size_t combine_smem(int k, int nout) {
  return ((size_t)k * ((nout + 1) & ~1) + 16 + nout) * sizeof(double);
}

__global__ void scw_sigma_kernel(const double* __restrict__ sig2, int k, int r, long long B, float* __restrict__ sigma) {
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= B * r) return;
  const long long b = idx / r;
  const int c = (int)(idx % r);
  sigma[idx] = (float)sqrt(fmax(sig2[b * k + c], 0.0));
}

// err[b] = sqrt(sum of the b-th matrix's residual partials): one warp per matrix, lanes strided, fixed-
// order butterfly (deterministic)
// (only: matrices with only[b] == 0 keep their error -- they were not part of the residual launch)
__global__ void scw_err_reduce_kernel(const double* __restrict__ part, int tiles, long long B, double* __restrict__ err,
                                      const int* __restrict__ only) {
  const long long b = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (b >= B) return;
  if (only && only[b] == 0) return;
  double s = 0.0;
  for (int t = lane; t < tiles; t += 32) s += part[b * tiles + t];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) err[b] = sqrt(s);
}

// err_b by the Pythagorean identity (reading c17): Algorithm 1's A_hat = [AV]_r V^T
// is A P with P = (V W_r)(V W_r)^T an orthogonal projector (V orthonormal, W_r the top-r
// eigenvectors of (AV)^T AV), so ||A - A_hat||_F^2 = ||A||_F^2 - ||A V W_r||_F^2 = ||A||_F^2 -
// sum_{i<r} sigma_i^2.  ||A||_F^2 comes from the SA product's transform warps (sq partials, fp64, fixed
// order), sigma_i^2 are the eigenvalues of (AV)^T AV.  The subtraction cancels when the error is small
// against ||A||: below tau ||A||^2 (or a non-finite value) the matrix is marked for the dense residual
// ||A - L R^T|| (dense[b] = 1), which then overwrites err[b].  One warp per matrix, fixed-order sums.
// ndense (zeroed by the caller) counts the marked matrices: the residual launch exits at once when none is.
__global__ void scw_err_pyth_kernel(const double* __restrict__ sq, int per, const double* __restrict__ sig2, int k,
                                    int r, long long B, double tau, double* __restrict__ err, int* __restrict__ dense,
                                    int* __restrict__ ndense) {
  const long long b = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (b >= B) return;
  double s = 0.0;
  for (int t = lane; t < per; t += 32) s += sq[b * per + t];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) {
    double kept = 0.0;
    for (int i = 0; i < r; ++i) kept += fmax(sig2[b * k + i], 0.0);
    const double e2 = s - kept;
    const bool need = !(e2 >= tau * s) || !(s < INFINITY);
    err[b] = need ? 0.0 : sqrt(e2);
    dense[b] = need ? 1 : 0;
    if (need) atomicAdd(ndense, 1);
  }
}

// ---------------------------------------------------------------- C = X X^T, register-tiled fp64
// grid (tiles^2, batch): CTA (ta, tc) computes the 64 x 64 block rows [64 ta, +64) x cols [64 tc, +64)
// of C[b] (k <= 128) for X_b fp32 [k][len]; 256 threads = 16 x 16, thread (ty, tx) owns rows
// ty + 16 i and cols tx + 16 j (i, j < 4: conflict-free / broadcast shared reads).  X chunks of 32
// columns are read row-contiguously (one 128-B line per warp load) and converted to fp64 on their
// way into shared memory (exact), stored transposed with an odd pitch; products accumulate in fp64.
// cross form (X2 != nullptr): C[b] = X_b X2_b^T (k x k2, no mirroring)
__global__ void __launch_bounds__(256) gram_rows_tiled_kernel(const float* __restrict__ X, int k, int len,
                                                              double* __restrict__ C, const float* __restrict__ X2,
                                                              int k2) {
  constexpr int KC = 32;
  constexpr int P = 65;
  __shared__ double xa[KC][P];
  __shared__ double xc[KC][P];
  const int b = blockIdx.y;
  const bool cross = X2 != nullptr;
  const int kc = cross ? k2 : k;
  const int ntc = (kc + 63) / 64;
  const int ta = blockIdx.x / ntc, tc = blockIdx.x % ntc;
  if (!cross && tc > ta) return;  // upper blocks are mirrored from the lower ones
  const float* Xb = X + (size_t)b * k * len;
  const float* Xc = cross ? X2 + (size_t)b * k2 * len : Xb;
  const int tid = threadIdx.x, ty = tid >> 4, tx = tid & 15;
  const int lane = tid & 31, wrow = tid >> 5;  // fill: warp w reads rows w, w + 8, ... (32 columns each)
  double acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;
  for (int j0 = 0; j0 < len; j0 += KC) {
    const bool inj = j0 + lane < len;
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      const int r = wrow + 8 * t;
      const int ra = ta * 64 + r, rc = tc * 64 + r;
      xa[lane][r] = (ra < k && inj) ? (double)Xb[(size_t)ra * len + j0 + lane] : 0.0;
      xc[lane][r] = (rc < kc && inj) ? (double)Xc[(size_t)rc * len + j0 + lane] : 0.0;
    }
    __syncthreads();
#pragma unroll 8
    for (int jj = 0; jj < KC; ++jj) {
      double av[4], cv[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) av[i] = xa[jj][ty + 16 * i];
#pragma unroll
      for (int j = 0; j < 4; ++j) cv[j] = xc[jj][tx + 16 * j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fma(av[i], cv[j], acc[i][j]);
    }
    __syncthreads();
  }
  double* Cb = C + (size_t)b * k * kc;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int ra = ta * 64 + ty + 16 * i;
    if (ra >= k) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int rc = tc * 64 + tx + 16 * j;
      if (rc >= kc) continue;
      Cb[(size_t)ra * kc + rc] = acc[i][j];
      if (!cross) Cb[(size_t)rc * k + ra] = acc[i][j];
    }
  }
}

// ---------------------------------------------------------------- C = X X^T for k <= 64 (round 2)
// The symmetric Gram of SCW's k x len row blocks (B = S A_b and (A_b V)^T): one 2-CTA cluster per matrix,
// each CTA one half of len; 136 threads own the 4 x 4 micro-tiles of the lower triangle of the padded
// 64 x 64 result (thread t -> micro-tile row ty >= column tx), reading two 16-byte pairs of the
// transposed fp64 chunk per K index for 16 DFMA -- half the products of the full 64 x 64 tile of
// gram_rows_tiled_kernel and 2 CTAs per matrix (500 CTAs at C4 instead of 250 on 148 SMs).  CTA 1 adds
// its partial into CTA 0's over DSMEM (fixed order: deterministic), CTA 0 writes both triangles.
constexpr int kGsThreads = 160, kGsKC = 32, kGsP = 66;  // 136 working threads; chunk pitch 66 doubles
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kGsThreads, 4)
    gram_rows_sym_kernel(const float* __restrict__ X, int k, int len, double* __restrict__ C) {
  __shared__ __align__(16) double xs[kGsKC][kGsP];
  __shared__ __align__(16) double part[136][16];
  const int b = blockIdx.x >> 1;
  const unsigned rank = cluster_ctarank();
  const int tid = threadIdx.x;
  // micro-tile of thread t: row block ty, column block tx <= ty (t = ty (ty + 1) / 2 + tx)
  int ty = (int)((sqrtf(8.0f * (float)tid + 1.0f) - 1.0f) * 0.5f);
  while (ty * (ty + 1) / 2 > tid) --ty;
  while ((ty + 1) * (ty + 2) / 2 <= tid) ++ty;
  const int tx = tid - ty * (ty + 1) / 2;
  const bool work = tid < 136;
  const int half = ((len + 2 * kGsKC - 1) / (2 * kGsKC)) * kGsKC;  // CTA 0: [0, half), CTA 1: [half, len)
  const int j0 = rank == 0 ? 0 : half, j1 = rank == 0 ? min(half, len) : len;
  const float* Xb = X + (size_t)b * k * len;
  double acc[4][4];
#pragma unroll
  for (int u = 0; u < 4; ++u)
#pragma unroll
    for (int v = 0; v < 4; ++v) acc[u][v] = 0.0;
  // fill: item e of a chunk = (column kk = e % 32, row group g = e / 32): four rows 4g .. 4g + 3 of one
  // column, read as four coalesced 128-B warp loads and stored as two 16-byte pairs of the transposed
  // chunk (a row-strided 8-byte transpose store was 4-way bank-conflicted: 40 % excess wavefronts)
  constexpr int kItems = 16 * kGsKC, kPer = (kItems + kGsThreads - 1) / kGsThreads;  // 512 items, 4 per thread
  // no register prefetch: the loads of one CTA overlap the products of the other three on its SM
  for (int jc = j0; jc < j1; jc += kGsKC) {
    __syncthreads();  // the previous chunk is consumed
#pragma unroll
    for (int t = 0; t < kPer; ++t) {
      const int e = tid + t * kGsThreads, kk = e & 31, g = e >> 5;
      if (e < kItems) {
        float v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int r = 4 * g + u;
          v[u] = (r < k && jc + kk < j1) ? __ldg(Xb + (size_t)r * len + jc + kk) : 0.0f;
        }
        *reinterpret_cast<double2*>(&xs[kk][4 * g]) = make_double2((double)v[0], (double)v[1]);
        *reinterpret_cast<double2*>(&xs[kk][4 * g + 2]) = make_double2((double)v[2], (double)v[3]);
      }
    }
    __syncthreads();
    if (work) {
#pragma unroll 8
      for (int kk = 0; kk < kGsKC; ++kk) {
        const double2 a01 = *reinterpret_cast<const double2*>(&xs[kk][4 * ty]);
        const double2 a23 = *reinterpret_cast<const double2*>(&xs[kk][4 * ty + 2]);
        const double2 c01 = *reinterpret_cast<const double2*>(&xs[kk][4 * tx]);
        const double2 c23 = *reinterpret_cast<const double2*>(&xs[kk][4 * tx + 2]);
        const double av[4] = {a01.x, a01.y, a23.x, a23.y}, cv[4] = {c01.x, c01.y, c23.x, c23.y};
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int v = 0; v < 4; ++v) acc[u][v] = fma(av[u], cv[v], acc[u][v]);
      }
    }
  }
  if (work && rank == 1) {
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int v = 0; v < 4; ++v) part[tid][u * 4 + v] = acc[u][v];
  }
  cluster_sync();
  if (work && rank == 0) {
    const uint32_t rp = mapa_shared(smem_u32(&part[tid][0]), 1);
    double* Cb = C + (size_t)b * k * k;
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        const int i = 4 * ty + u, j = 4 * tx + v;
        const double val = acc[u][v] + ld_dsmem_f64(rp + (uint32_t)(u * 4 + v) * 8u);
        if (i < k && j < k && j <= i) {
          Cb[(size_t)i * k + j] = val;
          Cb[(size_t)j * k + i] = val;
        }
      }
  }
  cluster_sync();  // CTA 1's partial stays readable until CTA 0 is done
}

// The same Gram on the fp64 tensor cores (DMMA m8n8k4, round 2): the 36 lower-triangle 8 x 8 tiles of the padded
// 64 x 64 result, 4 warps owning the tile rows {7, 0}, {6, 1}, {5, 2}, {4, 3} (9 tiles each); per k4 step a warp
// loads the <= 8 fragments v_t = X[8t .. 8t + 7][k .. k + 3] it needs (the A fragment of tile row t and the B
// fragment of tile column t are the same 8-byte pattern of the transposed chunk, pitch 68: conflict-free) and
// issues 9 DMMAs -- against 16 DFMA per 4 16-byte loads per thread for the register tiles above.  Same
// 2-CTA cluster split of len and DSMEM reduction.
constexpr int kGdThreads = 128, kGdKC = 32, kGdP = 68;
template <int MA>
__device__ __forceinline__ void gd_chunk(const double (*xs)[68], int fk, int fr, double (&acc)[9][2]) {
  constexpr int MB = 7 - MA;
#pragma unroll 2
  for (int k4 = 0; k4 < 32; k4 += 4) {
    double v[MA + 1];
#pragma unroll
    for (int t = 0; t <= MA; ++t) v[t] = xs[k4 + fk][8 * t + fr];
#pragma unroll
    for (int t = 0; t <= MA; ++t)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(acc[t][0]), "+d"(acc[t][1]) : "d"(v[MA]), "d"(v[t]));
#pragma unroll
    for (int t = 0; t <= MB; ++t)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(acc[MA + 1 + t][0]), "+d"(acc[MA + 1 + t][1]) : "d"(v[MB]), "d"(v[t]));
  }
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kGdThreads)
    gram_rows_dmma_kernel(const float* __restrict__ X, int k, int len, double* __restrict__ C) {
  __shared__ __align__(16) double xs[kGdKC][kGdP];
  __shared__ __align__(16) double part[4][9][2][32];
  const int b = blockIdx.x >> 1;
  const unsigned rank = cluster_ctarank();
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int fr = lane >> 2, fk = lane & 3;
  const int mA = 7 - w, mB = w;  // tile rows of this warp: mA + 1 + mB + 1 = 9 tiles
  const int half = ((len + 2 * kGdKC - 1) / (2 * kGdKC)) * kGdKC;
  const int j0 = rank == 0 ? 0 : half, j1 = rank == 0 ? min(half, len) : len;
  const float* Xb = X + (size_t)b * k * len;
  double acc[9][2];
#pragma unroll
  for (int t = 0; t < 9; ++t) acc[t][0] = acc[t][1] = 0.0;
  constexpr int kItems = 16 * kGdKC, kPer = kItems / kGdThreads;  // (column, 4-row group) items, 4 per thread
  for (int jc = j0; jc < j1; jc += kGdKC) {
    __syncthreads();
#pragma unroll
    for (int t = 0; t < kPer; ++t) {
      const int e = tid + t * kGdThreads, kk = e & 31, g = e >> 5;
      float v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int r = 4 * g + u;
        v[u] = (r < k && jc + kk < j1) ? __ldg(Xb + (size_t)r * len + jc + kk) : 0.0f;
      }
      *reinterpret_cast<double2*>(&xs[kk][4 * g]) = make_double2((double)v[0], (double)v[1]);
      *reinterpret_cast<double2*>(&xs[kk][4 * g + 2]) = make_double2((double)v[2], (double)v[3]);
    }
    __syncthreads();
    switch (w) {  // compile-time tile rows per warp (register-resident fragments and accumulators)
      case 0: gd_chunk<7>(xs, fk, fr, acc); break;
      case 1: gd_chunk<6>(xs, fk, fr, acc); break;
      case 2: gd_chunk<5>(xs, fk, fr, acc); break;
      default: gd_chunk<4>(xs, fk, fr, acc); break;
    }
  }
  if (rank == 1) {
#pragma unroll
    for (int t = 0; t < 9; ++t) {
      part[w][t][0][lane] = acc[t][0];
      part[w][t][1][lane] = acc[t][1];
    }
  }
  cluster_sync();
  if (rank == 0) {
    double* Cb = C + (size_t)b * k * k;
#pragma unroll
    for (int q = 0; q < 9; ++q) {  // tile q: (mA, q) for q <= mA, else (mB, q - mA - 1)
      const int mi = q <= mA ? mA : mB, t = q <= mA ? q : q - mA - 1;
      const int i = 8 * mi + fr;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int jj = 8 * t + 2 * fk + h;
        const double val = acc[q][h] + ld_dsmem_f64(mapa_shared(smem_u32(&part[w][q][h][lane]), 1));
        if (i < k && jj < k && jj <= i) {
          Cb[(size_t)i * k + jj] = val;
          Cb[(size_t)jj * k + i] = val;
        }
      }
    }
  }
  cluster_sync();
}

static void launch_gram_rows_tiled(const float* X, int k, int len, int batch, double* C, cudaStream_t s) {
  if (k <= 64 && batch > 0) {
    if (getenv("TSK_SCW_GRAM_DFMA"))
      gram_rows_sym_kernel<<<2 * batch, kGsThreads, 0, s>>>(X, k, len, C);
    else
      gram_rows_dmma_kernel<<<2 * batch, kGdThreads, 0, s>>>(X, k, len, C);
    return;
  }
  const int nt = (k + 63) / 64;
  gram_rows_tiled_kernel<<<dim3(nt * nt, batch), 256, 0, s>>>(X, k, len, C, nullptr, 0);
}

// C[b] = X_b X2_b^T (k x k2) for X [B][k][len], X2 [B][k2][len] fp32, fp64 products
static void launch_gram_cross(const float* X, int k, const float* X2, int k2, int len, int batch, double* C,
                              cudaStream_t s) {
  gram_rows_tiled_kernel<<<dim3(((k + 63) / 64) * ((k2 + 63) / 64), batch), 256, 0, s>>>(X, k, len, C, X2, k2);
}

// H[b] = M_b^T M_b for M [B][l][k] fp64 (one CTA per matrix, thread per entry of the lower triangle)
__global__ void gram_cols_f64_kernel(const double* __restrict__ M, int l, int k, double* __restrict__ H) {
  const int b = blockIdx.x;
  const double* Mb = M + (size_t)b * l * k;
  double* Hb = H + (size_t)b * k * k;
  for (int e = threadIdx.x; e < k * k; e += blockDim.x) {
    const int i = e / k, j = e % k;
    if (j > i) continue;
    double s = 0.0;
    for (int a = 0; a < l; ++a) s += Mb[(size_t)a * k + i] * Mb[(size_t)a * k + j];
    Hb[(size_t)i * k + j] = s;
    Hb[(size_t)j * k + i] = s;
  }
}

// C[b] = M_b W_b[:, :r] for M [B][l][k], W [B][k][k] (columns = eigenvectors) -> C [B][l][r]
__global__ void small_mm_f64_kernel(const double* __restrict__ M, const double* __restrict__ W, int l, int k, int r,
                                    double* __restrict__ C) {
  const int b = blockIdx.x;
  const double* Mb = M + (size_t)b * l * k;
  const double* Wb = W + (size_t)b * k * k;
  double* Cb = C + (size_t)b * l * r;
  for (int e = threadIdx.x; e < l * r; e += blockDim.x) {
    const int a = e / r, c = e % r;
    double s = 0.0;
    for (int x = 0; x < k; ++x) s += Mb[(size_t)a * k + x] * Wb[(size_t)x * k + c];
    Cb[(size_t)a * r + c] = s;
  }
}

constexpr int kCholSmemMax = 220 * 1024;  // dynamic part (the kernel also has ~0.5 KB static)

// ---------------------------------------------------------------- orthonormal basis by pivoted Cholesky
// Algorithm 1 line 1 needs only an orthonormal basis of rowspace(S A) ("used for
// orthogonalization ... can be replaced with QR").  With C = B B^T (fp64) and the pivoted
// Cholesky P C P^T = L L^T, V^T = L^{-1} P B has orthonormal rows spanning rowspace(B).  Pivots
// below 1e-13 of the largest diagonal end the factorisation (rank(B) < k, reading c2): the
// remaining directions are dropped (mu = 0).  Output in the convention of scw_vt_kernel:
// V^T[c] = sc_c sum_a W[a][c] B[a] with W[perm[i]][c] = L^{-1}[c][i], mu[c] = 1 (kept) or 0.
__global__ void __launch_bounds__(128) chol_basis_kernel(const double* __restrict__ Cg, int k,
                                                         double* __restrict__ W, double* __restrict__ mu) {
  extern __shared__ double cs[];  // [k][k+1] C -> L (lower), then [k][k+1] L^{-1}
  __shared__ int perm[128];
  __shared__ int piv_s, rank_s;
  __shared__ double dmax0_s;
  const int b = blockIdx.x, tid = threadIdx.x, nt = blockDim.x;
  const int ld = k + 1;
  double* L = cs;
  double* Li = cs + (size_t)k * ld;
  const double* Cb = Cg + (size_t)b * k * k;
  for (int e = tid; e < k * k; e += nt) L[(e / k) * ld + e % k] = Cb[e];
  for (int i = tid; i < k; i += nt) perm[i] = i;
  __syncthreads();
  if (tid == 0) {
    double d = 0.0;
    for (int i = 0; i < k; ++i) d = fmax(d, L[i * ld + i]);
    dmax0_s = d;
    rank_s = k;
  }
  __syncthreads();
  const double floor_piv = 1e-13 * dmax0_s;
  for (int j = 0; j < k; ++j) {
    if (tid < 32) {  // pivot: largest remaining diagonal (ties -> lowest index)
      double best = -1.0;
      int bi = j;
      for (int i = j + tid; i < k; i += 32) {
        const double d = L[i * ld + i];
        if (d > best) { best = d; bi = i; }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double ob = __shfl_xor_sync(0xffffffffu, best, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
      }
      if (tid == 0) {
        piv_s = bi;
        if (!(best > floor_piv)) rank_s = j;
      }
    }
    __syncthreads();
    if (rank_s == j) break;
    const int p = piv_s;
    if (p != j) {  // symmetric swap of rows / columns j and p (full matrix kept)
      for (int x = tid; x < k; x += nt) {
        const double t = L[j * ld + x];
        L[j * ld + x] = L[p * ld + x];
        L[p * ld + x] = t;
      }
      __syncthreads();
      for (int x = tid; x < k; x += nt) {
        const double t = L[x * ld + j];
        L[x * ld + j] = L[x * ld + p];
        L[x * ld + p] = t;
      }
      if (tid == 0) {
        const int t = perm[j];
        perm[j] = perm[p];
        perm[p] = t;
      }
      __syncthreads();
    }
    const double d = sqrt(L[j * ld + j]);
    __syncthreads();
    for (int i = j + 1 + tid; i < k; i += nt) L[i * ld + j] /= d;
    if (tid == 0) L[j * ld + j] = d;
    __syncthreads();
    // trailing update of the lower triangle (and the diagonal) of rows / cols > j
    const int rem = k - j - 1;
    for (int e = tid; e < rem * rem; e += nt) {
      const int i = j + 1 + e / rem, l = j + 1 + e % rem;
      if (l <= i) L[i * ld + l] -= L[i * ld + j] * L[l * ld + j];
    }
    // keep the upper part consistent for the pivot swaps of later steps
    __syncthreads();
    for (int e = tid; e < rem * rem; e += nt) {
      const int i = j + 1 + e / rem, l = j + 1 + e % rem;
      if (l > i) L[i * ld + l] = L[l * ld + i];
    }
    __syncthreads();
  }
  const int rk = rank_s;
  // L^{-1} (rk x rk lower): thread c solves column c by forward substitution
  for (int c = tid; c < rk; c += nt) {
    for (int i = 0; i < c; ++i) Li[i * ld + c] = 0.0;
    for (int i = c; i < rk; ++i) {
      double sacc = (i == c) ? 1.0 : 0.0;
      for (int l = c; l < i; ++l) sacc -= L[i * ld + l] * Li[l * ld + c];
      Li[i * ld + c] = sacc / L[i * ld + i];
    }
  }
  __syncthreads();
  double* Wb = W + (size_t)b * k * k;
  for (int e = tid; e < k * k; e += nt) {
    const int i = e / k, c = e % k;  // W[perm[i]][c] = Linv[c][i]
    Wb[(size_t)perm[i] * k + c] = (c < rk && i < rk) ? Li[c * ld + i] : 0.0;
  }
  for (int c = tid; c < k; c += nt) mu[(size_t)b * k + c] = c < rk ? 1.0 : 0.0;
}

// Same contract as chol_basis_kernel for k <= 64 (round 2): pivoted Cholesky of C without row / column
// swaps (the pivots are chosen among the indices not yet eliminated, the full symmetric matrix is updated in
// place) and X = L^{-1} accumulated in the same elimination loop, so a step is [warp 0 picks the pivot] |
// barrier | [all threads: trailing update; the previous step's rank-1 term added to the not-yet-pivoted rows
// of acc (acc_i = sum_{t<j} L(i, t) X_t); row j of X = (e_j - acc_p) / L_jj, stored in place of acc_p] |
// barrier -- no serial column solve afterwards (the kernel above: ~6 barriers per step, a mirror pass and
// one thread per column of L^{-1}; 231 us per 250 C4 matrices).  256 threads.
constexpr int kCb2Threads = 256, kCb2MaxK = 64;
__global__ void __launch_bounds__(kCb2Threads) chol_basis2_kernel(const double* __restrict__ Cg, int k,
                                                                  double* __restrict__ W, double* __restrict__ mu) {
  extern __shared__ double cb_sm[];
  const int ld = k + 1;
  double* A = cb_sm;                 // [k][ld] the symmetric trailing matrix (original indexing)
  double* AX = cb_sm + (size_t)k * ld;  // [k][ld] acc_i (not yet pivoted i), X row j in row piv[j]
  __shared__ double ub[2][kCb2MaxK];    // u_j(i) = A(i, p_j) / sqrt(d_j), i not eliminated before step j
  __shared__ int piv[kCb2MaxK], done[kCb2MaxK];
  __shared__ double dmax0_s, rs_s;
  __shared__ int p_s, rank_s;
  const int b = blockIdx.x, tid = threadIdx.x, nt = blockDim.x;
  const double* Cb = Cg + (size_t)b * k * k;
  for (int e = tid; e < k * k; e += nt) {
    const int i = e / k, l = e - (e / k) * k;
    A[i * ld + l] = Cb[e];
    AX[i * ld + l] = 0.0;
  }
  for (int i = tid; i < k; i += nt) {
    done[i] = 0;
    ub[0][i] = ub[1][i] = 0.0;
  }
  __syncthreads();
  if (tid < 32) {
    double d = 0.0;
    for (int i = tid; i < k; i += 32) d = fmax(d, A[i * ld + i]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) d = fmax(d, __shfl_xor_sync(0xffffffffu, d, o));
    if (tid == 0) {
      dmax0_s = d;
      rank_s = k;
    }
  }
  __syncthreads();
  const double floor_piv = 1e-13 * dmax0_s;
  for (int j = 0; j < k; ++j) {
    if (tid < 32) {  // pivot: largest remaining diagonal (ties -> lowest index)
      double best = -1.0;
      int bi = k;
      for (int i = tid; i < k; i += 32) {
        const double d = done[i] ? -1.0 : A[i * ld + i];
        if (d > best) { best = d; bi = i; }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double ob = __shfl_xor_sync(0xffffffffu, best, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
      }
      if (tid == 0) {
        if (!(best > floor_piv)) {
          rank_s = j;
        } else {
          p_s = bi;
          piv[j] = bi;
          done[bi] = 1;
          rs_s = rsqrt(best);
        }
      }
    }
    __syncthreads();
    if (rank_s == j) break;
    const int p = p_s;
    const double rs = rs_s;                 // 1 / L_jj
    const double rd = rs * rs;              // 1 / d_j
    const double* up = ub[(j - 1) & 1];     // u_{j-1} (zero at j = 0)
    double* un = ub[j & 1];
    const double* xprev = j > 0 ? AX + (size_t)piv[j - 1] * ld : nullptr;  // X row j - 1 (pivot order)
    // u_j and the trailing update of the not-eliminated rows / columns (column p itself is read only);
    // thread (ty, tx) of the 16 x 16 grid owns rows ty + 16 a and columns tx + 16 b (no index division)
    const int ty = tid >> 4, tx = tid & 15;
    if (tid < k) un[tid] = done[tid] ? 0.0 : A[tid * ld + p] * rs;
    double ci[4], cl[4], ui[4], xc[4];
    bool di[4], dl[4];
#pragma unroll
    for (int a = 0; a < 4; ++a) {
      const int i = ty + 16 * a, l = tx + 16 * a;
      di[a] = i >= k || done[i];
      dl[a] = l >= k || done[l];
      ci[a] = i < k ? A[i * ld + p] * rd : 0.0;
      cl[a] = l < k ? A[l * ld + p] : 0.0;
      ui[a] = i < k ? up[i] : 0.0;
      xc[a] = (j > 0 && l < j) ? xprev[l] : 0.0;
    }
#pragma unroll
    for (int a = 0; a < 4; ++a) {
      const int i = ty + 16 * a;
      if (i >= k) continue;
      // acc rows: add the step j - 1 term L(i, j-1) X_{j-1} = u_{j-1}(i) X_{j-1} (rows not yet pivoted,
      // and the new pivot's row p, whose X row j is formed from it after the barrier)
      const bool acc_row = j > 0 && (!done[i] || i == p);
#pragma unroll
      for (int bq = 0; bq < 4; ++bq) {
        const int l = tx + 16 * bq;
        if (l >= k) continue;
        if (!di[a] && !dl[bq]) A[i * ld + l] = fma(-ci[a], cl[bq], A[i * ld + l]);
        if (acc_row && l < j) AX[i * ld + l] = fma(ui[a], xc[bq], AX[i * ld + l]);
      }
    }
    __syncthreads();
    // row j of X = L^{-1}: X_jc = (delta_jc - acc_p(c)) / L_jj, c <= j, in place of acc_p
    for (int c = tid; c <= j; c += nt) AX[p * ld + c] = ((c == j ? 1.0 : 0.0) - (c < j ? AX[p * ld + c] : 0.0)) * rs;
    __syncthreads();
  }
  const int rk = rank_s;
  double* Wb = W + (size_t)b * k * k;
  for (int e = tid; e < k * k; e += nt) {
    const int i = e / k, c = e - (e / k) * k;  // W[piv[i]][c] = Linv[c][i] = X row c (in row piv[c]), column i
    if (i < rk) Wb[(size_t)piv[i] * k + c] = (c < rk && i <= c) ? AX[(size_t)piv[c] * ld + i] : 0.0;
  }
  // indices never pivoted (rank < k): zero rows of W (done[] marks exactly the pivoted indices)
  for (int e = tid; e < k * k; e += nt) {
    const int a = e / k;
    if (!done[a]) Wb[e] = 0.0;
  }
  for (int c = tid; c < k; c += nt) mu[(size_t)b * k + c] = c < rk ? 1.0 : 0.0;
}

// below err^2 = tau ||A||^2 the Pythagorean error is replaced by the dense residual (reading c17)
constexpr double kScwPythTau = 3e-3;

static inline unsigned nb(long long n, int t) { return (unsigned)((n + t - 1) / t); }


// err_b = ||A_b - L_b R_b^T||_F for factors with row pitch ldf (a multiple of 4): L R^T on tcgen05
// (3xTF32, K = r, one 128 x 128 tile per unit) with the residual epilogue of gemm_tc.cu reading
// the A tile and reducing (a - s)^2 in fp64; fixed-order reduction of the per-warp partials.
static tsk_status residual_tc(Ctx* ctx, const float* Ac, int bc, int m, int n, const float* Lc, const float* Rc,
                              int r, int ldf, double* part, double* err, const int* only = nullptr,
                              const int* only_any = nullptr) {
  GemmProblem gp;
  gp.X = Lc;
  gp.Y = Rc;
  gp.M = m;
  gp.N = n;
  gp.n = r;
  gp.D = bc;
  gp.x_row_stride = ldf;
  gp.x_slice_stride = (long long)m * ldf;
  gp.y_row_stride = ldf;
  gp.y_slice_stride = (long long)n * ldf;
  gp.batch = 1;
  gp.bn = 128;
  gp.resA = Ac;
  gp.res_stride = (long long)m * n;
  gp.res_ld = n;
  gp.res_part = part;
  gp.only = only;
  gp.only_any = only_any;
  tsk_status st = gemm_tf32x3(ctx, gp);
  if (st != TSK_OK) return st;
  const int per = (int)(nb(m, 128) * nb(n, 128)) * 8;  // partials per matrix
  scw_err_reduce_kernel<<<nb((long long)bc * 32, 256), 256, 0, ctx->stream>>>(part, per, bc, err, only);
  ctx->count_launch();
  return launch_status("scw residual (tcgen05)");
}

static void scw_attrs() {
  static uint64_t attr = 0;
  if (!(attr & device_bit())) {
    cudaFuncSetAttribute(scw_combine_kernel<64, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
    cudaFuncSetAttribute(scw_combine_kernel<128, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
    cudaFuncSetAttribute(scw_combine_kernel<64, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
    cudaFuncSetAttribute(scw_combine_kernel<128, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
    cudaFuncSetAttribute(chol_basis_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kCholSmemMax);
    cudaFuncSetAttribute(scw_vt_dmma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kVtSmem);
    cudaFuncSetAttribute(chol_basis2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         2 * kCb2MaxK * (kCb2MaxK + 1) * 8);
    attr |= device_bit();
  }
}

tsk_status scw_run(Ctx* ctx, const float* A, long long B, int m, int n, const float* S, int k, int r, float* L,
                   float* R, float* sigma, double* err) {
  if (B == 0) return TSK_OK;
  if (k > 128 || r > 64) return TSK_EINVAL;
  const cudaStream_t s0 = ctx->stream;
  const long long chunk = std::min<long long>(B, 512);
  const size_t kn = (size_t)k * n, km = (size_t)k * m, kk = (size_t)k * k;
  float* Bm_all = reinterpret_cast<float*>(ctx->workspace(WS_SCW_0, chunk * kn * 4));
  float* Vt_all = reinterpret_cast<float*>(ctx->workspace(WS_SCW_1, chunk * kn * 4));
  float* Zt_all = reinterpret_cast<float*>(ctx->workspace(WS_SCW_2, chunk * km * 4));
  // small matrices per matrix + one int flag per possible part offset (the eigensolver fallback gate)
  double* small = reinterpret_cast<double*>(ctx->workspace(WS_SCW_3, chunk * (4 * kk + 2 * k) * 8 + chunk * 4 + 64));
  const int tiles = (int)(nb(n, 128) * nb(m, 128)) * 8;  // residual partials per matrix
  // factor row pitch: r for the caller's L / R, r rounded up to 4 (16-byte TMA rows) for the error path
  const int ldf = (L || R) ? r : (r + 3) & ~3;
  float* Lw = reinterpret_cast<float*>(ctx->workspace(WS_SCW_4, chunk * ((size_t)m + n) * ldf * 4));
  // residual partials, then the ||A||^2 partials of the SA product (8 per unit, nb(n, 128) units per
  // matrix) and the dense-residual marks of the Pythagorean error path
  const int sq_per = (int)nb(n, 128) * 8;
  double* part = reinterpret_cast<double*>(
      ctx->workspace(WS_SCW_5, chunk * ((size_t)tiles + sq_per) * 8 + chunk * 8 + 64));
  if (!Bm_all || !Vt_all || !Zt_all || !small || !Lw || !part) return TSK_ENOMEM;
  double* sq_all = part + chunk * tiles;
  // eigensolver scratch per matrix: the parts run concurrently on different streams
  const long long eig_ws = std::max(syev_ws_doubles(k), jacobi_ws_doubles(k));
  double* eigws_all = reinterpret_cast<double*>(ctx->workspace(WS_SCW_EIG, (size_t)chunk * eig_ws * 8));
  if (!eigws_all) return TSK_ENOMEM;
  int* dense_all = reinterpret_cast<int*>(sq_all + chunk * sq_per);
  int* ndense_all = dense_all + chunk;  // one counter per part (indexed by the part's offset)
  // Pythagorean error path (reading c17) unless TSK_SCW_DENSE; tau: the cancellation threshold
  static const bool force_dense = getenv("TSK_SCW_DENSE") != nullptr;
  static const double env_tau = getenv("TSK_SCW_PYTH_TAU") ? atof(getenv("TSK_SCW_PYTH_TAU")) : kScwPythTau;
  const double pyth_tau = ctx->scw_tau > 0.0 ? ctx->scw_tau : env_tau;
  const bool pyth = err && !force_dense && ctx->scw_err_mode == 0;
  double* Cb_all = small;
  double* Wc_all = small + chunk * kk;
  double* H_all = small + 2 * chunk * kk;
  double* W2_all = small + 3 * chunk * kk;
  double* mu_all = small + 4 * chunk * kk;
  double* sig2_all = mu_all + chunk * k;
  scw_attrs();
  // S is the broadcast TMA operand of the SA product: its row pitch must be a multiple of 16 bytes, so
  // for m % 4 != 0 it is copied once into a padded buffer (the tensor map's extent stays m: the pad is
  // never read)
  const int ms = (m + 3) & ~3;
  if (ms != m) {
    float* Sp = reinterpret_cast<float*>(ctx->workspace(WS_SCW_S, (size_t)k * ms * 4));
    if (!Sp) return TSK_ENOMEM;
    if (cudaMemcpy2DAsync(Sp, (size_t)ms * 4, S, (size_t)m * 4, (size_t)m * 4, k, cudaMemcpyDeviceToDevice,
                          s0) != cudaSuccess)
      return TSK_ECUDA;
    S = Sp;
  }
  // Each chunk runs as two halves on two streams, the second started one phase (its SA product)
  // behind the first, so the latency-bound small solves of one half (row Grams, pivoted Cholesky,
  // batched Jacobi, factor combinations) overlap the HBM/tensor-bound products of the other.
  const bool two = chunk >= 64 && k <= 116 && ctx->side_ready();
  auto half = [&](long long b0, int bc, long long off0, cudaStream_t s, cudaEvent_t after_sa) -> tsk_status {
    ctx->stream = s;
    tsk_status st;
    const size_t off = (size_t)off0;
    const float* Ac = A + (size_t)b0 * m * n;
    float* Bm = Bm_all + off * kn;
    float* Vt = Vt_all + off * kn;
    float* Zt = Zt_all + off * km;
    double* Cb = Cb_all + off * kk;
    double* Wc = Wc_all + off * kk;
    double* H = H_all + off * kk;
    double* W2 = W2_all + off * kk;
    double* mu = mu_all + off * k;
    double* sig2 = sig2_all + off * k;
    double* eigws = eigws_all + off * eig_ws;
    // 1. B = S A on tcgen05 (3xTF32): (S A_b)^T = A_b^T S^T with X = A_b read transposed (the
    // contraction runs over the rows of A_b), Y = S broadcast to every matrix; one unit per
    // (matrix, 128-column tile of A_b), stored transposed as B [k][n]
    {
      GemmProblem gp;
      gp.X = Ac;
      gp.Y = S;
      gp.M = n;
      gp.N = k;
      gp.n = m;
      gp.D = bc;
      gp.xt = 1;
      gp.x_row_stride = n;
      gp.x_slice_stride = (long long)m * n;
      gp.ybc = 1;
      gp.y_row_stride = ms;
      gp.y_slice_stride = ms;
      gp.batch = 1;
      gp.bn = k <= 64 ? 64 : 128;
      gp.dout = Bm;
      gp.dstride = (long long)k * n;
      gp.ldd = n;
      if (pyth) gp.sq_part = sq_all + off * sq_per;
      if ((st = gemm_tf32x3(ctx, gp)) != TSK_OK) return st;
    }
    if (after_sa) cudaEventRecord(after_sa, s);
    // 2. orthonormal row basis of B: fp64 Gram, pivoted Cholesky, V^T = L^{-1} P B (k > 116 does
    // not fit the factor and its inverse in shared memory: eigen-orthonormalisation instead)
    launch_gram_rows_tiled(Bm, k, n, bc, Cb, s);
    ctx->count_launch(1);
    if ((st = launch_status("scw gram(SA)")) != TSK_OK) return st;
    if ((size_t)2 * k * (k + 1) * 8 <= (size_t)kCholSmemMax) {
      if (k <= kCb2MaxK && !getenv("TSK_SCW_CHOL1"))
        chol_basis2_kernel<<<bc, kCb2Threads, (size_t)2 * k * (k + 1) * 8, s>>>(Cb, k, Wc, mu);
      else
        chol_basis_kernel<<<bc, 128, (size_t)2 * k * (k + 1) * 8, s>>>(Cb, k, Wc, mu);
      ctx->count_launch(1);
      if ((st = launch_status("scw chol_basis")) != TSK_OK) return st;
    } else if ((st = jacobi_eig_batched(ctx, Cb, k, bc, Wc, mu, nullptr, 1e-10, nullptr, eigws)) != TSK_OK) {
      return st;
    }
    if (k <= 64 && (n & 1) == 0 && !getenv("TSK_SCW_VT_DFMA"))
      scw_vt_dmma_kernel<<<dim3((n + kVtCols - 1) / kVtCols, bc), 128, kVtSmem, s>>>(Bm, Wc, mu, k, n, (long long)kk, Vt);
    else
      launch_combine2<true>(Bm, Wc, mu, k, n, k, k, (long long)kk, Vt, 0, bc, s);
    ctx->count_launch();
    if ((st = launch_status("scw vt")) != TSK_OK) return st;
    // 3. Z^T = V^T A^T
    {
      // Z^T[b] = V^T[b] A[b]^T on tcgen05 (3xTF32): X = A_b (m rows, K = n), Y = V^T_b (k rows),
      // one unit per (matrix, 128-row tile), result stored transposed as Z^T [k][m]
      GemmProblem gp;
      gp.X = Ac;
      gp.Y = Vt;
      gp.M = m;
      gp.N = k;
      gp.n = n;
      gp.D = bc;
      gp.x_row_stride = n;
      gp.x_slice_stride = (long long)m * n;
      gp.y_row_stride = n;
      gp.y_slice_stride = (long long)k * n;
      gp.batch = 1;
      gp.bn = k <= 64 ? 64 : 128;
      gp.dout = Zt;
      gp.dstride = (long long)k * m;
      gp.ldd = m;
      // the Pythagorean error is first-order in a scale bias of AV: one TMEM accumulation chain per
      // 32-deep chunk (the tensor core's truncating accumulation, reading c17), fp32 sums across chunks;
      // the same on the dense error path, so both formulas see the same factors
      static const int av_chain = getenv("TSK_SCW_AV_CHAIN") ? atoi(getenv("TSK_SCW_AV_CHAIN")) : 0;
      gp.chain = av_chain > 0 ? av_chain : (err ? 1 : 0);
      if ((st = gemm_tf32x3(ctx, gp)) != TSK_OK) return st;
    }
    // 4. SVD of AV through its Gram
    launch_gram_rows_tiled(Zt, k, m, bc, H, s);
    ctx->count_launch(1);
    if ((st = launch_status("scw gram(AV)")) != TSK_OK) return st;
    // top-r eigenpairs of (AV)^T (AV): the tridiagonal eigensolver (syev.cu) for the batch; a problem whose
    // wanted eigenvalues form an unresolved cluster (e.g. rank(A) < r: a null cluster among them) sets the
    // flag, and the Jacobi eigensolver -- enqueued behind it, gated on the flag on the device -- redoes the
    // batch (no host round trip)
    // on the error-only path the eigenvalues come first (bisection only) and the vectors -- needed for the
    // rank-r factors of the dense residual -- only for the matrices the Pythagorean step marks
    const bool vals_first = pyth && !L && !R;
    int* gflag = reinterpret_cast<int*>(small + chunk * (4 * kk + 2 * k)) + off;
    cudaMemsetAsync(gflag, 0, sizeof(int), s);
    if ((st = syev_top_batched(ctx, H, k, r, bc, W2, k, sig2, gflag, 1e-9, k, eigws, vals_first ? 1 : 0)) != TSK_OK)
      return st;
    if (!vals_first && (st = jacobi_eig_batched(ctx, H, k, bc, W2, sig2, nullptr, 1e-10, gflag, eigws)) != TSK_OK)
      return st;
    // 5. errors by the Pythagorean identity first: on the error-only path (no caller factors) the
    // factors are then formed only for the matrices it marks for the dense residual
    if (pyth) {
      cudaMemsetAsync(ndense_all + off, 0, sizeof(int), s);
      scw_err_pyth_kernel<<<nb((long long)bc * 32, 256), 256, 0, s>>>(sq_all + off * sq_per, sq_per, sig2, k, r, bc,
                                                                      pyth_tau, err + b0, dense_all + off,
                                                                      ndense_all + off);
      ctx->count_launch();
    }
    if (vals_first) {
      if ((st = syev_top_batched(ctx, H, k, r, bc, W2, k, sig2, gflag, 1e-9, k, eigws, 2, dense_all + off)) != TSK_OK)
        return st;
      if ((st = jacobi_eig_batched(ctx, H, k, bc, W2, sig2, nullptr, 1e-10, gflag, eigws)) != TSK_OK) return st;
    }
    // 6. factors (all matrices when the caller asked for them)
    const int* fmask = (pyth && !L && !R) ? dense_all + off : nullptr;
    float* Lc = L ? L + (size_t)b0 * m * r : Lw + (size_t)off * m * ldf;
    float* Rc = R ? R + (size_t)b0 * n * r : Lw + (size_t)chunk * m * ldf + (size_t)off * n * ldf;
    if (L || R || err) {
      launch_combine2<false>(Zt, W2, nullptr, k, m, r, k, (long long)kk, Lc, ldf, bc, s, fmask);
      launch_combine2<false>(Vt, W2, nullptr, k, n, r, k, (long long)kk, Rc, ldf, bc, s, fmask);
      ctx->count_launch(2);
    }
    if (sigma) {
      scw_sigma_kernel<<<nb((long long)bc * r, 256), 256, 0, s>>>(sig2, k, r, bc, sigma + (size_t)b0 * r);
      ctx->count_launch();
    }
    // 7. dense residual for the marked matrices (all of them with TSK_SCW_DENSE); the error path always
    // has pitch-aligned workspace factors
    if (err && (st = residual_tc(ctx, Ac, bc, m, n, Lc, Rc, r, ldf, part + (size_t)off * tiles, err + b0,
                                 pyth ? dense_all + off : nullptr, pyth ? ndense_all + off : nullptr)) != TSK_OK)
      return st;
    if ((st = launch_status("scw")) != TSK_OK) return st;
    return TSK_OK;
  };
  const int nparts_max = getenv("TSK_SCW_PARTS") ? std::max(1, std::min(Ctx::kSide + 1, atoi(getenv("TSK_SCW_PARTS")))) : 2;
  for (long long b0 = 0; b0 < B; b0 += chunk) {
    const int bc = (int)std::min(chunk, B - b0);
    tsk_status st = TSK_OK;
    const int parts = two ? std::min(nparts_max, bc / 32) : 1;
    if (parts >= 2) {
      cudaEventRecord(ctx->ev[0], s0);  // fork: the side streams start after the work before this call
      for (int j = 1; j < parts; ++j) cudaStreamWaitEvent(ctx->side[j - 1], ctx->ev[0], 0);
      for (int j = 0; j < parts && st == TSK_OK; ++j) {
        const int o0 = (int)((long long)bc * j / parts), o1 = (int)((long long)bc * (j + 1) / parts);
        cudaStream_t sj = j == 0 ? s0 : ctx->side[j - 1];
        if (j > 0) cudaStreamWaitEvent(sj, ctx->ev[j], 0);  // one phase behind part j - 1
        st = half(b0 + o0, o1 - o0, o0, sj, j + 1 < parts ? ctx->ev[j + 1] : nullptr);
      }
      ctx->stream = s0;
      for (int j = 1; j < parts; ++j) {  // join
        cudaEventRecord(ctx->ev[Ctx::kSide + j], ctx->side[j - 1]);
        cudaStreamWaitEvent(s0, ctx->ev[Ctx::kSide + j], 0);
      }
    } else {
      st = half(b0, bc, 0, s0, nullptr);
      ctx->stream = s0;
    }
    if (st != TSK_OK) return st;
  }
  return TSK_OK;
}

// Two-sided SCW (Algorithm 3) for a batch of test matrices:
//   1. Q^T = orthonormal basis of rowspace(S A_b)    (k x n; as steps 1-2 of SCW)
//   2. P^T = orthonormal basis of rowspace(W A_b^T)  (l x m) = col(A_b W^T) (line 2, QR -> CholQR)
//   3. M   = P^T A_b Q = P^T (A_b Q)                 (l x k; A_b Q as step 3 of SCW, fp64 cross Gram)
//   4. [M]_r through M^T M = W2 diag(sigma^2) W2^T   (k x k Jacobi)
//   5. A_hat = P [M]_r Q^T = L R^T,  L = P (M W2_r) (m x r),  R = Q W2_r (n x r)
//   6. e_b = ||A_b - L R^T||_F                        (dense residual, fp64 reduction)
tsk_status scw2_run(Ctx* ctx, const float* A, long long B, int m, int n, const float* S, int k, const float* W, int l,
                    int r, float* L, float* R, float* sigma, double* err) {
  if (B == 0) return TSK_OK;
  if (k > 128 || l > 128 || r > 64 || r > k || r > l) return TSK_EINVAL;
  cudaStream_t s = ctx->stream;
  const long long chunk = std::min<long long>(B, 256);
  const size_t kn = (size_t)k * n, km = (size_t)k * m, kk = (size_t)k * k, lm = (size_t)l * m, ll = (size_t)l * l;
  float* Bm = reinterpret_cast<float*>(ctx->workspace(WS_SCW_0, chunk * kn * 4));
  float* Vt = reinterpret_cast<float*>(ctx->workspace(WS_SCW_1, chunk * kn * 4));
  float* Zt = reinterpret_cast<float*>(ctx->workspace(WS_SCW_2, chunk * km * 4));
  float* Yt = reinterpret_cast<float*>(ctx->workspace(WS_SCW2_0, chunk * lm * 4));
  float* Pt = reinterpret_cast<float*>(ctx->workspace(WS_SCW2_1, chunk * lm * 4));
  // per matrix: Cq, Wq, H2, W2 [k][k]; Cp, Wp [l][l]; Mx [l][k]; CL [l][r]; muq, sig2 [k]; mup [l]
  // (the sum was short by k(k - l) - l doubles per matrix: for k > l + 1 the last arrays of a chunk
  // ran past the allocation -- found by scripts/random_sweep2.py)
  const size_t nsmall = chunk * (4 * kk + 2 * ll + (size_t)l * k + (size_t)l * r + 2 * (size_t)k + (size_t)l);
  double* small = reinterpret_cast<double*>(ctx->workspace(WS_SCW2_2, nsmall * 8));
  const int tiles = (int)(nb(n, 128) * nb(m, 128)) * 8;
  const int ldf = (L || R) ? r : (r + 3) & ~3;
  float* Lw = reinterpret_cast<float*>(ctx->workspace(WS_SCW_4, chunk * ((size_t)m + n) * ldf * 4));
  double* part = reinterpret_cast<double*>(ctx->workspace(WS_SCW_5, chunk * (size_t)tiles * 8 + 64));
  if (!Bm || !Vt || !Zt || !Yt || !Pt || !small || !Lw || !part) return TSK_ENOMEM;
  double* Cq = small;                      // [k][k]
  double* Wq = Cq + chunk * kk;            // [k][k]
  double* Cp = Wq + chunk * kk;            // [l][l]
  double* Wp = Cp + chunk * ll;            // [l][l]
  double* Mx = Wp + chunk * ll;            // [l][k]
  double* H2 = Mx + chunk * (size_t)l * k; // [k][k]
  double* W2 = H2 + chunk * kk;            // [k][k]
  double* CL = W2 + chunk * kk;            // [l][r]
  double* muq = CL + chunk * (size_t)l * r;
  double* sig2 = muq + chunk * k;
  double* mup = sig2 + chunk * k;
  scw_attrs();
  if ((size_t)2 * std::max(k, l) * (std::max(k, l) + 1) * 8 > (size_t)kCholSmemMax) return TSK_EINVAL;
  tsk_status st;
  for (long long b0 = 0; b0 < B; b0 += chunk) {
    const int bc = (int)std::min(chunk, B - b0);
    const float* Ac = A + (size_t)b0 * m * n;
    // 1. Q^T: S A_b (tcgen05, A_b transposed), fp64 Gram, pivoted Cholesky, V^T = L^-1 P B
    {
      GemmProblem gp;
      gp.X = Ac; gp.Y = S; gp.M = n; gp.N = k; gp.n = m; gp.D = bc;
      gp.xt = 1; gp.x_row_stride = n; gp.x_slice_stride = (long long)m * n;
      gp.ybc = 1; gp.y_row_stride = m; gp.y_slice_stride = m;
      gp.batch = 1; gp.bn = k <= 64 ? 64 : 128;
      gp.dout = Bm; gp.dstride = (long long)k * n; gp.ldd = n;
      if ((st = gemm_tf32x3(ctx, gp)) != TSK_OK) return st;
    }
    launch_gram_rows_tiled(Bm, k, n, bc, Cq, s);
    chol_basis_kernel<<<bc, 128, (size_t)2 * k * (k + 1) * 8, s>>>(Cq, k, Wq, muq);
    if (k <= 64) scw_combine_kernel<64, true><<<dim3(nb(n, 256), bc), 128, combine_smem(k, k), s>>>(Bm, Wq, muq, k, n, k, k, (long long)kk, Vt, 0);
    else scw_combine_kernel<128, true><<<dim3(nb(n, 256), bc), 128, combine_smem(k, k), s>>>(Bm, Wq, muq, k, n, k, k, (long long)kk, Vt, 0);
    ctx->count_launch(3);
    if ((st = launch_status("scw2 Q")) != TSK_OK) return st;
    // 2. P^T: W A_b^T = (A_b W^T)^T (tcgen05, W broadcast, transposed store), same orthonormalisation
    {
      GemmProblem gp;
      gp.X = Ac; gp.Y = W; gp.M = m; gp.N = l; gp.n = n; gp.D = bc;
      gp.x_row_stride = n; gp.x_slice_stride = (long long)m * n;
      gp.ybc = 1; gp.y_row_stride = n; gp.y_slice_stride = n;
      gp.batch = 1; gp.bn = l <= 64 ? 64 : 128;
      gp.dout = Yt; gp.dstride = (long long)l * m; gp.ldd = m;
      if ((st = gemm_tf32x3(ctx, gp)) != TSK_OK) return st;
    }
    launch_gram_rows_tiled(Yt, l, m, bc, Cp, s);
    chol_basis_kernel<<<bc, 128, (size_t)2 * l * (l + 1) * 8, s>>>(Cp, l, Wp, mup);
    if (l <= 64) scw_combine_kernel<64, true><<<dim3(nb(m, 256), bc), 128, combine_smem(l, l), s>>>(Yt, Wp, mup, l, m, l, l, (long long)ll, Pt, 0);
    else scw_combine_kernel<128, true><<<dim3(nb(m, 256), bc), 128, combine_smem(l, l), s>>>(Yt, Wp, mup, l, m, l, l, (long long)ll, Pt, 0);
    ctx->count_launch(3);
    if ((st = launch_status("scw2 P")) != TSK_OK) return st;
    // 3. A_b Q as Z^T = Q^T A_b^T (tcgen05), then M = P^T (A_b Q) as an fp64 cross Gram of rows
    {
      GemmProblem gp;
      gp.X = Ac; gp.Y = Vt; gp.M = m; gp.N = k; gp.n = n; gp.D = bc;
      gp.x_row_stride = n; gp.x_slice_stride = (long long)m * n;
      gp.y_row_stride = n; gp.y_slice_stride = (long long)k * n;
      gp.batch = 1; gp.bn = k <= 64 ? 64 : 128;
      gp.dout = Zt; gp.dstride = (long long)k * m; gp.ldd = m;
      if ((st = gemm_tf32x3(ctx, gp)) != TSK_OK) return st;
    }
    launch_gram_cross(Pt, l, Zt, k, m, bc, Mx, s);
    // 4. [M]_r through M^T M
    gram_cols_f64_kernel<<<bc, 256, 0, s>>>(Mx, l, k, H2);
    ctx->count_launch(2);
    if ((st = launch_status("scw2 M")) != TSK_OK) return st;
    if ((st = jacobi_eig_batched(ctx, H2, k, bc, W2, sig2, nullptr, 1e-10)) != TSK_OK) return st;
    // 5. factors: L = P (M W2_r), R = Q W2_r
    small_mm_f64_kernel<<<bc, 256, 0, s>>>(Mx, W2, l, k, r, CL);
    float* Lc = L ? L + (size_t)b0 * m * r : Lw;
    float* Rc = R ? R + (size_t)b0 * n * r : Lw + (size_t)chunk * m * ldf;
    if (k <= 64 && l <= 64) {
      scw_combine_kernel<64, false><<<dim3(nb(m, 256), bc), 128, combine_smem(l, r), s>>>(Pt, CL, nullptr, l, m, r, r,
                                                                                 (long long)l * r, Lc, ldf);
      scw_combine_kernel<64, false><<<dim3(nb(n, 256), bc), 128, combine_smem(k, r), s>>>(Vt, W2, nullptr, k, n, r, k,
                                                                                 (long long)kk, Rc, ldf);
    } else {
      scw_combine_kernel<128, false><<<dim3(nb(m, 256), bc), 128, combine_smem(l, r), s>>>(Pt, CL, nullptr, l, m, r, r,
                                                                                  (long long)l * r, Lc, ldf);
      scw_combine_kernel<128, false><<<dim3(nb(n, 256), bc), 128, combine_smem(k, r), s>>>(Vt, W2, nullptr, k, n, r, k,
                                                                                  (long long)kk, Rc, ldf);
    }
    ctx->count_launch(3);
    if (sigma) {
      scw_sigma_kernel<<<nb((long long)bc * r, 256), 256, 0, s>>>(sig2, k, r, bc, sigma + (size_t)b0 * r);
      ctx->count_launch();
    }
    // 6. dense residual
    if (err && (st = residual_tc(ctx, Ac, bc, m, n, Lc, Rc, r, ldf, part, err + b0)) != TSK_OK) return st;
    if ((st = launch_status("scw2")) != TSK_OK) return st;
  }
  return TSK_OK;
}

}  // namespace tsk
