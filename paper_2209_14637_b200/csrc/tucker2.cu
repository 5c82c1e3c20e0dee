// Two-sided variant: the mode-2 Gram and Tucker2 by HOOI over modes 1-2
// (Eq. (9); Appendix Algorithm 5).
//
// Every HOOI step is a Gram of a projected unfolding (BASELINE north_star: "each sweep is the
// same Gram contraction on the projected unfolding"), all on the tcgen05 3xTF32 kernels:
//   HOSVD init:  G1 = sum_d A_d A_d^T  (CTA-pair Gram)        -> S = top-k eigenvectors
//                G2 = sum_d A_d^T A_d  (TS kernel, both operands read transposed) -> W = top-l
//   sweep s:     Y_d = A_d W^T  [D][m][l]   (batched TS kernel, W broadcast, row-major output)
//                G1' = sum_d Y_d Y_d^T      (CTA-pair Gram over K = l)  -> S = top-k
//                Z_d = A_d^T S^T [D][n][k]  (batched TS kernel, A_d transposed, S broadcast)
//                G2' = sum_d Z_d Z_d^T      (CTA-pair Gram over K = k)  -> W = top-l, energy
//   residual:    ||A - G x1 S^T x2 W^T||^2 = ||A||^2 - ||G||^2 with ||G||^2 = sum of the top-l
//                eigenvalues of G2' (orthonormal S, W; reading t4) and ||A||^2 = trace(G1).
// Readings t1-t3: modes 1-2 only, HOSVD init, mode 1 then mode 2 in each sweep,
// stop on the relative change of the residual.
#include <algorithm>
#include <cmath>
#include <vector>

#include "ptx.cuh"
#include "tsk_internal.h"

namespace tsk {

__global__ void trace_kernel(const double* __restrict__ G, int m, double* __restrict__ out) {
  __shared__ double red[256];
  double s = 0.0;
  for (int i = threadIdx.x; i < m; i += blockDim.x) s += G[(size_t)i * m + i];
  red[threadIdx.x] = s;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if ((int)threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = red[0];
}

// out[c] = s_c^T G s_c for the rows s_c of S [k][m] (one CTA per row; fixed-order reduction)
__global__ void quad_form_kernel(const double* __restrict__ G, const float* __restrict__ S, int m,
                                 double* __restrict__ out) {
  __shared__ double red[256];
  const int c = blockIdx.x;
  const float* w = S + (size_t)c * m;
  double acc = 0.0;
  for (int i = threadIdx.x; i < m; i += blockDim.x) {
    const double* Gi = G + (size_t)i * m;
    double gi = 0.0;
    for (int j = 0; j < m; ++j) gi += Gi[j] * (double)w[j];
    acc += (double)w[i] * gi;
  }
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if ((int)threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) out[c] = red[0];
}

tsk_status gram_mode2(Ctx* ctx, const float* A, long long D, int m, int n, double* G64, int accumulate) {
  GemmProblem p;
  p.X = A;
  p.Y = A;
  p.M = n;
  p.N = n;
  p.n = m;  // contraction over the rows of every A_d
  p.D = D;
  p.xt = 1;
  p.yt = 1;
  p.x_row_stride = n;
  p.x_slice_stride = (long long)m * n;
  p.y_row_stride = n;
  p.y_slice_stride = (long long)m * n;
  p.sym = 1;
  p.out64 = G64;
  p.ldo64 = n;
  p.accumulate = accumulate;
  return gemm_tf32x3(ctx, p);
}

// Y_d = A_d W^T for every d, row-major [D][m][l]  (X = A_d, Y = W broadcast)
static tsk_status project_right(Ctx* ctx, const float* A, long long D, int m, int n, const float* W, int l,
                                float* Y, int ldy) {
  GemmProblem p;
  p.X = A;
  p.Y = W;
  p.M = m;
  p.N = l;
  p.n = n;
  p.D = D;
  p.x_row_stride = n;
  p.x_slice_stride = (long long)m * n;
  p.ybc = 1;
  p.y_row_stride = n;
  p.y_slice_stride = n;
  p.batch = 1;
  p.bn = l <= 64 ? 64 : 128;
  p.dout = Y;
  p.drow = 1;
  p.dstride = (long long)m * ldy;
  p.ldd = ldy;
  return gemm_tf32x3(ctx, p);
}

// Z_d = A_d^T S^T for every d, row-major [D][n][k]  (X = A_d read transposed, Y = S broadcast)
static tsk_status project_left(Ctx* ctx, const float* A, long long D, int m, int n, const float* S, int k,
                               float* Z, int ldz) {
  GemmProblem p;
  p.X = A;
  p.Y = S;
  p.M = n;
  p.N = k;
  p.n = m;
  p.D = D;
  p.xt = 1;
  p.x_row_stride = n;
  p.x_slice_stride = (long long)m * n;
  p.ybc = 1;
  p.y_row_stride = m;
  p.y_slice_stride = m;
  p.batch = 1;
  p.bn = k <= 64 ? 64 : 128;
  p.dout = Z;
  p.drow = 1;
  p.dstride = (long long)n * ldz;
  p.ldd = ldz;
  return gemm_tf32x3(ctx, p);
}

// sum_d X_d X_d^T for X [D][rows][K] row-major (K % 4 == 0), fp64 [rows][rows]
static tsk_status gram_rows_stack(Ctx* ctx, const float* X, long long D, int rows, int K, double* G64) {
  GemmProblem p;
  p.X = X;
  p.Y = X;
  p.M = rows;
  p.N = rows;
  p.n = K;
  p.D = D;
  p.x_row_stride = K;
  p.x_slice_stride = (long long)rows * K;
  p.y_row_stride = K;
  p.y_slice_stride = (long long)rows * K;
  p.sym = 1;
  p.out64 = G64;
  p.ldo64 = rows;
  return gemm_tf32x3(ctx, p);
}

tsk_status hooi_tucker2(Ctx* ctx, const float* A, long long D, int m, int n, int k, int l, float* S, float* W,
                        const tsk_hooi_opts* o, tsk_hooi_info* info) {
  const int max_sweeps = std::min(64, (o && o->max_sweeps > 0) ? o->max_sweeps : 10);
  const double rel_tol = (o && o->rel_tol > 0) ? o->rel_tol : 1e-6;
  double* G1 = reinterpret_cast<double*>(ctx->workspace(WS_T2_G1, (size_t)m * m * 8 + 64));
  double* G2 = reinterpret_cast<double*>(ctx->workspace(WS_T2_G2, (size_t)n * n * 8 + 64));
  const int lp = (l + 3) & ~3, kp = (k + 3) & ~3;  // 16-byte row pitch of the projected stacks
  float* Y = reinterpret_cast<float*>(ctx->workspace(WS_T2_Y, (size_t)D * m * lp * 4));
  float* Z = reinterpret_cast<float*>(ctx->workspace(WS_T2_Z, (size_t)D * n * kp * 4));
  double* lamW = reinterpret_cast<double*>(ctx->workspace(WS_T2_SMALL, (size_t)(l + k + 8) * 8));  // [l] | ||A||^2 | [k]
  if (!G1 || !G2 || !Y || !Z || !lamW) return TSK_ENOMEM;
  double* scal = lamW + l;  // [0]: ||A||^2
  tsk_status st;
  tsk_train_opts eo{};
  tsk_train_info ei{};

  // HOSVD init (reading t1)
  GemmProblem p;
  p.X = A;
  p.Y = A;
  p.M = m;
  p.N = m;
  p.n = n;
  p.D = D;
  p.x_row_stride = n;
  p.x_slice_stride = (long long)m * n;
  p.y_row_stride = n;
  p.y_slice_stride = (long long)m * n;
  p.sym = 1;
  p.out64 = G1;
  p.ldo64 = m;
  if ((st = gemm_tf32x3(ctx, p)) != TSK_OK) return st;
  trace_kernel<<<1, 256, 0, ctx->stream>>>(G1, m, scal);
  ctx->count_launch();
  if ((st = topk_eigen(ctx, G1, m, k, S, nullptr, &eo, &ei)) < 0) return st;
  if ((st = gram_mode2(ctx, A, D, m, n, G2, 0)) != TSK_OK) return st;
  if ((st = topk_eigen(ctx, G2, n, l, W, nullptr, &eo, &ei)) < 0) return st;
  double a2 = 0.0;
  if (cudaMemcpyAsync(&a2, scal, 8, cudaMemcpyDeviceToHost, ctx->stream) != cudaSuccess ||
      cudaStreamSynchronize(ctx->stream) != cudaSuccess)
    return TSK_ECUDA;
  if (lp != l || kp != k) {  // zero the pitch padding once (the projections never write it)
    if (cudaMemsetAsync(Y, 0, (size_t)D * m * lp * 4, ctx->stream) != cudaSuccess ||
        cudaMemsetAsync(Z, 0, (size_t)D * n * kp * 4, ctx->stream) != cudaSuccess)
      return TSK_ECUDA;
  }

  std::vector<double> hist;
  std::vector<double> part(k);
  int sweeps = 0;
  bool conv = false;
  for (int s = 0; s < max_sweeps; ++s) {
    // mode 1: B = A x2 W^T, S <- top-k left singular vectors of B_(1) (through its Gram)
    if ((st = project_right(ctx, A, D, m, n, W, l, Y, lp)) != TSK_OK) return st;
    if ((st = gram_rows_stack(ctx, Y, D, m, lp, G1)) != TSK_OK) return st;
    if (s == 0) {
      // residual of the HOSVD init: ||G||^2 = sum_d ||S A_d W^T||^2 = tr(S G1' S^T) with this G1'
      quad_form_kernel<<<k, 256, 0, ctx->stream>>>(G1, S, m, scal + 1);
      ctx->count_launch();
      if (cudaMemcpyAsync(part.data(), scal + 1, (size_t)k * 8, cudaMemcpyDeviceToHost, ctx->stream) !=
              cudaSuccess ||
          cudaStreamSynchronize(ctx->stream) != cudaSuccess)
        return TSK_ECUDA;
      double e0 = 0.0;
      for (double v : part) e0 += v;
      hist.push_back(std::sqrt(std::max(a2 - e0, 0.0)));
    }
    if ((st = topk_eigen(ctx, G1, m, k, S, nullptr, &eo, &ei)) < 0) return st;
    // mode 2 with the new S (Algorithm 5 line 4: modes < n use the factors of this sweep)
    if ((st = project_left(ctx, A, D, m, n, S, k, Z, kp)) != TSK_OK) return st;
    if ((st = gram_rows_stack(ctx, Z, D, n, kp, G2)) != TSK_OK) return st;
    if ((st = topk_eigen(ctx, G2, n, l, W, lamW, &eo, &ei)) < 0) return st;
    std::vector<double> lam(l);
    if (cudaMemcpyAsync(lam.data(), lamW, (size_t)l * 8, cudaMemcpyDeviceToHost, ctx->stream) != cudaSuccess ||
        cudaStreamSynchronize(ctx->stream) != cudaSuccess)
      return TSK_ECUDA;
    double energy = 0.0;
    for (double v : lam) energy += v;
    hist.push_back(std::sqrt(std::max(a2 - energy, 0.0)));
    ++sweeps;
    const double prev = hist[hist.size() - 2], cur = hist.back();
    if (std::fabs(prev - cur) <= rel_tol * std::max(prev, 1e-300)) {
      conv = true;
      break;
    }
  }
  if (info) {
    info->sweeps = sweeps;
    info->converged = conv ? 1 : 0;
    info->a_fro2 = a2;
    for (int i = 0; i < 65; ++i) info->residual_history[i] = i < (int)hist.size() ? hist[i] : 0.0;
  }
  return conv ? TSK_OK : TSK_WARN_NOT_CONVERGED;
}

}  // namespace tsk
