// Matrix-free Tucker1 sketch by randomized block Krylov (readings mf1-mf4
// in DESIGN.md).  The sketch of Algorithm 2 line 2 (S <- Tucker1: the top-k left
// singular vectors of A_(1)) approximated from products with the training slices only --
// the m x m Gram G = sum_d A_d A_d^T is never formed:
//
//   Q_0 = orth(Omega)                                   Omega [m][p] (given, or hash-uniform)
//   j = 1..q:  Z_d = A_d^T Q_{j-1}   [D][n][p]          batched TS kernel, A_d read transposed
//              Y_j = sum_d A_d Z_d   [m][p] fp64        TS kernel, contraction over K = n D
//              Krylov: Y_j -= sum_{i<j} Q_i Q_i^T Y_j, twice (block Gram-Schmidt, fp64)
//              Q_j = CholQR2(Y_j)                       (repaired on breakdown, reading mf3)
//   K = [Q_0 | ... | Q_q]  (Krylov)  or  Q_q (subspace iteration)        m x w
//   Z_d = A_d^T K  [D][n][w];  H = sum_d Z_d^T Z_d  (= K^T G K, w x w)  TS kernel, sym, both transposed
//   (theta, W_k) = top-k of H (sketch_topk's eigensolver, fp64 products);  X = K W_k;
//   S = X^T (sign rule c5), lambda = theta[:k]
//
// 2q + 1 passes over the training stack, all products on the 3xTF32 tensor-core path.
#include <algorithm>
#include <cmath>
#include <vector>

#include "dense64.cuh"
#include "eig_kernels.cuh"
#include "tsk_internal.h"

namespace tsk {

static inline unsigned nb_(long long n, int t) { return (unsigned)((n + t - 1) / t); }

// inv[c] = 1/sqrt(lam[c]) when lam[c] > thr2 (a kept direction), else 0
__global__ void mf_inv_sqrt_kernel(const double* __restrict__ lam, int p, double thr2, double* __restrict__ inv) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c < p) inv[c] = lam[c] > thr2 ? 1.0 / sqrt(lam[c]) : 0.0;
}

// Z_d = A_d^T Kt^T for every d: [D][n][ldz] fp32 (X = A_d read transposed, Y = Kt [w][ms] broadcast)
static tsk_status mf_project(Ctx* ctx, const float* A, long long D, int m, int n, const float* Kt, int ms, int w,
                             float* Z, int ldz) {
  GemmProblem p;
  p.X = A;
  p.Y = Kt;
  p.M = n;
  p.N = w;
  p.n = m;
  p.D = D;
  p.xt = 1;
  p.x_row_stride = n;
  p.x_slice_stride = (long long)m * n;
  p.ybc = 1;
  p.y_row_stride = ms;
  p.y_slice_stride = ms;
  p.batch = 1;
  p.bn = w <= 64 ? 64 : 128;
  p.dout = Z;
  p.drow = 1;
  p.dstride = (long long)n * ldz;
  p.ldd = ldz;
  return gemm_tf32x3(ctx, p);
}

// Y = sum_d A_d Z_d  [m][pz] fp64  (Z: [D][n][pz], read as the transposed Y operand)
static tsk_status mf_expand(Ctx* ctx, const float* A, long long D, int m, int n, const float* Z, int pz, double* Y) {
  GemmProblem p;
  p.X = A;
  p.Y = Z;
  p.M = m;
  p.N = pz;
  p.n = n;
  p.D = D;
  p.x_row_stride = n;
  p.x_slice_stride = (long long)m * n;
  p.yt = 1;
  p.y_row_stride = pz;
  p.y_slice_stride = (long long)n * pz;
  p.bn = pz <= 64 ? 64 : 128;
  p.out64 = Y;
  p.ldo64 = pz;
  return gemm_tf32x3(ctx, p);
}

// H = sum_d Z_d^T Z_d  [w][w] fp64 (Z: [D][n][w]; symmetric, both operands read transposed)
static tsk_status mf_rr_gram(Ctx* ctx, const float* Z, long long D, int n, int w, double* H) {
  GemmProblem p;
  p.X = Z;
  p.Y = Z;
  p.M = w;
  p.N = w;
  p.n = n;
  p.D = D;
  p.xt = 1;
  p.yt = 1;
  p.x_row_stride = w;
  p.x_slice_stride = (long long)n * w;
  p.y_row_stride = w;
  p.y_slice_stride = (long long)n * w;
  p.sym = 1;
  p.out64 = H;
  p.ldo64 = w;
  return gemm_tf32x3(ctx, p);
}

tsk_status matrix_free_sketch(Ctx* ctx, const float* A, long long D, int m, int n, int k, float* S, double* lambda,
                              const tsk_mf_opts* o, tsk_mf_info* info) {
  if (D < 1 || m < 1 || n < 1 || k < 1 || k > m) return TSK_EINVAL;
  if (n % 4) return TSK_ESHAPE;
  const bool krylov = !(o && o->subspace);
  int pp = k + ((o && o->oversample > 0) ? o->oversample : 16);
  pp = (pp + 3) & ~3;
  if (pp > m) pp = m;
  if (k > pp) return TSK_EINVAL;
  const int wmax = std::min(m, 256);
  int q = (o && o->power_iters >= 0) ? o->power_iters : -1;
  if (q < 0) q = krylov ? std::min(2, wmax / pp - 1) : 2;
  if (q < 0) return TSK_EINVAL;
  const int nbk = krylov ? q + 1 : 1;  // blocks in K
  const int w = nbk * pp;
  if (w > wmax || q > 64) return TSK_EINVAL;
  const int pz = (pp + 3) & ~3;       // 16-byte pitch of the fp32 product operands
  const int wz = nbk * pz;
  const int ms = (m + 3) & ~3;
  const size_t mp = (size_t)m * pp;
  cudaStream_t s = ctx->stream;

  double* Kb = reinterpret_cast<double*>(ctx->workspace(WS_MF_K, (size_t)nbk * mp * 8));
  double* big = reinterpret_cast<double*>(ctx->workspace(WS_MF_Y, ((size_t)m * pz + 3 * mp + (size_t)m * k) * 8));
  float* Z = reinterpret_cast<float*>(ctx->workspace(WS_MF_Z, (size_t)D * n * wz * 4));
  float* Kt = reinterpret_cast<float*>(ctx->workspace(WS_MF_Q32, (size_t)wz * ms * 4));
  double* small = reinterpret_cast<double*>(
      ctx->workspace(WS_MF_SMALL, ((size_t)wz * wz + 2 * (size_t)wz * k + 3 * (size_t)pp * pp + 2 * wz + 16) * 8));
  double* hostbuf = reinterpret_cast<double*>(ctx->pinned((size_t)(wz + 16) * 8));
  if (!Kb || !big || !Z || !Kt || !small || !hostbuf) return TSK_ENOMEM;
  double *Yp = big, *Yj = big + (size_t)m * pz, *T = Yj + mp, *Q1 = T + mp, *X = Q1 + mp;
  // H [wz][wz] | W_k [wz][k] | S_H [k][wz] fp32 | C, R, Vc [pp][pp] | lam [wz] | inv [wz] | flags
  double *H = small, *W = H + (size_t)wz * wz, *C = W + 2 * (size_t)wz * k, *R = C + (size_t)pp * pp;
  double *Vc = R + (size_t)pp * pp, *lam = Vc + (size_t)pp * pp, *inv = lam + wz;
  int* flags = reinterpret_cast<int*>(inv + wz);
  tsk_status st;
  int repairs = 0;
  // zero the K^T pad rows once (q_to_f32t writes rows c < pp of each block only)
  if (cudaMemsetAsync(Kt, 0, (size_t)wz * ms * 4, s) != cudaSuccess) return TSK_ECUDA;

  // Y <- Y - sum_{i<nprev} Q_i Q_i^T Y, twice (block classical Gram-Schmidt, CGS2)
  auto project_out = [&](double* Yb, int nprev) -> tsk_status {
    for (int pass = 0; pass < 2; ++pass)
      for (int i = 0; i < nprev; ++i) {
        const double* Qi = Kb + (size_t)i * mp;
        if ((st = gemm_tn_f64(ctx, Qi, pp, 0, Yb, pp, 0, m, pp, pp, 1, C, pp, 0, 0, WS_MF_SCR)) != TSK_OK) return st;
        if ((st = gemm_nn_f64(ctx, Qi, pp, 0, C, pp, 0, m, pp, pp, 1, nullptr, T, pp, 0)) != TSK_OK) return st;
        cheb_step_kernel<<<nb_((long long)mp, 256), 256, 0, s>>>(Yb, Yb, T, (long long)mp, 0.0, 1.0, 1.0, Yb);
        ctx->count_launch();
      }
    return TSK_OK;
  };
  auto flags_failed = [&]() -> int {
    int hf[2] = {0, 0};
    if (cudaMemcpyAsync(hf, flags, sizeof(hf), cudaMemcpyDeviceToHost, s) != cudaSuccess ||
        cudaStreamSynchronize(s) != cudaSuccess)
      return -1;
    return (hf[0] | hf[1]) ? 1 : 0;
  };
  // Q (block slot) <- orth(Yb) orthogonal to the first nprev blocks.  CholQR2; on breakdown the
  // numerically dependent directions (eigenvalues of Yb^T Yb below (1e-10 ||Yb||)^2 after the
  // projection) are replaced by pseudo-random ones, projected out of K, and CholQR2 is redone.
  auto orth_block = [&](double* Yb, int nprev, double* Qout) -> tsk_status {
    cudaMemsetAsync(flags, 0, 2 * sizeof(int), s);
    if ((st = cholqr2(ctx, Yb, Q1, Qout, m, pp, C, R, flags)) != TSK_OK) return st;
    int f = flags_failed();
    if (f < 0) return TSK_ECUDA;
    if (!f) return TSK_OK;
    ++repairs;
    // rank-revealing split of the block: Yb^T Yb = V diag(l) V^T (Jacobi, decreasing l)
    if ((st = gemm_tn_f64(ctx, Yb, pp, 0, Yb, pp, 0, m, pp, pp, 1, C, pp, 0, 1, WS_MF_SCR)) != TSK_OK) return st;
    if ((st = jacobi_eig_batched(ctx, C, pp, 1, Vc, lam)) != TSK_OK) return st;
    if (cudaMemcpyAsync(hostbuf, lam, (size_t)pp * 8, cudaMemcpyDeviceToHost, s) != cudaSuccess ||
        cudaStreamSynchronize(s) != cudaSuccess)
      return TSK_ECUDA;
    const double thr2 = 1e-20 * std::max(hostbuf[0], 0.0);
    int keep = 0;
    while (keep < pp && hostbuf[keep] > thr2) ++keep;
    mf_inv_sqrt_kernel<<<nb_(pp, 128), 128, 0, s>>>(lam, pp, thr2, inv);
    ctx->count_launch();
    // kept directions Yb V diag(1/sqrt(l)) (orthonormal), dropped ones -> fresh pseudo-random columns
    if ((st = gemm_nn_f64(ctx, Yb, pp, 0, Vc, pp, 0, m, pp, pp, 1, inv, T, pp, 0)) != TSK_OK) return st;
    if (keep < pp) {
      hash_fill_kernel<<<nb_((long long)mp, 256), 256, 0, s>>>(Yb, m, pp, 0x6B72796C6F76ull + repairs, 1.0, 0);
      copy_cols_kernel<<<nb_((long long)m * keep, 256), 256, 0, s>>>(T, pp, 0, Yb, pp, 0, m, keep);
      ctx->count_launch(2);
    } else {
      cudaMemcpyAsync(Yb, T, mp * 8, cudaMemcpyDeviceToDevice, s);
    }
    if ((st = project_out(Yb, nprev)) != TSK_OK) return st;
    cudaMemsetAsync(flags, 0, 2 * sizeof(int), s);
    if ((st = cholqr2(ctx, Yb, Q1, Qout, m, pp, C, R, flags)) != TSK_OK) return st;
    f = flags_failed();
    return f == 0 ? TSK_OK : TSK_ECUDA;
  };

  // 1. Q_0 = orth(Omega)
  if (o && o->omega) {
    if (cudaMemcpyAsync(Yj, o->omega, mp * 8, cudaMemcpyDeviceToDevice, s) != cudaSuccess) return TSK_ECUDA;
  } else {
    hash_fill_kernel<<<nb_((long long)mp, 256), 256, 0, s>>>(Yj, m, pp, 0x4B72796C6F76ull, 1.0, 0);
    ctx->count_launch();
  }
  if ((st = orth_block(Yj, 0, Kb)) != TSK_OK) return st;

  // 2. power / Krylov steps
  for (int j = 1; j <= q; ++j) {
    double* Qprev = Kb + (size_t)(krylov ? j - 1 : 0) * mp;
    q_to_f32t_kernel<<<nb_((long long)pp * ms, 256), 256, 0, s>>>(Qprev, m, pp, ms, Kt);
    ctx->count_launch();
    if ((st = mf_project(ctx, A, D, m, n, Kt, ms, pz, Z, pz)) != TSK_OK) return st;
    if ((st = mf_expand(ctx, A, D, m, n, Z, pz, Yp)) != TSK_OK) return st;
    if (pz != pp) {
      copy_cols_kernel<<<nb_((long long)mp, 256), 256, 0, s>>>(Yp, pz, 0, Yj, pp, 0, m, pp);
      ctx->count_launch();
    } else {
      cudaMemcpyAsync(Yj, Yp, mp * 8, cudaMemcpyDeviceToDevice, s);
    }
    if (krylov) {
      if ((st = project_out(Yj, j)) != TSK_OK) return st;
      if ((st = orth_block(Yj, j, Kb + (size_t)j * mp)) != TSK_OK) return st;
    } else {
      if ((st = orth_block(Yj, 0, Kb)) != TSK_OK) return st;
    }
  }

  // 3. Rayleigh-Ritz on span(K) through one more pass: H = sum_d (A_d^T K)^T (A_d^T K)
  for (int b = 0; b < nbk; ++b) {
    q_to_f32t_kernel<<<nb_((long long)pp * ms, 256), 256, 0, s>>>(Kb + (size_t)b * mp, m, pp, ms,
                                                                    Kt + (size_t)b * pz * ms);
    ctx->count_launch();
  }
  if ((st = mf_project(ctx, A, D, m, n, Kt, ms, wz, Z, wz)) != TSK_OK) return st;
  if ((st = mf_rr_gram(ctx, Z, D, n, wz, H)) != TSK_OK) return st;
  // top-k eigenpairs of H: the eigensolver of sketch_topk with fp64 products (w <= 256)
  tsk_train_opts eo{};
  // H carries the 3xTF32 error of the Z_d products (~1e-6 relative, tests): a Ritz residual of 1e-9 theta_1
  // is far below it (the eigensolver's fp64 default, 1e-11, took twice the iterations)
  eo.tol = 1e-9;
  tsk_train_info ei{};
  float* Sh = reinterpret_cast<float*>(W + (size_t)wz * k);  // [k][wz] fp32 (unused output)
  if ((st = topk_eigen_ex(ctx, H, wz, k, Sh, lam, &eo, &ei, 1, W)) < 0) return st;
  hostbuf = reinterpret_cast<double*>(ctx->pinned((size_t)(wz + 16) * 8));  // the eigensolver may regrow it
  if (!hostbuf) return TSK_ENOMEM;

  // 4. X = K W_k = sum_b Q_b W_k[b pz : b pz + pp, :];  S = X^T (sign rule c5)
  for (int b = 0; b < nbk; ++b) {
    double* dst = b == 0 ? X : T;
    if ((st = gemm_nn_f64(ctx, Kb + (size_t)b * mp, pp, 0, W + (size_t)b * pz * k, k, 0, m, pp, k, 1, nullptr, dst,
                          k, 0)) != TSK_OK)
      return st;
    if (b > 0) {
      cheb_step_kernel<<<nb_((long long)m * k, 256), 256, 0, s>>>(X, X, T, (long long)m * k, 0.0, 1.0, -1.0, X);
      ctx->count_launch();
    }
  }
  write_sketch_kernel<<<k, 256, 0, s>>>(X, m, k, S);
  ctx->count_launch();
  if (lambda && cudaMemcpyAsync(lambda, lam, (size_t)k * 8, cudaMemcpyDeviceToDevice, s) != cudaSuccess)
    return TSK_ECUDA;
  if (info) {
    if (cudaMemcpyAsync(hostbuf, lam, (size_t)k * 8, cudaMemcpyDeviceToHost, s) != cudaSuccess ||
        cudaStreamSynchronize(s) != cudaSuccess)
      return TSK_ECUDA;
    double kf = 0.0;
    for (int c = 0; c < k; ++c) kf += hostbuf[c];
    info->block = pp;
    info->power_iters = q;
    info->width = w;
    info->passes = 2 * q + 1;
    info->repairs = repairs;
    info->kyfan = kf;
  }
  return launch_status("matrix_free_sketch");
}

}  // namespace tsk
